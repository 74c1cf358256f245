timeout 900 ncu --set full --clock-control none --import-source on -k regex:bc_team -s 1 -c 1 -o gpurun_out/r01_team_rmat20 python tools/probe_perf.py --graph rmat20 --k 296 --reps 2 > gpurun_out/prof2.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches_rmat20_team.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline >> gpurun_out/prof2.log 2>&1
tail -3 gpurun_out/prof2.log
