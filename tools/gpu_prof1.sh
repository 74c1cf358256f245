timeout 900 ncu --set full --clock-control none --import-source on -k regex:bc_team -s 1 -c 1 -o gpurun_out/team_c2 python tools/probe_perf.py --graph rmat20 --k 296 --reps 2 --param cluster=2 > gpurun_out/prof1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bc_team -s 1 -c 1 -o gpurun_out/team_ba python tools/probe_perf.py --graph ba --k 1024 --reps 2 >> gpurun_out/prof1.log 2>&1
ls -la gpurun_out
