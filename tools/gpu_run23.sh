timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench23.json 2> gpurun_out/bench23.err; tail -c 2500 gpurun_out/bench23.json
echo ba; timeout 200 python tools/probe_perf.py --graph ba --k 1024 --reps 2 2>&1 | grep "rep 1"
echo er; timeout 200 python tools/probe_perf.py --graph er --k 4093 --reps 2 2>&1 | grep "rep 1"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bc_team -s 1 -c 1 -o gpurun_out/r01_team_rmat20_v2 python tools/probe_perf.py --graph rmat20 --k 296 --reps 2 > gpurun_out/prof23.log 2>&1; tail -2 gpurun_out/prof23.log
