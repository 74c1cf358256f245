timeout 900 ncu --set full --clock-control none --import-source on -k regex:bc_warp -s 1 -c 1 -o gpurun_out/warp_grid1024 python tools/probe_perf.py --graph grid1024 --k 16 --reps 2 --param slots=16 > gpurun_out/prof3.log 2>&1
tail -3 gpurun_out/prof3.log
