# ncu evidence for every bench kernel (one gpurun call); reports land in gpurun_out/
mkdir -p gpurun_out
NCU="timeout 1200 ncu --set full --clock-control none --import-source on"
$NCU -k regex:bc_team -s 2 -c 1 -o gpurun_out/r02_ncu_rmat20 python tools/probe_perf.py --graph rmat20 --k 512 --reps 2 > gpurun_out/r02_ncu_rmat20.log 2>&1; echo rmat20 $?
$NCU -k regex:bc_team -s 2 -c 1 -o gpurun_out/r02_ncu_ba python tools/probe_perf.py --graph ba --k 296 --reps 2 > gpurun_out/r02_ncu_ba.log 2>&1; echo ba $?
$NCU -k regex:bc_sources -s 2 -c 1 -o gpurun_out/r02_ncu_er python tools/probe_perf.py --graph er --k 4093 --reps 2 > gpurun_out/r02_ncu_er.log 2>&1; echo er $?
$NCU -k regex:bc_flat -s 1 -c 1 -o gpurun_out/r02_ncu_grid2048 python tools/probe_perf.py --graph grid2048 --k 148 --reps 2 > gpurun_out/r02_ncu_grid.log 2>&1; echo grid $?
$NCU -k regex:bc_team -s 1 -c 1 -o gpurun_out/r02_ncu_rmat24 python tools/probe_perf.py --graph rmat24 --k 7 --reps 2 > gpurun_out/r02_ncu_rmat24.log 2>&1; echo rmat24 $?
for wl in rmat20 grid2048; do
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches_$wl.csv python bench.py --workload $wl --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo launches $wl $?
done
