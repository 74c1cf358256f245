# final refresh: smoke, gpu suite, bench lines, ncu of the kernels changed since the last evidence run
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo smoke rc=$?; tail -3 gpurun_out/r2_smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2_pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/r2_pytest.log
for wl in rmat20 grid2048 er4096 ba65536; do
  timeout 1200 python bench.py --workload $wl --steps 3 --warmup 3 > gpurun_out/r2_bench_$wl.json 2> gpurun_out/r2_bench_$wl.err; echo "$wl rc=$?"; head -c 250 gpurun_out/r2_bench_$wl.json; echo
done
timeout 1800 python bench.py --workload rmat24 --sources 296 --steps 2 --warmup 3 > gpurun_out/r2_bench_rmat24.json 2> gpurun_out/r2_bench_rmat24.err; echo "rmat24 rc=$?"; head -c 250 gpurun_out/r2_bench_rmat24.json; echo
R=/tmp/ncu_reps; mkdir -p $R
NCU="timeout 1200 ncu --set full --clock-control none --import-source on"
$NCU -k regex:bc_flat -s 1 -c 1 -o $R/r02_ncu_flat_grid2048 python tools/probe_perf.py --graph grid2048 --k 148 --reps 2 > gpurun_out/ncu_grid.log 2>&1; echo ncu grid $?
python tools/ncu_summarize.py $R/r02_ncu_flat_grid2048.ncu-rep --sources 148 > gpurun_out/r02_ncu_flat_grid2048.md
$NCU -k regex:bc_team -s 1 -c 1 -o $R/r02_ncu_team_ba65536 python tools/probe_perf.py --graph ba --k 296 --reps 2 > gpurun_out/ncu_ba.log 2>&1; echo ncu ba $?
python tools/ncu_summarize.py $R/r02_ncu_team_ba65536.ncu-rep --sources 296 > gpurun_out/r02_ncu_team_ba65536.md
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches_grid2048.csv python bench.py --workload grid2048 --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo launches grid $?
grep -h "DRAM traffic per source" gpurun_out/r02_ncu_*.md
