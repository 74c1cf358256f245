# full GPU evidence: smoke, the whole -m gpu suite, bench lines per workload, BA/ER ncu
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo smoke rc=$?; tail -4 gpurun_out/r2_smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2_pytest.log 2>&1; echo pytest rc=$?; tail -5 gpurun_out/r2_pytest.log
for wl in rmat20 grid2048 er4096 ba65536; do
  timeout 1200 python bench.py --workload $wl --steps 3 --warmup 3 > gpurun_out/r2_bench_$wl.json 2> gpurun_out/r2_bench_$wl.err; echo "$wl rc=$?"; head -c 250 gpurun_out/r2_bench_$wl.json; echo
done
timeout 1800 python bench.py --workload rmat24 --sources 296 --steps 2 --warmup 3 > gpurun_out/r2_bench_rmat24.json 2> gpurun_out/r2_bench_rmat24.err; echo "rmat24 rc=$?"; head -c 250 gpurun_out/r2_bench_rmat24.json; echo
NCU="timeout 1200 ncu --set full --clock-control none --import-source on"
$NCU -k regex:bc_team -s 1 -c 1 -o gpurun_out/r02_ncu_ba python tools/probe_perf.py --graph ba --k 296 --reps 2 > gpurun_out/r02_ncu_ba.log 2>&1; echo ba $?
$NCU -k regex:bc_sources -s 1 -c 1 -o gpurun_out/r02_ncu_er python tools/probe_perf.py --graph er --k 4093 --reps 2 > gpurun_out/r02_ncu_er.log 2>&1; echo er $?
