# full GPU evidence: smoke, the whole -m gpu suite, bench lines per workload
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo smoke rc=$?; tail -4 gpurun_out/r2_smoke.log
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r2_pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/r2_pytest.log
for wl in rmat20 grid2048 er4096 ba65536; do
  timeout 1200 python bench.py --workload $wl --steps 3 --warmup 3 > gpurun_out/r2_bench_$wl.json 2> gpurun_out/r2_bench_$wl.err; echo "$wl rc=$?"; head -c 300 gpurun_out/r2_bench_$wl.json; echo
done
