# One bench line per BASELINE config (1 GPU); rmat24 on a 592-source sample.
for wl in rmat20 er4096 ba65536 grid2048; do
  timeout 1200 python bench.py --workload $wl --steps 3 --warmup 3 > gpurun_out/bench_$wl.json 2> gpurun_out/bench_$wl.err
  echo "$wl rc=$?"; tail -c 400 gpurun_out/bench_$wl.json
done
timeout 1800 python bench.py --workload rmat24 --sources 592 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_rmat24.json 2> gpurun_out/bench_rmat24.err
echo "rmat24 rc=$?"; tail -c 400 gpurun_out/bench_rmat24.json
