timeout 1800 python bench.py --workload rmat24 --sources 592 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_rmat24.json 2> gpurun_out/bench_rmat24.err
echo "rmat24 rc=$?"; cat gpurun_out/bench_rmat24.json
timeout 600 python bench.py --workload er4096 --steps 3 --warmup 3 > gpurun_out/bench_er4096.json 2> gpurun_out/bench_er4096.err
echo "er rc=$?"; tail -c 700 gpurun_out/bench_er4096.json
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
