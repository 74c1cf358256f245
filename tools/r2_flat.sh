# flat kernel checks (one gpurun call)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_flat.py tests/test_gpu_sigma.py -x -q > gpurun_out/flat_tests.log 2>&1; echo tests rc=$?; tail -4 gpurun_out/flat_tests.log
for t in 512 1024; do
timeout 600 python tools/probe_perf.py --graph grid2048 --k 1024 --reps 2 --prof --param flat_threads=$t 2>&1 | grep -E "^rep|phase share|per source" | tail -3
done
