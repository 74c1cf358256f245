# flat kernel v2 checks (one gpurun call)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_flat.py tests/test_gpu_sigma.py -x -q > gpurun_out/flat_tests.log 2>&1; echo tests rc=$?; tail -15 gpurun_out/flat_tests.log
timeout 300 python tools/probe_perf.py --graph grid512 --k 296 --reps 2 --prof 2>&1 | tail -6
timeout 600 python tools/probe_perf.py --graph grid2048 --k 296 --reps 2 --prof 2>&1 | tail -6
timeout 600 python tools/probe_perf.py --graph grid2048 --k 1024 --reps 2 2>&1 | tail -3
