mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_flat.py -x -q > gpurun_out/flat_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/flat_tests.log
bash tools/r2_ab.sh "--graph grid2048 --k 1024 --reps 2 --prof" default
