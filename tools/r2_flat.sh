mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_flat.py tests/test_gpu_sigma.py -x -q > gpurun_out/flat_tests.log 2>&1; echo tests rc=$?; tail -4 gpurun_out/flat_tests.log
WBC_LIB=paper_1701_05975_b200/lib_var/libwbc_ssp.so timeout 600 python tools/probe_perf.py --graph grid2048 --k 148 --reps 2 --prof 2>&1 | grep -E "^rep|per source" | tail -2 | sed 's/abort_near.*//'
bash tools/r2_ab.sh "--graph grid2048 --k 1024 --reps 2 --prof" default
