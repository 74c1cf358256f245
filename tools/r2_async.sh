mkdir -p gpurun_out
WBC_LIB=paper_1701_05975_b200/lib_var/libwbc_async.so timeout 600 python -m pytest tests/test_gpu_flat.py tests/test_gpu_sigma.py -x -q > gpurun_out/async_tests.log 2>&1; echo async tests rc=$?; tail -4 gpurun_out/async_tests.log
bash tools/r2_ab.sh "--graph grid2048 --k 1024 --reps 2 --prof" default async
