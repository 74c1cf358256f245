timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q 2>&1 | tail -4
timeout 1500 python tools/check_rmat24.py 2>&1 | tail -5
