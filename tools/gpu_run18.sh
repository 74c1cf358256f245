timeout 900 python -m pytest tests/test_gpu_team.py -q -x -k "k or warp" 2>&1 | tail -15
timeout 900 python -m pytest tests/test_gpu_team.py tests/test_gpu_parity.py -q 2>&1 | tail -3
echo grid; timeout 300 python tools/probe_perf.py --graph grid2048 --k 1024 --reps 1 --prof 2>&1 | grep -A2 "rep 0"
echo grid8; timeout 300 python tools/probe_perf.py --graph grid2048 --k 8 --reps 1 --prof --param slots=8 2>&1 | grep -A2 "rep 0" | tail -2
