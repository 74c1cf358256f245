timeout 900 python -m pytest tests/test_gpu_team.py -q -x 2>&1 | tail -3
echo grid8; timeout 300 python tools/probe_perf.py --graph grid2048 --k 8 --reps 1 --prof --param slots=8 2>&1 | grep -A3 "rep 0"
echo grid; timeout 300 python tools/probe_perf.py --graph grid2048 --k 1024 --reps 1 --prof 2>&1 | grep -A3 "rep 0"
