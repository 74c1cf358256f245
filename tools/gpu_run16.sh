timeout 900 python -m pytest tests/ -m gpu -q -x 2>&1 | tail -2
echo grid; timeout 300 python tools/probe_perf.py --graph grid2048 --k 553 --reps 1 --prof 2>&1 | grep -A2 "rep 0"
echo grid8; timeout 300 python tools/probe_perf.py --graph grid2048 --k 8 --reps 1 --prof --param slots=8 2>&1 | grep -A2 "rep 0" | tail -1
echo "rmat20"; timeout 200 python tools/probe_perf.py --graph rmat20 --k 592 --reps 2 2>&1 | grep "rep 1"
echo "er"; timeout 200 python tools/probe_perf.py --graph er --k 4093 --reps 2 2>&1 | grep "rep 1"
