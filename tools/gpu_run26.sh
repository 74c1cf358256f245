timeout 900 python -m pytest tests/test_gpu_team.py -q -x 2>&1 | tail -2
echo grid; timeout 300 python tools/probe_perf.py --graph grid2048 --k 1024 --reps 1 2>&1 | grep "rep 0"
timeout 600 python tools/probe_multi.py --graph rmat20 --k 592 --clusters 2 --nears 16 --l2hots=-1,300000,150000 2>&1 | tail -3
timeout 2400 python tools/probe_multi.py --graph rmat24 --k 296 --clusters 8,16 --nears 8 --l2hots=-1,4000000,2000000,1000000 2>&1 | tail -9
