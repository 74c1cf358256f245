timeout 1200 python -m pytest tests/test_gpu_team.py tests/test_gpu_parity.py -q -x 2>&1 | tail -2
timeout 600 python tools/probe_multi.py --graph rmat20 --k 592 --clusters 2,4 --nears 16 2>&1 | tail -2
timeout 600 python tools/probe_multi.py --graph ba --k 1024 --clusters 1 --nears 8 2>&1 | tail -1
echo grid; timeout 300 python tools/probe_perf.py --graph grid2048 --k 622 --reps 1 2>&1 | grep "rep 0"
