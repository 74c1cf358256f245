timeout 300 python tools/debug_team.py 1 13 2>&1 | tail -8
timeout 600 python -m pytest tests/test_gpu_team.py -x -q 2>&1 | tail -3
for c in 1 2 4; do echo "cluster=$c"; timeout 200 python tools/probe_perf.py --graph rmat20 --k 592 --reps 2 --param cluster=$c 2>&1 | grep "rep 1"; done
