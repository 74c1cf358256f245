timeout 600 python -m pytest tests/test_gpu_team.py -x -q 2>&1 | tail -3
for c in 0 1 2 4 8; do echo "cluster=$c"; timeout 200 python tools/probe_perf.py --graph rmat20 --k 592 --reps 2 --param cluster=$c 2>&1 | grep "rep 1"; done
timeout 200 python tools/probe_perf.py --graph rmat20 --k 592 --reps 1 --prof --param cluster=1 2>&1 | tail -2
timeout 200 python tools/probe_perf.py --graph rmat20 --k 592 --reps 1 --prof --param cluster=4 2>&1 | tail -2
for c in 0 1 2; do echo "ba cluster=$c"; timeout 200 python tools/probe_perf.py --graph ba --k 1024 --reps 2 --param cluster=$c 2>&1 | grep "rep 1"; done
