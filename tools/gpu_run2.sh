set -x
timeout 600 python -m pytest tests/test_gpu_team.py -x -q 2>&1 | tail -15
for c in 0 1 2 4 8 16; do timeout 200 python tools/probe_perf.py --graph rmat20 --k 592 --reps 2 --param cluster=$c 2>&1 | grep rep; done
timeout 200 python tools/probe_perf.py --graph rmat20 --k 592 --reps 1 --prof --param cluster=8 2>&1 | tail -3
for c in 1 2 4; do timeout 200 python tools/probe_perf.py --graph ba --k 1024 --reps 2 --param cluster=$c 2>&1 | grep rep; done
