timeout 900 python -m pytest tests/test_gpu_team.py -q -x 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
for c in 1 2 4; do echo "cluster=$c"; timeout 200 python tools/probe_perf.py --graph rmat20 --k 592 --reps 2 --param cluster=$c 2>&1 | grep "rep 1"; done
for c in 1 2; do echo "ba cluster=$c"; timeout 200 python tools/probe_perf.py --graph ba --k 1024 --reps 2 --param cluster=$c 2>&1 | grep "rep 1"; done
timeout 200 python tools/probe_perf.py --graph rmat20 --k 592 --reps 1 --prof --param cluster=2 2>&1 | tail -2
