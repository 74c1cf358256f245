export QUIET=1 NSRC=16 REPS=3
for c in 1 2 4; do echo "c=$c"; timeout 300 python tools/debug_team.py $c 13 2>&1 | grep "BAD"; done
timeout 900 python -m pytest tests/test_gpu_team.py -q 2>&1 | tail -3
WBC_GPU_CLUSTER=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q 2>&1 | tail -3
WBC_GPU_CLUSTER=2 timeout 900 python -m pytest tests/test_gpu_parity.py -q 2>&1 | tail -3
for c in 1 2 4; do echo "cluster=$c"; timeout 200 python tools/probe_perf.py --graph rmat20 --k 592 --reps 2 --param cluster=$c 2>&1 | grep "rep 1"; done
for c in 1 2; do echo "ba cluster=$c"; timeout 200 python tools/probe_perf.py --graph ba --k 1024 --reps 2 --param cluster=$c 2>&1 | grep "rep 1"; done
for c in 0 1; do echo "er cluster=$c"; timeout 200 python tools/probe_perf.py --graph er --k 4093 --reps 2 --param cluster=$c 2>&1 | grep "rep 1"; done
