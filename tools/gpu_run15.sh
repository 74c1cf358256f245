timeout 900 python -m pytest tests/test_gpu_team.py tests/test_gpu_parity.py -q -x 2>&1 | tail -2
for sl in 8 553; do echo "grid warp slots=$sl"; timeout 300 python tools/probe_perf.py --graph grid2048 --k $sl --reps 1 --prof --param cluster=1 --param threads=32 --param slots=$sl 2>&1 | grep -A2 "rep 0"; done
echo "rmat20 c2"; timeout 200 python tools/probe_perf.py --graph rmat20 --k 592 --reps 2 2>&1 | grep "rep 1"
echo "ba"; timeout 200 python tools/probe_perf.py --graph ba --k 1024 --reps 2 2>&1 | grep "rep 1"
echo "er warp"; timeout 200 python tools/probe_perf.py --graph er --k 4093 --reps 2 --param cluster=1 --param threads=32 2>&1 | grep "rep 1"
