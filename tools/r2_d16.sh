timeout 900 python -m pytest tests/test_gpu_team.py -x -q -k "dist16 or fill or random_equivalence or hub" > gpurun_out/d16_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/d16_tests.log
for g in rmat20 ba; do for d in 0 1; do echo "== $g dist16=$d"; timeout 600 python tools/probe_perf.py --graph $g --k 2048 --reps 2 --param dist16=$d 2>&1 | grep -E "^rep" | tail -1; done; done
for d in 0 1; do echo "== rmat24 dist16=$d"; timeout 900 python tools/probe_perf.py --graph rmat24 --k 296 --reps 2 --param dist16=$d 2>&1 | grep -E "^rep" | tail -1; done
