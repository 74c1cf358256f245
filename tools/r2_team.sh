mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_team.py tests/test_gpu_parity.py -x -q > gpurun_out/team_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/team_tests.log
for g in "rmat20 --k 2048" "ba --k 4096" "rmat24 --k 296"; do echo "== $g"; timeout 900 python tools/probe_perf.py --graph $g --reps 3 2>&1 | grep -E "^rep" | tail -1; done
