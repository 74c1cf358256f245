mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_flat.py tests/test_gpu_sigma.py -x -q > gpurun_out/flat_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/flat_tests.log
for tool in memcheck racecheck synccheck; do
  echo "== $tool"; timeout 1500 compute-sanitizer --tool $tool python tools/sanitize_cases.py 2>&1 | tail -14
done > gpurun_out/r02_sanitizers.log 2>&1
grep -E "==|SUMMARY|Error" gpurun_out/r02_sanitizers.log
bash tools/r2_ab.sh "--graph grid2048 --k 1024 --reps 2" default
