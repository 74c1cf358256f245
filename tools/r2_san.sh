mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "dyadic" > gpurun_out/dyadic.log 2>&1; echo dyadic rc=$?; tail -2 gpurun_out/dyadic.log
for tool in memcheck racecheck synccheck; do
  echo "== $tool"; timeout 1500 compute-sanitizer --tool $tool python tools/sanitize_cases.py 2>&1 | tail -16
done > gpurun_out/r02_sanitizers.log 2>&1
tail -60 gpurun_out/r02_sanitizers.log
