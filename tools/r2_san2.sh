mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  echo "== $tool"; timeout 1500 compute-sanitizer --tool $tool python tools/sanitize_cases.py 2>&1 | tail -18
done > gpurun_out/r02_sanitizers.log 2>&1
grep -E "==|SUMMARY|Error|MISMATCH| ok" gpurun_out/r02_sanitizers.log
