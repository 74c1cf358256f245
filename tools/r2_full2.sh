bash tools/r2_full.sh
for tool in memcheck racecheck synccheck; do
  echo "== $tool"; timeout 1500 compute-sanitizer --tool $tool python tools/sanitize_cases.py 2>&1 | tail -16
done > gpurun_out/r02_sanitizers.log 2>&1
grep -E "==|SUMMARY|Error|MISMATCH" gpurun_out/r02_sanitizers.log
