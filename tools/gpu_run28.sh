python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
for tool in memcheck racecheck synccheck; do
  echo "== $tool"; timeout 1200 compute-sanitizer --tool $tool --print-limit 10 python tools/sanitize_cases.py 2>&1 | tail -12
done
