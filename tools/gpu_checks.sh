# One gpurun call's worth of round-end evidence (run from the repo root):
#   gpurun --timeout 3600 -- 'mkdir -p gpurun_out; bash tools/gpu_checks.sh > gpurun_out/checks.log 2>&1'
set -x
python -c "import __graft_entry__ as g; g.smoke()"
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_rmat20.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_rmat20.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bc_team -s 1 -c 1 \
  -o gpurun_out/team_rmat20 python tools/probe_perf.py --graph rmat20 --k 296 --reps 2 > /dev/null
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool python tools/sanitize_cases.py 2>&1 | tail -3
done
for wl in er4096 ba65536 grid2048; do
  timeout 1200 python bench.py --workload $wl --steps 3 --warmup 3 > gpurun_out/bench_$wl.json
done
timeout 1800 python bench.py --workload rmat24 --sources 592 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_rmat24.json
