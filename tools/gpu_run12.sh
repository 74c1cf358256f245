timeout 900 python -m pytest tests/test_gpu_team.py tests/test_gpu_parity.py -q -x 2>&1 | tail -2
for c in 2 4; do echo "cluster=$c"; timeout 200 python tools/probe_perf.py --graph rmat20 --k 592 --reps 2 --param cluster=$c 2>&1 | grep "rep 1"; done
echo ba; timeout 200 python tools/probe_perf.py --graph ba --k 1024 --reps 2 2>&1 | grep "rep 1"
timeout 200 python tools/probe_perf.py --graph rmat20 --k 592 --reps 1 --prof --param cluster=2 2>&1 | tail -1
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench12.json 2> gpurun_out/bench12.err; tail -c 3000 gpurun_out/bench12.json
