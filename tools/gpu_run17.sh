nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv
for i in 1 2; do timeout 200 python tools/probe_perf.py --graph rmat20 --k 592 --reps 2 2>&1 | grep "rep 1"; done
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['clocks'], d['roofline']['kernel'])"
