timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 600 python bench.py --workload er4096 --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('er', d['value'], d['e2e'])"
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('rmat20', d['value'], d['e2e'], d['roofline']['frac'])"
