set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
for gr in er ba rmat20; do timeout 300 python tools/probe_perf.py --graph $gr --k 1024 --prof --reps 2 2>&1 | tail -6; done
timeout 600 python tools/probe_perf.py --graph grid2048 --k 296 --prof --reps 1 2>&1 | tail -6
