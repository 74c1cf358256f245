timeout 600 python -m pytest tests/test_gpu_team.py -q -k "hub or grid or random" 2>&1 | grep -E "Error|assert|passed|failed|FAILED" | head -30
