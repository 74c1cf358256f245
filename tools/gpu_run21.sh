timeout 600 python -m pytest tests/test_cli.py -q 2>&1 | tail -3
nproc; free -g | head -2
timeout 2400 python tools/probe_multi.py --graph rmat24 --k 296 --clusters 2,4,8,16 2>&1 | tail -8
