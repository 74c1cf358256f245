timeout 600 python tools/probe_multi.py --graph rmat20 --k 592 --clusters 2 --nears 0,16 2>&1 | tail -2
timeout 600 python tools/probe_multi.py --graph ba --k 1024 --clusters 1 --nears 0,8 2>&1 | tail -2
