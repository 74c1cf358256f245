timeout 600 python tools/probe_multi.py --graph rmat20 --k 592 --clusters 2 --nears 0,1,2,4,8,16 2>&1 | tail -7
timeout 600 python tools/probe_multi.py --graph ba --k 1024 --clusters 1 --nears 0,1,2,4,8,16,32 2>&1 | tail -8
timeout 2400 python tools/probe_multi.py --graph rmat24 --k 296 --clusters 16 --nears 0,4,8,38,76 2>&1 | tail -6
