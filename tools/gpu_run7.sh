for d in 0 1 2 3; do echo "dbg=$d"; timeout 300 python tools/debug_team.py 1 13 $d 2>&1 | grep "bad dist"; done
