export QUIET=1 NSRC=16 REPS=3
for d in 0 4 8 16 0; do echo "dbg=$d"; timeout 300 python tools/debug_team.py 1 13 $d 2>&1 | grep "BAD"; done
