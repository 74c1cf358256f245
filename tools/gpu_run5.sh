timeout 300 python tools/debug_team.py 1 13 2>&1 | tail -12
timeout 300 python tools/debug_team.py 4 13 2>&1 | tail -9
timeout 600 compute-sanitizer --tool racecheck --print-limit 5 python tools/debug_team.py 1 11 2>&1 | tail -30
