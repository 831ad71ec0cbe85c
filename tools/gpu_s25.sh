which compute-sanitizer; ls /usr/local/cuda/bin/compute-sanitizer
timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --print-limit 5 python tools/smoke_setup.py 1 2>&1 | tail -5
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 5 python tools/smoke_setup.py 1 2>&1 | tail -8
