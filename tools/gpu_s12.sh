timeout 60 python tools/smoke_setup.py 1 || { echo "SMOKE FAILED"; exit 1; }
TC2=1 timeout 120 python tools/probe_setup.py 2 2>&1 | grep -v "^\[probe\]\|^{" | grep -A12 "tc2:\|W phase" | head -20
timeout 300 python tools/tc2_ab.py 2 3 2>&1 | grep -v "^$"
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
