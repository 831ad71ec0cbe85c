timeout 60 python tools/smoke_setup.py 1 || { echo "SMOKE FAILED"; exit 1; }
TC2=0 timeout 120 python tools/probe_setup.py 2 2>&1 | grep -v "^{" | grep -A40 "^assembly" | head -40
KERNELS=0 timeout 300 python tools/tc2_ab.py 2 3 4 2>&1 | grep -v "^$"
timeout 700 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
