timeout 60 python tools/smoke_setup.py 1 || { echo "SMOKE FAILED"; exit 1; }
timeout 600 python tools/tc2_ab.py 4 5 2>&1 | grep -v "^$"
