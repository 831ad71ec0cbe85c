timeout 60 python tools/smoke_setup.py 1 || { echo "SMOKE FAILED"; exit 1; }
timeout 300 python -m pytest tests -m gpu -x -q -k "two_per_sm" 2>&1 | tail -3
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
