for i in 1 2 3; do timeout 120 python tools/tc2_ab.py 2 2>&1 | grep -v "^$" | tail -3; echo "rc=$?"; done
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
