TC2=2 timeout 120 python tools/probe_setup.py 2 2>&1 | grep "tc3\|rror" | head -3 || exit 1
TC2=2 PROBE_LIB=librbf_nopost.so timeout 120 python tools/probe_setup.py 2 2>&1 | grep "tc3\|rror" | head -3
KERNELS=0,2 timeout 300 python tools/tc2_ab.py 2 3 2>&1 | grep -v "^$"
timeout 300 python -m pytest tests -m gpu -x -q -k "two_per_sm" 2>&1 | tail -2
