TC2=2 PROBE_LIB=librbf_nopost.so timeout 120 python tools/probe_setup.py 2 2>&1 | grep "tc3\|rror" | head -3
