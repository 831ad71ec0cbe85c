TC2=1 timeout 300 python tools/probe_setup.py 2 2>&1 | grep -v "^\[probe\]\|^{"
