mkdir -p gpurun_out/s5
TC2=1 timeout 300 python tools/probe_setup.py 2 2>&1 | grep tc2
timeout 600 python tools/tc2_ab.py 2 3 2>&1 | grep -v "^$"
