mkdir -p gpurun_out/s3
TC2=1 timeout 300 python tools/probe_setup.py 2 > gpurun_out/s3/probe_tc2_cfg2.txt 2>&1; tail -3 gpurun_out/s3/probe_tc2_cfg2.txt
