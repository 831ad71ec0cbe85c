mkdir -p gpurun_out/s4
timeout 300 python tools/mv_ab.py 2 1:1 1:0 2:0 2:1 > gpurun_out/s4/ab.log 2>&1
cat gpurun_out/s4/ab.log | grep -v "^$"
P="python tools/prof_cfg2.py 2"
timeout 300 $P > gpurun_out/s4/plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_matvec' -c 2 -o gpurun_out/s4/mv $P > gpurun_out/s4/ncu.log 2>&1; tail -2 gpurun_out/s4/ncu.log
