mkdir -p gpurun_out/s4
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_rasm_setup_tc2 -c 1 -o gpurun_out/s4/tc2 python tools/prof_setup.py 2 > gpurun_out/s4/ncu.log 2>&1; tail -3 gpurun_out/s4/ncu.log
ncu -i gpurun_out/s4/tc2.ncu-rep --page raw --csv > gpurun_out/s4/raw.csv 2>/dev/null
ncu -i gpurun_out/s4/tc2.ncu-rep --page source --print-source cuda,sass --csv > gpurun_out/s4/src.csv 2>/dev/null
python tools/ncu_kernel_summary.py gpurun_out/s4/raw.csv
python tools/ncu_line_summary.py gpurun_out/s4/src.csv 40 > gpurun_out/s4/lines.txt
python tools/ncu_sass_hot.py gpurun_out/s4/src.csv 40 > gpurun_out/s4/sass.txt
