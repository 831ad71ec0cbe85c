mkdir -p gpurun_out/s1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/s1/smi.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s1/pytest.log 2>&1; tail -3 gpurun_out/s1/pytest.log
timeout 300 python tools/probe_setup.py 2 > gpurun_out/s1/probe_cfg2.txt 2>&1; head -12 gpurun_out/s1/probe_cfg2.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s1/bench.log 2>&1; tail -1 gpurun_out/s1/bench.log | cut -c1-600
