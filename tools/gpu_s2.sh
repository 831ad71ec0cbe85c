mkdir -p gpurun_out/s2
timeout 600 python tools/tc2_ab.py 1 2 3 > gpurun_out/s2/ab.txt 2>&1; cat gpurun_out/s2/ab.txt | tail -12
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s2/pytest.log 2>&1; tail -15 gpurun_out/s2/pytest.log
