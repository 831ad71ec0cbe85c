#!/bin/bash
# Quick iteration on the GPU: parity tests, setup probe, short cfg2/cfg4 bench lines.
tag=${TAG:-it}
O=gpurun_out/$tag
mkdir -p $O
timeout 900 python -m pytest ${TESTS:-tests/test_gpu_parity_r2.py tests/test_gpu_parity.py tests/test_gpu_poison.py} -m gpu -x -q -rs > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
if [ -f tools/probe/librbf.so ] && [ "${PROBE:-1}" = "1" ]; then
  timeout 300 python tools/probe_setup.py 2 > $O/probe_cfg2.txt 2>&1
fi
if [ "${DIAG:-0}" = "1" ]; then
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/diag_bench tools/diag_bench.cu && /tmp/diag_bench > $O/diag_bench.txt 2>&1
fi
timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_cfg2.log 2>&1
if [ "${CFG4:-1}" = "1" ]; then
  timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_cfg4.log 2>&1
fi
