#!/bin/bash
# Round-2 (second half) evidence: bench line (cfg4, no flags), reference arm, pytest -m gpu,
# smoke, and the cfg4 launch list with the host-driven solve loop (profiles/r02_*).
O=gpurun_out/${TAG:-f2}
mkdir -p $O
nproc > $O/nproc.txt; nvidia-smi > $O/nvsmi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.txt 2>&1; echo "rc=$?" >> $O/smoke.txt
timeout 900 python bench.py > $O/bench_cfg4.log 2>&1; echo "rc=$?" >> $O/bench_cfg4.log
timeout 900 python bench.py --impl reference > $O/bench_ref.log 2>&1; echo "rc=$?" >> $O/bench_ref.log
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
RBF_BENCH_NO_GRAPH=1 timeout 900 $CMD > $O/plain_nog.log 2>&1 && \
RBF_BENCH_NO_GRAPH=1 timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg4_hostloop.csv $CMD > $O/ncu_launch.log 2>&1
echo "launch rc=$?" >> $O/ncu_launch.log
