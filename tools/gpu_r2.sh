#!/bin/bash
# Round-2 GPU session: tests, bench (cfg4 default + cfg2), launch list, ncu captures.
# Usage (repo root, under gpurun): TAG=x bash tools/gpu_r2.sh
tag=${TAG:-s}
O=gpurun_out/$tag
mkdir -p $O
nproc > $O/nproc.txt; lscpu | head -20 >> $O/nproc.txt; free -g >> $O/nproc.txt; nvidia-smi > $O/nvsmi.txt 2>&1
if [ "${TESTS:-1}" = "1" ]; then
  timeout 600 python -m pytest tests/test_gpu_parity_r2.py -x -q > $O/pytest_r2.log 2>&1; echo "rc=$?" >> $O/pytest_r2.log
  timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
fi
if [ "${BENCH:-1}" = "1" ]; then
  timeout 900 python bench.py --steps 5 --warmup 3 > $O/bench.log 2>&1; echo "bench rc=$?" >> $O/bench.log
  timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_cfg2.log 2>&1; echo "rc=$?" >> $O/bench_cfg2.log
fi
if [ "${NCU:-1}" = "1" ]; then
  CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg4.csv $CMD > $O/ncu_launch.log 2>&1
  echo "launch rc=$?" >> $O/ncu_launch.log
  P4="python tools/prof_cfg2.py 4 --no-graph"
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
     -k regex:'k_matvec|k_rasm_apply|k_rasm_setup_tc|k_axpy_dot|k_arnoldi' -c 12 --csv --log-file $O/dram_cfg4.csv $P4 > $O/ncu_dram4.log 2>&1
  echo "dram rc=$?" >> $O/ncu_dram4.log
  P2="python tools/prof_cfg2.py 2 --no-graph"
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'k_matvec|k_rasm_apply|k_rasm_setup_tc|k_arnoldi_mgs2' -c 8 -o $O/prof2 $P2 > $O/ncu_full.log 2>&1
  echo "full rc=$?" >> $O/ncu_full.log
fi
