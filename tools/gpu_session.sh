#!/bin/bash
# One gpurun session: build check, GPU tests, bench, launch list and a full ncu capture.
# Usage (from the repo root, under gpurun): bash tools/gpu_session.sh [tag]
tag=${1:-s}
O=gpurun_out/$tag
mkdir -p $O
nproc > $O/nproc.txt; lscpu | head -20 >> $O/nproc.txt; nvidia-smi > $O/nvsmi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py --steps 5 --warmup 3 > $O/bench.log 2>&1; echo "bench rc=$?" >> $O/bench.log
if [ "${NCU:-1}" = "1" ]; then
  CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
  timeout 600 $CMD > $O/plain.log 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $CMD > $O/ncu_launch.log 2>&1
  echo "launch rc=$?" >> $O/ncu_launch.log
  # the same with the host-driven GMRES loop (same kernels, listed one by one)
  RBF_BENCH_NO_GRAPH=1 timeout 600 $CMD > $O/plain_nog.log 2>&1 && \
  RBF_BENCH_NO_GRAPH=1 timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_nograph.csv $CMD > $O/ncu_launch_nog.log 2>&1
  echo "launch nograph rc=$?" >> $O/ncu_launch_nog.log
  P="python tools/prof_cfg2.py 2 --no-graph"
  timeout 300 $P > $O/plain2.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'k_matvec|k_rasm_apply|k_rasm_setup_tc|k_arnoldi_fused|k_arnoldi_mgs2|k_nlist|k_pack_w' -c 16 -o $O/prof $P > $O/ncu_full.log 2>&1
  echo "full rc=$?" >> $O/ncu_full.log
fi
