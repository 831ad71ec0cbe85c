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
# per-launch DRAM bytes and pipe activity of the cfg4 hot kernels (roofline traffic), and
# one ncu --set full capture of the hot kernels on cfg2
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none \
   -k regex:'k_matvec|k_rasm_apply|k_rasm_setup_tc|k_axpy_dot|k_nlist' -c 14 --csv --log-file $O/dram_cfg4.csv python tools/prof_cfg2.py 4 --no-graph > $O/ncu_dram4.log 2>&1
echo "dram rc=$?" >> $O/ncu_dram4.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'k_matvec|k_rasm_apply|k_rasm_setup_tc|k_arnoldi_mgs2|k_axpy_dot|k_evaluate' -c 10 -o $O/prof2 python tools/prof_cfg2.py 2 --no-graph > $O/ncu_full.log 2>&1
echo "full rc=$?" >> $O/ncu_full.log
ncu -i $O/prof2.ncu-rep --page raw --csv > $O/prof2_raw.csv 2>/dev/null
python tools/ncu_kernel_summary.py $O/prof2_raw.csv > $O/prof2_summary.txt 2>&1
