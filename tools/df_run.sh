mkdir -p gpurun_out/df1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "rasm_apply_parity or solve_parity_cfg1 or big_rasm or paper_geometry or large_own or lu_pivot or poison" > gpurun_out/df1/pytest_quick.log 2>&1; echo rc=$? >> gpurun_out/df1/pytest_quick.log
timeout 300 python tools/probe_setup.py 2 > gpurun_out/df1/probe_df.txt 2>&1
RBF_SETUP_V1=1 timeout 300 python tools/probe_setup.py 2 > gpurun_out/df1/probe_v1.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/df1/pytest_all.log 2>&1; echo rc=$? >> gpurun_out/df1/pytest_all.log
