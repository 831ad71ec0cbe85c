#!/bin/bash
# quick GPU check: GPU tests, matvec timing on cfg2/cfg3, bench (no cpu baseline)
mkdir -p gpurun_out/q
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/q/pytest.log 2>&1; tail -3 gpurun_out/q/pytest.log
for cfg in ${CFGS:-2}; do timeout 300 python tools/mv_ab.py $cfg 2:1 2>&1 | grep -v "^max"; done
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | tee gpurun_out/q/bench.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value',d['value'],'steps',d.get('step_ms'),'it',d['iterations'],'setup',d['setup_ms'],'solve',d.get('solve_ms'),'other',d.get('other_ms'),'phase',d['phase_ms'],'mv',d['matvec_ms'],d['matvec_gpairs_s'],'pc',d['rasm_apply_ms'],'e2e',d['e2e']['value'], 'clk', d['clocks'])"
