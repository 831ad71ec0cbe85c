timeout 60 python tools/smoke_setup.py 1 || { echo "SMOKE FAILED"; exit 1; }
python - <<'PY' || { echo "TC3 SMOKE FAILED"; exit 1; }
import subprocess, sys
r = subprocess.run([sys.executable, "-c", "import paper_0909_5413_b200 as P; P.set_option('setup_kernel', 2); import runpy, sys; sys.argv=['x','1']; runpy.run_path('tools/smoke_setup.py', run_name='__main__')"], timeout=60)
sys.exit(r.returncode)
PY
KERNELS=0,2 timeout 300 python tools/tc2_ab.py 2 3 2>&1 | grep -v "^$"
timeout 300 python -m pytest tests -m gpu -x -q -k "two_per_sm" 2>&1 | tail -3
