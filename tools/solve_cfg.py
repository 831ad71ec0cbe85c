"""Setup + solve of one config with a report (not part of the product)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0909_5413_b200 as P  # noqa: E402
import rbf_workloads as W  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
maxit = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
wl = W.config(cfg)
xy = torch.from_numpy(wl.xy).cuda()
f = torch.from_numpy(wl.f).cuda()
torch.cuda.synchronize()
t0 = time.perf_counter()
c = P.Context(xy, wl.sigma, wl.cell, wl.rc, wl.rings, wl.box)
torch.cuda.synchronize()
t1 = time.perf_counter()
try:
    lam, rep = c.solve(c.to_local(f), rtol=wl.tol, max_iters=maxit, timing=True)
except P.RbfError as e:
    print("solve error", e)
    rep = None
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"cfg{cfg}: setup {t1 - t0:.3f} s {c.setup_times()} info {c.info()}")
if rep is not None:
    print(f"solve {t2 - t1:.3f} s: it {rep.iterations} restarts {rep.restarts} converged {rep.converged} "
          f"est {rep.resid_est:.3e} precond {rep.resid_precond:.3e} true {rep.resid_true:.3e} "
          f"mv {rep.ms_matmult:.1f} pc {rep.ms_pcapply:.1f} orth {rep.ms_orth:.1f} ms")
c.close()
