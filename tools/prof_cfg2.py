"""Profiling driver: one setup + matvec + RASM apply + short solve on a config
(default cfg2), for ncu captures.  Not part of the product."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0909_5413_b200 as P  # noqa: E402
import rbf_workloads as W  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
if "--no-graph" in sys.argv:  # host-driven GMRES loop: every kernel launched on its own
    P.set_option("solve_graph", 0)
wl = W.config(cfg)
xy = torch.from_numpy(wl.xy).cuda()
c = P.Context(xy, wl.sigma, wl.cell, wl.rc, wl.rings, wl.box)
f = c.to_local(torch.from_numpy(wl.f).cuda())
w = torch.randn(c.n_local, dtype=torch.float64, device="cuda")
for _ in range(2):
    y = c.matvec(w)
    z = c.rasm_apply(w)
lam, rep = c.solve(f, rtol=wl.tol, max_iters=5)
q = xy[: min(c.n, 1 << 20)] * 0.999
s_ = c.evaluate(q, lam)
torch.cuda.synchronize()
print("ok", rep.iterations, c.info())
c.close()
