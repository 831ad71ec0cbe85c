"""MGS vs CGS2 (reading Q23) vs DCGS2 (reading Q27) on one config: graph-path solve time and host-loop orth phase;
not part of the product.  Usage: CFG=2 orth_cmp.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0909_5413_b200 as P  # noqa: E402
import rbf_workloads as W  # noqa: E402

wl = W.config(int(os.environ.get("CFG", "2")))
xy = torch.from_numpy(wl.xy).cuda()
f = torch.from_numpy(wl.f).cuda()
c = P.Context(xy, wl.sigma, wl.cell, wl.rc, wl.rings, wl.box)
fl = c.to_local(f)
for orth in (sys.argv[1:] or ["mgs", "cgs2", "dcgs2", "mgs", "cgs2", "dcgs2"]):
    g = []
    for _ in range(3):
        lam, r = c.solve(fl, rtol=wl.tol, orth=orth)
        g.append(r.ms_total)
    lam, rt = c.solve(fl, rtol=wl.tol, orth=orth, timing=True)
    print(f"{orth:6s} it {r.iterations} resid_true {r.resid_true:.2e} graph solve ms "
          f"{[round(x, 2) for x in g]} | hostloop total {rt.ms_total:.2f} mv {rt.ms_matmult:.2f} "
          f"pc {rt.ms_pcapply:.2f} orth {rt.ms_orth:.2f}", flush=True)
c.close()
