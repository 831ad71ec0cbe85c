"""Orthogonalisation phase time of a cfg2 solve for library-option variants (rbf_set_option,
e.g. mgs_pairs=0,fused_arnoldi=1); not part of the product.
Usage: orth_ab.py opt=val,opt2=val ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0909_5413_b200 as P  # noqa: E402
import rbf_workloads as W  # noqa: E402

wl = W.config(int(os.environ.get("CFG", "2")))
xy = torch.from_numpy(wl.xy).cuda()
f = torch.from_numpy(wl.f).cuda()
for spec in sys.argv[1:]:
    for kv in spec.split(","):
        if kv:
            k, v = kv.split("=")
            P.set_option(k, int(v))
    res = []
    for rep in range(3):
        c = P.Context(xy, wl.sigma, wl.cell, wl.rc, wl.rings, wl.box)
        lam, r = c.solve(c.to_local(f), rtol=wl.tol, timing=True)
        res.append((r.ms_orth, r.ms_total, r.iterations))
        c.close()
    print(spec, "orth ms", [round(x[0], 2) for x in res], "solve ms", [round(x[1], 2) for x in res], "it", res[-1][2], flush=True)
