"""A/B of the RASM setup kernels: option setup_kernel = 0 (one factorisation per SM) vs 1
(two per SM, rows retired to L2).  Per config: setup time (median of 3), the apply
difference between the two on a random vector, and one solve's iterations.
Not part of the product.  Usage: tc2_ab.py CFG [CFG ...]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0909_5413_b200 as P  # noqa: E402
import rbf_workloads as W  # noqa: E402

for cfg in [int(a) for a in sys.argv[1:]] or [2]:
    wl = W.config(cfg)
    xy = torch.from_numpy(wl.xy).cuda()
    z = {}
    for v in [int(k) for k in os.environ.get("KERNELS", "0,1").split(",")]:
        with P.options(setup_kernel=v):
            su = []
            for r in range(3):
                c = P.Context(xy, wl.sigma, wl.cell, wl.rc, wl.rings, wl.box)
                su.append(c.setup_times()["rasm"])
                if r < 2:
                    c.close()
            g = torch.Generator(device="cuda").manual_seed(5)
            u = torch.randn(c.n_local, dtype=torch.float64, device="cuda", generator=g)
            z[v] = c.rasm_apply(u).clone()
            it = None
            if cfg <= 2:
                f = c.to_local(torch.from_numpy(wl.f).cuda())
                _, rep = c.solve(f, rtol=wl.rtol if hasattr(wl, "rtol") else 1e-13)
                it = rep.iterations
            c.close()
            torch.cuda.synchronize()
        print(f"cfg{cfg} setup_kernel={v}: rasm setup {statistics.median(su):.2f} ms (all {[round(x, 2) for x in su]}), "
              f"solve iterations {it}", flush=True)
    ks = sorted(z)
    for k in ks[1:]:
        d = (z[ks[0]] - z[k]).norm().item() / z[ks[0]].norm().item()
        print(f"cfg{cfg}: apply relative difference kernel {k} vs {ks[0]}: {d:.3e}", flush=True)
