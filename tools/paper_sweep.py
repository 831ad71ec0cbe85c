"""Iteration counts of the paper's test problem (Franke data) at
h/sigma in {1.0, 0.9, 0.8} and several mesh sizes, lattice and quasi-scattered;
prints a markdown table.  Not part of the product."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0909_5413_b200 as P  # noqa: E402
import rbf_workloads as W  # noqa: E402

# geometry: "ours" = cell 4 sigma + one whole ring; "B5" / "B6" = the paper's boxes
# B = 5 / 6 sigma, D = 1.9 B (reading Q24)
# "B5T" / "B6T" add the paper's T-box matvec (reading Q25): T = B + 4 sigma at h/sigma >= 0.9,
# B + 6 sigma at 0.8; T = B + 6 sigma for scattered data
GEOMS = {"ours": {}, "B5": dict(b_over_sigma=5.0, d_over_b=1.9), "B6": dict(b_over_sigma=6.0, d_over_b=1.9),
         "B5T": dict(b_over_sigma=5.0, d_over_b=1.9), "B6T": dict(b_over_sigma=6.0, d_over_b=1.9)}


def tau_of(geo, r, scattered, sigma):
    if not geo.endswith("T"):
        return 0.0
    if geo == "B6T" or scattered or r < 0.85:
        return 3.0 * sigma
    return 2.0 * sigma


sel = sys.argv[1:] or list(GEOMS)
print("| geometry | h/sigma | points | N | iterations | true residual | setup ms | solve ms |")
print("|---|---|---|---|---|---|---|---|")
for geo in sel:
  for r in (1.0, 0.9, 0.8):
    for n, sc in ((101, None), (201, None), (401, None), (1001, None), (101, 9), (401, 9)):
        wl = W.make_paper_lattice(n, r, scatter_seed=sc, **GEOMS[geo])
        xy = torch.from_numpy(wl.xy).cuda()
        f = torch.from_numpy(wl.f).cuda()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        tau = tau_of(geo, r, sc is not None, wl.sigma)
        c = P.Context(xy, wl.sigma, wl.cell, wl.rc, wl.rings, wl.box, overlap_width=wl.overlap_width,
                      trunc_width=tau)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        lam, rep = c.solve(c.to_local(f), rtol=wl.tol)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        kind = "lattice" if sc is None else "scattered"
        print(f"| {geo} | {r} | {kind} {n}x{n} | {wl.n} | {rep.iterations} | {rep.resid_true:.1e} | "
              f"{1e3 * (t1 - t0):.1f} | {1e3 * (t2 - t1):.1f} |", flush=True)
        c.close()
