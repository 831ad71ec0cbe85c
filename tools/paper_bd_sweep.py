"""The paper's parameter study (Figs. bar_it / bar_ti): iterations and time
for B/sigma in {3..7} x D/B in {1.5..2.3} on a Franke lattice (rtol 1e-13), with the
paper's T-box matvec (T = B + 4 sigma at h/sigma >= 0.9, B + 6 sigma at 0.8); one B200.
Not part of the product.  Usage: paper_bd_sweep.py [n_side] [h_over_sigma]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0909_5413_b200 as P  # noqa: E402
import rbf_workloads as W  # noqa: E402

n_side = int(sys.argv[1]) if len(sys.argv) > 1 else 1001
hs = float(sys.argv[2]) if len(sys.argv) > 2 else 0.9
print(f"Franke lattice {n_side}^2, h/sigma = {hs}, rtol 1e-13, T-box per P:307")
print("| B/sigma | D/B | iterations | setup ms | solve ms | total ms | max Omega | LU cells |")
print("|---|---|---|---|---|---|---|---|")
for b in (3.0, 4.0, 5.0, 6.0, 7.0):
    for d in (1.5, 1.7, 1.9, 2.1, 2.3):
        wl = W.make_paper_lattice(n_side, hs, b_over_sigma=b, d_over_b=d)
        tau = (2.0 if hs >= 0.85 else 3.0) * wl.sigma
        xy = torch.from_numpy(wl.xy).cuda()
        f = torch.from_numpy(wl.f).cuda()
        best = None
        for _ in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            c = P.Context(xy, wl.sigma, wl.cell, wl.rc, wl.rings, wl.box,
                          overlap_width=wl.overlap_width, trunc_width=tau)
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            lam, rep = c.solve(c.to_local(f), rtol=1e-13, max_iters=500)
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            info = c.info()
            c.close()
            if best is None or t2 - t0 < best[2]:
                best = (1e3 * (t1 - t0), 1e3 * (t2 - t1), t2 - t0, rep.iterations, rep.converged)
        it = best[3] if best[4] else f"> {best[3]}"
        print(f"| {b:.0f} | {d} | {it} | {best[0]:.1f} | {best[1]:.1f} | {best[0] + best[1]:.1f} | "
              f"{info['max_ov']} | {info['n_lu']} |", flush=True)
