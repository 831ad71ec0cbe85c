"""Oracle (plain C, all host cores) timings per phase, next to the GPU numbers of the same
tree (SURVEY.md §8.d "Oracle timing"); not part of the product.  Prints a markdown table.
Usage: OMP_NUM_THREADS=$(nproc) oracle_timing.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
import rbf_workloads as W  # noqa: E402


def t(fn, reps=1):
    best = None
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    return best, out


cores = os.environ.get("OMP_NUM_THREADS", str(os.cpu_count()))
print(f"host cores used: {cores}; CPU: {os.popen('lscpu | grep \"Model name\"').read().strip()}")
print("| config | phase | oracle (s) |")
print("|---|---|---|")
wl = W.config(1)
dt, r = t(lambda: O.solve(wl.xy, wl.f, wl.sigma, wl.rc, wl.box, wl.cell, rtol=wl.tol))
print(f"| cfg1 (N={wl.n}) | full solve ({r.iterations} it) | {dt:.3f} |", flush=True)
for k in (2, 5):
    wl = W.config(k)
    w = np.random.default_rng(1).standard_normal(wl.n)
    dt, _ = t(lambda: O.matvec_cells(wl.xy, w, wl.sigma, wl.rc, wl.box, wl.cell), reps=3)
    print(f"| cfg{k} (N={wl.n}) | matvec (cell list, median of 3 -> best) | {dt:.3f} |", flush=True)
    if k == 2:
        dt, P = t(lambda: O.Rasm(wl.xy, wl.sigma, wl.rc, wl.box, wl.cell, 1))
        print(f"| cfg{k} | RASM setup ({P.nsub} subdomains) | {dt:.3f} |", flush=True)
        dt, _ = t(lambda: P.apply(w), reps=3)
        print(f"| cfg{k} | RASM apply | {dt:.3f} |", flush=True)
        P.close()
