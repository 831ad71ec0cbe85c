"""Timing of rbf_evaluate on a config's data -> the interior corner lattice
(design evidence).  Usage: python tools/eval_ab.py [cfg]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_0909_5413_b200 as P  # noqa: E402
import rbf_workloads as W  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
wl = W.config(cfg)
n = wl.meta.get("n_side", 2048)
h = 2.0 / n
cq = -1.0 + (np.arange(n - 1) + 1) * h
X, Y = np.meshgrid(cq, cq)
q = torch.from_numpy(np.stack([X.ravel(), Y.ravel()], 1).copy()).cuda()
xy = torch.from_numpy(wl.xy).cuda()
with P.Context(xy, wl.sigma, wl.cell, wl.rc, wl.rings, wl.box) as c:
    lam = torch.randn(c.n_local, dtype=torch.float64, device="cuda")
    out = torch.empty(q.shape[0], dtype=torch.float64, device="cuda")
    npairs = c.evaluate_count_pairs(q)
    res = {}
    for v in ("warm", "run"):
        c.evaluate(q, lam, out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            c.evaluate(q, lam, out)
        e1.record()
        e1.synchronize()
        res[v] = (e0.elapsed_time(e1) / 5, out.clone())
    d = (res["warm"][1] - res["run"][1]).abs().max().item()
    for v in ("run",):
        ms = res[v][0]
        print(f"{v}: {ms:.3f} ms/call (incl. query sort), {npairs / ms / 1e6:.1f} Gpairs/s, "
              f"useful FP64 {npairs * 38 / ms / 1e9 / 36.86:.3f} of peak")
    print(f"cfg{cfg}: {q.shape[0]} queries, {npairs} in-cutoff pairs, max |run1 - run2| = {d:.3e}")
