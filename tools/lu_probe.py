"""LU-path routing on a few workloads: subdomains on the LU path and how many were
factored with partial pivoting (rbf_lu_stats), with and without the no-pivot pass."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0909_5413_b200 as P  # noqa: E402
import rbf_workloads as W  # noqa: E402

cases = [("clustered3000 r1", W.make_clustered(3000, seed=11), 1),
         ("clustered3000 r2", W.make_clustered(3000, seed=11), 2),
         ("clustered20000 r1", W.make_clustered(20000, seed=5), 1),
         ("clustered20000 r2", W.make_clustered(20000, seed=5), 2),
         ("lattice48 r2", W.make_lattice(48, jitter_frac=0.1, seed=5), 2)]
for name, wl, rings in cases:
    for knob in ("1", "0"):
        P.set_option("lu_nopiv", int(knob))
        xy = torch.from_numpy(wl.xy).cuda()
        with P.Context(xy, wl.sigma, wl.cell, wl.rc, rings, wl.box) as c:
            print(name, "nopiv" if knob == "1" else "pivot-all", c.lu_stats(), c.info()["max_ov"], flush=True)
P.set_option("lu_nopiv", 1)
