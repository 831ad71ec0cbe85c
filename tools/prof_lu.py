"""rbf_setup with 2 overlap rings (625-point subdomains, all on the blocked LU path)
on a jittered lattice, for ncu captures of k_rasm_setup_lu.  Not part of the product."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0909_5413_b200 as P  # noqa: E402
import rbf_workloads as W  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
rings = int(sys.argv[2]) if len(sys.argv) > 2 else 2
wl = W.make_lattice(n, jitter_frac=0.1, seed=3)
xy = torch.from_numpy(wl.xy).cuda()
for _ in range(2):
    c = P.Context(xy, wl.sigma, wl.cell, wl.rc, rings, wl.box)
    torch.cuda.synchronize()
    print("ok", c.setup_times(), c.info(), flush=True)
    c.close()
