"""A/B of the matvec neighbour-list entry width (option mv_index16) on a config:
device time per matvec and bitwise agreement.  Not part of the product."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0909_5413_b200 as P  # noqa: E402
import rbf_workloads as W  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
wl = W.config(cfg)
xy = torch.from_numpy(wl.xy).cuda()
res = {}
for v in (1, 0, 1, 0):
    P.set_option("mv_index16", v)
    c = P.Context(xy, wl.sigma, wl.cell, wl.rc, 0, wl.box)  # no RASM: matvec only
    w = torch.randn(c.n_local, dtype=torch.float64, device="cuda",
                    generator=torch.Generator("cuda").manual_seed(1))
    y = torch.empty_like(w)
    for _ in range(3):
        c.matvec(w, y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        c.matvec(w, y)
    e1.record()
    e1.synchronize()
    res[v] = (e0.elapsed_time(e1) / 20, y.clone(), c.matvec_stats())
    c.close()
    del c
    P.trim_memory()
P.set_option("mv_index16", 0)
print(f"cfg{cfg}: 16-bit {res[1][0]:.3f} ms, 32-bit {res[0][0]:.3f} ms, bitwise equal "
      f"{bool(torch.equal(res[1][1], res[0][1]))}, stats {res[1][2]}")
