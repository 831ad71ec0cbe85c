"""A/B timing of matvec variants G:VAR (options mv_targets_per_lane, mv_variant) on a config;
not part of the product.
Usage: mv_ab.py CFG 2:0 1:1 ..."""
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
for v in sys.argv[2:] or ["2:0", "1:1"]:
    g_, var_ = v.split(":")
    P.set_option("mv_targets_per_lane", int(g_))
    P.set_option("mv_variant", int(var_))
    c = P.Context(xy, wl.sigma, wl.cell, wl.rc, wl.rings, wl.box)
    npairs = c.count_pairs()
    w = torch.randn(c.n_local, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(1))
    y = torch.empty_like(w)
    for _ in range(3):
        c.matvec(w, y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        c.matvec(w, y)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 50
    res[v] = y.clone()
    print(f"cfg{cfg} G:VAR={v}: {ms:.4f} ms/matvec, {npairs / ms / 1e6:.1f} Gpairs/s, "
          f"useful FP64 frac {npairs * 38 / (ms * 1e-3) / 36.86e12:.3f}, stats {c.matvec_stats()} pairs {npairs}", flush=True)
    c.close()
vals = list(res.values())
for k, b in zip(list(res)[1:], vals[1:]):
    print("max |diff| vs first variant", k, float((vals[0] - b).abs().max()))
