"""A/B of two librbf.so builds on one config: neighbour-list build (setup 'nlist'), matvec and
evaluation times, and bitwise comparison of their outputs (saved by the 'prev' run, compared
by the next).  Not part of the product.  Usage: trim_ab.py CFG LIB TAG"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_0909_5413_b200.rbf as R  # noqa: E402
R.LIB_PATH = os.path.abspath(sys.argv[2])
import paper_0909_5413_b200 as P  # noqa: E402
import rbf_workloads as W  # noqa: E402

cfg, tag = int(sys.argv[1]), sys.argv[3]
wl = W.config(cfg)
xy = torch.from_numpy(wl.xy).cuda()
n = 2048 if cfg <= 2 else 7071
hq = 2.0 / n
cq = -1.0 + (np.arange(n - 1) + 1) * hq
X, Y = np.meshgrid(cq, cq)
q = torch.from_numpy(np.stack([X.ravel(), Y.ravel()], 1).copy()).cuda()
del X, Y
nl = []
for r in range(3):
    c = P.Context(xy, wl.sigma, wl.cell, wl.rc, wl.rings, wl.box)
    nl.append(c.setup_times()["nlist"])
    if r < 2:
        c.close()
g = torch.Generator(device="cuda").manual_seed(7)
w = torch.randn(c.n_local, dtype=torch.float64, device="cuda", generator=g)
y = c.matvec(w).clone()
s = c.evaluate(q, w).clone()
npairs = c.evaluate_count_pairs(q)


def tm(fn, k=10):
    fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / k


t_mv = tm(lambda: c.matvec(w, y))
t_ev = tm(lambda: c.evaluate(q, w), 5)
out = f"/tmp/trim_{cfg}"
if tag == "prev":
    np.save(out + "_y.npy", y.cpu().numpy())
    np.save(out + "_s.npy", s.cpu().numpy())
else:
    y0, s0 = np.load(out + "_y.npy"), np.load(out + "_s.npy")
    print(f"cfg{cfg}: matvec bitwise equal {np.array_equal(y0, y.cpu().numpy())}, "
          f"evaluate bitwise equal {np.array_equal(s0, s.cpu().numpy())}")
print(f"cfg{cfg} {tag}: nlist {sorted(nl)[1]:.2f} ms, matvec {t_mv:.3f} ms, evaluate {t_ev:.3f} ms "
      f"({npairs} pairs, {npairs / (t_ev * 1e-3) / 1e9:.1f} Gpairs/s)", flush=True)
c.close()
