"""Design probe (not part of the product): can the ALU-bound matvec and the HBM-bound
RASM apply share the GPU?  Times, on a config, the matvec alone, the apply alone, both
back to back on one stream, and both at once on two streams (independent inputs, joined
every iteration).  Usage: overlap_probe.py [CFG]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0909_5413_b200 as P  # noqa: E402
import paper_0909_5413_b200.rbf as R  # noqa: E402
import rbf_workloads as W  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
wl = W.config(cfg)
c = P.Context(torch.from_numpy(wl.xy).cuda(), wl.sigma, wl.cell, wl.rc, wl.rings, wl.box)
n = c.n_local
g = torch.Generator("cuda").manual_seed(1)
w, r = (torch.randn(n, dtype=torch.float64, device="cuda", generator=g) for _ in range(2))
y, z = torch.empty_like(w), torch.empty_like(w)
L = R.lib()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731


def mv(s):
    L.rbf_matvec(c._h, p(w), p(y), C.c_void_p(s.cuda_stream))


def ap(s):
    L.rbf_rasm_apply(c._h, p(r), p(z), C.c_void_p(s.cuda_stream))


def timed(body, reps=50):
    for _ in range(3):
        body()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s1)
    for _ in range(reps):
        body()
    e1.record(s1)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def conc():
    ev = torch.cuda.Event()
    ev.record(s1)
    s2.wait_event(ev)
    ap(s2)  # the apply first: its persistent CTAs take one slot per SM, the matvec the rest
    mv(s1)
    ev2 = torch.cuda.Event()
    ev2.record(s2)
    s1.wait_event(ev2)


t_mv = timed(lambda: mv(s1))
t_ap = timed(lambda: ap(s1))
t_seq = timed(lambda: (mv(s1), ap(s1)))
t_conc = timed(conc)
print(f"cfg{cfg}: matvec {t_mv:.4f} ms, apply {t_ap:.4f} ms, sequential {t_seq:.4f} ms, "
      f"concurrent {t_conc:.4f} ms (saves {t_seq - t_conc:.4f} ms per iteration)")
