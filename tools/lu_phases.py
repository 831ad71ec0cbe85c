"""Phase clocks of the LU-path kernel (probe build: tools/build_probe.sh -> tools/probe/
librbf.so): cycles summed over CTAs per phase for one setup of each case (lu_ab.py cases).
Not part of the product."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0909_5413_b200 as P  # noqa: E402
import paper_0909_5413_b200.rbf as R  # noqa: E402
from lu_ab import make  # noqa: E402

R.LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "probe", "librbf.so")
L = R.lib()
L.rbf_debug_probe.argtypes = [C.c_void_p]
L.rbf_debug_probe.restype = C.c_int
OFF = 64 * 8 + 65536 * 3 + 512 + 128
names = ["assembly", "panel", "writeback+L11", "U12 solve", "update", "back subst", "X copy"]


def read():
    buf = np.zeros(OFF + 512 * 10, dtype=np.int64)
    assert L.rbf_debug_probe(buf.ctypes.data_as(C.c_void_p)) == 0
    return buf[OFF:].reshape(512, 10).copy()


for case in sys.argv[1:]:
    wl, rings = make(case)
    xy = torch.from_numpy(wl.xy).cuda()
    c = P.Context(xy, wl.sigma, wl.cell, wl.rc, rings, wl.box)  # warm-up
    c.close()
    a0 = read()
    c = P.Context(xy, wl.sigma, wl.cell, wl.rc, rings, wl.box)
    torch.cuda.synchronize()
    st = c.setup_times()
    c.close()
    d = read() - a0
    tot = d[:, :7].sum(0).astype(float)
    cells, sn = d[:, 7].sum(), d[:, 8].sum()
    ctas = int((d[:, 7] > 0).sum())
    print(f"{case}: rasm {st['rasm']:.2f} ms, {cells} cells (sum n {sn}), {ctas} CTAs; "
          f"per-CTA mean busy {tot.sum() / max(ctas, 1) / 1.965e6:.2f} ms at 1965 MHz")
    for k, nm in enumerate(names):
        print(f"   {nm:14s} {100 * tot[k] / tot.sum():5.1f}%  {tot[k] / max(ctas, 1) / 1.965e6:8.2f} ms per CTA")
