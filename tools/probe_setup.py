"""Phase timing of the RASM setup kernel (probe build in tools/probe/librbf.so)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_0909_5413_b200.rbf as R  # noqa: E402
import rbf_workloads as W  # noqa: E402

R.LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "probe", os.environ.get("PROBE_LIB", "librbf.so"))
L = R.lib()
L.rbf_debug_probe.argtypes = [C.c_void_p]
L.rbf_debug_probe.restype = C.c_int
wl = W.config(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
xy = torch.from_numpy(wl.xy).cuda()
for _ in range(2):
    c = R.Context(xy, wl.sigma, wl.cell, wl.rc, wl.rings, wl.box)
    torch.cuda.synchronize()
    print(c.setup_times())
    c.close()
buf = np.zeros(64 * 8 + 65536 * 3 + 512 + 128, dtype=np.int64)
assert L.rbf_debug_probe(buf.ctypes.data_as(C.c_void_p)) == 0
out = buf[:512].reshape(64, 8)
tr = buf[512:512 + 65536 * 3].reshape(65536, 3)[:42025]
dur = (tr[:, 2] - tr[:, 1]) / 1e3
print(f"CTA duration us: mean {dur.mean():.1f} min {dur.min():.1f} max {dur.max():.1f}")
t0 = tr[:, 1].min()
print(f"kernel span us: {(tr[:, 2].max() - t0) / 1e3:.1f}, SMs used {len(set(tr[:, 0]))}")
for sm in (0, 1, 77):
    sel = np.where(tr[:, 0] == sm)[0]
    st = np.sort(tr[sel, 1])
    en = np.sort(tr[sel, 2])
    gaps = (st[1:] - en[:-1]) / 1e3
    print(f"sm {sm}: ctas {len(sel)}, mean gap between CTAs {gaps.mean():.2f} us, busy {(en - st).sum() / 1e3:.0f} us")
out = out[out[:, 4] > 0]
d = np.diff(out[:, :5], axis=1)
names = ["assembly", "cholesky", "W+Sinv", "X write"]
for i, nm in enumerate(names):
    print(f"{nm:10s} mean {d[:, i].mean():10.0f} cyc  min {d[:, i].min():8d} max {d[:, i].max():8d}")
print("total", (out[:, 4] - out[:, 0]).mean())
if (out[:, 5] > 0).all():
    print(f"X phase: thread 0's tasks {(out[:, 5] - out[:, 3]).mean():.0f}, own part + barrier "
          f"{(out[:, 6] - out[:, 5]).mean():.0f}, bulk copy issue + read-out {(out[:, 4] - out[:, 6]).mean():.0f} cycles")
col = buf[512 + 65536 * 3:512 + 65536 * 3 + 512].reshape(2, 64, 4)
c0, cd = col[0], col[1]
base = c0[0, 0]
print("per tile column j of one interior CTA (cycles).  Column-loop kernel: warp 0 [step1+2, wait at sync 1, panel+sync 2], "
      "diagonal warp [finish, 8x8 factor], column total.")
for j in range(30):
    if c0[j, 0] == 0:
        break
    print(f"{j:2d} w0: {c0[j, 1] - c0[j, 0]:6d} {c0[j, 2] - c0[j, 1]:6d} {c0[j, 3] - c0[j, 2]:6d} | "
          f"dw: {cd[j, 1] - cd[j, 0]:6d} {cd[j, 2] - cd[j, 1]:6d} | col {c0[j, 3] - c0[j, 0]:6d}")
wc = buf[512 + 65536 * 3 + 512:].reshape(32, 4)
print("W phase (right-looking), warp 0 per column kt: [wait at the step barrier, chain update + finish, other updates]; S^-1 warps total")
for jt in range(31):
    if wc[jt, 0] == 0:
        continue
    print(f"kt {jt:2d}: {wc[jt, 1] - wc[jt, 0]:6d} {wc[jt, 2] - wc[jt, 1]:6d} {wc[jt, 3] - wc[jt, 2]:6d}")
print("S^-1 (warp 15):", wc[31, 1] - wc[31, 0])
