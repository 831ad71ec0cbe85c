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
R.set_option("setup_kernel", int(os.environ.get("TC2", "1")))
wl = W.config(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
xy = torch.from_numpy(wl.xy).cuda()
for _ in range(2):
    c = R.Context(xy, wl.sigma, wl.cell, wl.rc, wl.rings, wl.box)
    torch.cuda.synchronize()
    print(c.setup_times())
    c.close()
buf = np.zeros(64 * 8 + 65536 * 3 + 512 + 128 + 5120 + 4096 + 512, dtype=np.int64)
assert L.rbf_debug_probe(buf.ctypes.data_as(C.c_void_p)) == 0
t2 = buf[512 + 65536 * 3 + 512 + 128 + 5120:512 + 65536 * 3 + 512 + 128 + 5120 + 4096].reshape(512, 8)
t2c = buf[512 + 65536 * 3 + 512 + 128 + 5120 + 4096:512 + 65536 * 3 + 512 + 128 + 5120 + 4096 + 256].reshape(32, 8)
t2w = buf[512 + 65536 * 3 + 512 + 128 + 5120 + 4096 + 256:].reshape(32, 8)
if t2[:, 0].sum() > 0 and os.environ.get("TC2") == "2":
    sel = t2[:, 0] > 0
    cells = t2[sel, 0].sum()
    print(f"tc3: {sel.sum()} CTAs, {cells} cells; per cell (cycles): factor warps: runs+pos {t2[sel, 1].sum() / cells:.0f}, "
          f"cholesky {t2[sel, 2].sum() / cells:.0f}, wait for post {t2[sel, 3].sum() / cells:.0f}, copy {t2[sel, 4].sum() / cells:.0f}; "
          f"post warps: W {t2[sel, 5].sum() / cells:.0f}, Sinv {t2[sel, 6].sum() / cells:.0f}, X {t2[sel, 7].sum() / cells:.0f}")
    sys.exit(0)
if t2[:, 0].sum() > 0:
    sel = t2[:, 0] > 0
    cells = t2[sel, 0].sum()
    print(f"tc2: {sel.sum()} CTAs, {cells} cells; per cell (cycles of one CTA): runs+pos {t2[sel, 1].sum() / cells:.0f}, "
          f"cholesky {t2[sel, 2].sum() / cells:.0f}, W+Sinv {t2[sel, 3].sum() / cells:.0f} (W warps {t2[sel, 5].sum() / cells:.0f}, "
          f"Sinv warps {t2[sel, 6].sum() / cells:.0f}), X {t2[sel, 4].sum() / cells:.0f}")
    print("per column (one interior cell, CTA 7): w0 step1, step2, wait b1, panel(w0), b2 wait(w0) | dw finish->factor start, factor | column")
    for j in range(32):
        c_ = t2c[j]
        if c_[0] == 0:
            continue
        print(f"{j:2d}: {c_[1]-c_[0]:6d} {c_[2]-c_[1]:6d} {c_[3]-c_[2]:6d} {c_[4]-c_[3]:6d} | {c_[5]-c_[0]:6d} {c_[6]-c_[5]:6d} | "
              f"{(t2c[j + 1][0] - c_[0]) if j + 1 < 32 and t2c[j + 1][0] else 0:6d}")
    print("W phase per step jt (warp 0): wait_group, bar.sync, fetch issue, dot product, finish, to next step")
    for jt in range(31, -1, -1):
        c_ = t2w[jt]
        if c_[0] == 0:
            continue
        nxt = t2w[jt - 1][0] if jt >= 1 and t2w[jt - 1][0] else c_[5]
        print(f"{jt:2d}: {c_[1]-c_[0]:6d} {c_[2]-c_[1]:6d} {c_[3]-c_[2]:6d} {c_[4]-c_[3]:6d} {c_[5]-c_[4]:6d} {nxt-c_[5]:6d}")
    sys.exit(0)
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
wc = buf[512 + 65536 * 3 + 512:512 + 65536 * 3 + 512 + 128].reshape(32, 4)
t2 = buf[512 + 65536 * 3 + 512 + 128 + 5120:512 + 65536 * 3 + 512 + 128 + 5120 + 4096].reshape(512, 8)
t2c = buf[512 + 65536 * 3 + 512 + 128 + 5120 + 4096:512 + 65536 * 3 + 512 + 128 + 5120 + 4096 + 256].reshape(32, 8)
t2w = buf[512 + 65536 * 3 + 512 + 128 + 5120 + 4096 + 256:].reshape(32, 8)
if t2[:, 0].sum() > 0 and os.environ.get("TC2") == "2":
    sel = t2[:, 0] > 0
    cells = t2[sel, 0].sum()
    print(f"tc3: {sel.sum()} CTAs, {cells} cells; per cell (cycles): factor warps: runs+pos {t2[sel, 1].sum() / cells:.0f}, "
          f"cholesky {t2[sel, 2].sum() / cells:.0f}, wait for post {t2[sel, 3].sum() / cells:.0f}, copy {t2[sel, 4].sum() / cells:.0f}; "
          f"post warps: W {t2[sel, 5].sum() / cells:.0f}, Sinv {t2[sel, 6].sum() / cells:.0f}, X {t2[sel, 7].sum() / cells:.0f}")
    sys.exit(0)
if t2[:, 0].sum() > 0:
    sel = t2[:, 0] > 0
    cells = t2[sel, 0].sum()
    print(f"tc2: {sel.sum()} CTAs, {cells} cells; per cell (cycles, CTA-time): runs+pos {t2[sel, 1].sum() / cells:.0f}, "
          f"cholesky {t2[sel, 2].sum() / cells:.0f}, W+Sinv {t2[sel, 3].sum() / cells:.0f} (W warps {t2[sel, 5].sum() / cells:.0f}, "
          f"Sinv warps {t2[sel, 6].sum() / cells:.0f}), X {t2[sel, 4].sum() / cells:.0f}")
print("W phase (right-looking), warp 0 per column kt: [wait at the step barrier, chain update + finish, other updates]; S^-1 warps total")
for jt in range(31):
    if wc[jt, 0] == 0:
        continue
    print(f"kt {jt:2d}: {wc[jt, 1] - wc[jt, 0]:6d} {wc[jt, 2] - wc[jt, 1]:6d} {wc[jt, 3] - wc[jt, 2]:6d}")
print("S^-1 (warp 15):", wc[31, 1] - wc[31, 0])
