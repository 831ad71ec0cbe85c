"""Per-kernel A/B of two librbf.so builds on one config: RASM setup, matvec and RASM apply
times (median of repeats) in a fresh process per build.  Not part of the product.
Usage: lib_ab.py CFG lib1 [lib2 ...]"""
import os
import statistics
import subprocess
import sys

if len(sys.argv) > 2 and sys.argv[1] == "--one":
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch

    import paper_0909_5413_b200.rbf as R
    import rbf_workloads as W
    R.LIB_PATH = os.path.abspath(sys.argv[3])
    import paper_0909_5413_b200 as P
    wl = W.config(int(sys.argv[2]))
    xy = torch.from_numpy(wl.xy).cuda()
    su, mv, pc = [], [], []
    for r in range(3):
        c = P.Context(xy, wl.sigma, wl.cell, wl.rc, wl.rings, wl.box)
        su.append(c.setup_times()["rasm"])
        w = torch.randn(c.n_local, dtype=torch.float64, device="cuda")
        y = torch.empty_like(w)
        for fn, out in ((lambda: c.matvec(w, y), mv), (lambda: c.rasm_apply(w, y), pc)):
            for _ in range(3):
                fn()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20):
                fn()
            e1.record()
            e1.synchronize()
            out.append(e0.elapsed_time(e1) / 20)
        c.close()
    print(f"{sys.argv[3]}: setup {statistics.median(su):.2f} ms, matvec {statistics.median(mv):.4f} ms, "
          f"rasm apply {statistics.median(pc):.4f} ms", flush=True)
else:
    for lib in sys.argv[2:]:
        subprocess.run([sys.executable, __file__, "--one", sys.argv[1], lib], check=False)
