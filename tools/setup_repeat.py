"""rbf_setup + rbf_solve repeated on one config, printing the setup phases per repetition and
any device allocation slower than 5 ms (option log_slow_alloc).  Not part of the product."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0909_5413_b200 as P  # noqa: E402
import rbf_workloads as W  # noqa: E402

P.set_option("log_slow_alloc", 5)
wl = W.config(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
xy = torch.from_numpy(wl.xy).cuda()
f = torch.from_numpy(wl.f).cuda()
for r in range(int(sys.argv[2]) if len(sys.argv) > 2 else 8):
    t0 = time.perf_counter()
    c = P.Context(xy, wl.sigma, wl.cell, wl.rc, wl.rings, wl.box)
    t1 = time.perf_counter()
    lam, rep = c.solve(c.to_local(f), rtol=wl.tol)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    st = c.setup_times()
    c.close()
    print(f"rep {r}: setup host {1e3 * (t1 - t0):.1f} ms {({k: round(v, 2) for k, v in st.items()})}, solve host "
          f"{1e3 * (t2 - t1):.1f} ms", file=sys.stderr, flush=True)
