"""Time the RASM setup of LU-path workloads with an A/B build of librbf.so
(tools/build_variant.sh) and compare its RASM apply with a saved reference vector.
Usage: lu_var.py path/to/librbf.so tag case [case ...] (cases as in lu_ab.py); the apply
of the first tag run for a case is saved under gpurun_out/lu_var_<case>.pt and later
tags are compared with it.  Not part of the product."""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0909_5413_b200 as P  # noqa: E402
import paper_0909_5413_b200.rbf as R  # noqa: E402
from lu_ab import make  # noqa: E402

R.LIB_PATH = os.path.abspath(sys.argv[1])
tag = sys.argv[2]
reps = int(os.environ.get("REPS", "3"))
for case in sys.argv[3:]:
    wl, rings = make(case)
    xy = torch.from_numpy(wl.xy).cuda()
    ts = []
    for r in range(reps + 1):
        torch.cuda.synchronize()
        with P.Context(xy, wl.sigma, wl.cell, wl.rc, rings, wl.box) as c:
            if r > 0:
                ts.append(c.setup_times()["rasm"])
            if r == reps:
                g = torch.Generator(device="cpu").manual_seed(7)
                u = torch.randn(c.n_local, dtype=torch.float64, generator=g).cuda()
                z = c.rasm_apply(u).cpu()
    ref = f"gpurun_out/lu_var_{case}.pt"
    cmp = ""
    if os.path.exists(ref):
        z0 = torch.load(ref)
        cmp = f" vs first: max rel {((z - z0).abs().max() / z0.abs().max()).item():.2e} bitwise={torch.equal(z, z0)}"
    else:
        torch.save(z, ref)
    print(f"{tag} {case}: rasm setup {statistics.median(ts):.2f} ms {[round(t, 2) for t in ts]}{cmp}", flush=True)
