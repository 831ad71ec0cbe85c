"""One rbf_setup on a config (default cfg2) for ncu captures of the setup kernels."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0909_5413_b200 as P  # noqa: E402
import rbf_workloads as W  # noqa: E402

wl = W.config(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
xy = torch.from_numpy(wl.xy).cuda()
c = P.Context(xy, wl.sigma, wl.cell, wl.rc, wl.rings, wl.box)
torch.cuda.synchronize()
print("ok", c.setup_times())
c.close()
