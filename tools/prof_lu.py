"""rbf_setup on workloads whose subdomains take the blocked LU path, for ncu captures of
k_rasm_setup_lu.  Not part of the product.
  prof_lu.py [n_side] [rings]          jittered lattice (2 rings: 625-point subdomains)
  prof_lu.py clu [N]                   cfg5 recipe at N points (cluster cells as in cfg5)
Options as NAME=VALUE in the environment variable LU_OPTS (e.g. "lu_update=0")."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0909_5413_b200 as P  # noqa: E402
import paper_0909_5413_b200.rbf as R  # noqa: E402
import rbf_workloads as W  # noqa: E402

if os.environ.get("RBF_TOOL_LIB"):  # an A/B build from tools/build_variant.sh
    R.LIB_PATH = os.path.abspath(os.environ["RBF_TOOL_LIB"])
for kv in filter(None, os.environ.get("LU_OPTS", "").split(",")):
    k, v = kv.split("=")
    P.set_option(k, int(v))
if len(sys.argv) > 1 and sys.argv[1] == "clu":
    wl = W.make_clustered(int(sys.argv[2]) if len(sys.argv) > 2 else 262144, seed=5)
    rings = 1
else:
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    rings = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    wl = W.make_lattice(n, jitter_frac=0.1, seed=3)
xy = torch.from_numpy(wl.xy).cuda()
for _ in range(2):
    c = P.Context(xy, wl.sigma, wl.cell, wl.rc, rings, wl.box)
    torch.cuda.synchronize()
    print("ok", c.setup_times(), c.info(), flush=True)
    c.close()
