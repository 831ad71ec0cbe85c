"""One rbf_setup on a config with the in-tree (or given) librbf.so; prints the setup times."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_0909_5413_b200.rbf as R
if len(sys.argv) > 2:
    R.LIB_PATH = os.path.abspath(sys.argv[2])
import rbf_workloads as W
wl = W.config(int(sys.argv[1]))
xy = torch.from_numpy(wl.xy).cuda()
c = R.Context(xy, wl.sigma, wl.cell, wl.rc, wl.rings, wl.box)
torch.cuda.synchronize()
print("ok", c.setup_times(), flush=True)
