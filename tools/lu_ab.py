"""A/B of LU-path options on workloads whose subdomains take the LU path: setup time
(median of reps) and the RASM apply of a fixed vector compared between the variants.
Usage: lu_ab.py option=v1,v2 [case ...]; cases: lat2 (200^2 jittered lattice, 2 rings,
625-point subdomains), lat3 (3 rings), clu256k (cfg5 recipe at 262,144 points: the same
cluster cell sizes), cfg5.  Not part of the product."""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0909_5413_b200 as P  # noqa: E402
import rbf_workloads as W  # noqa: E402


def make(case):
    if case == "lat2":
        return W.make_lattice(200, jitter_frac=0.1, seed=3), 2
    if case == "lat3":
        return W.make_lattice(200, jitter_frac=0.1, seed=3), 3
    if case == "clu256k":
        return W.make_clustered(262144, seed=5), 1
    if case == "cfg5":
        return W.config(5), 1
    raise ValueError(case)


def main():
    name, vals = sys.argv[1].split("=")
    vals = [int(v) for v in vals.split(",")]
    cases = sys.argv[2:] or ["lat2", "lat3", "clu256k"]
    reps = int(os.environ.get("REPS", "3"))
    for case in cases:
        wl, rings = make(case)
        xy = torch.from_numpy(wl.xy).cuda()
        out = {}
        for v in vals:
            P.set_option(name, v)
            ts, z = [], None
            for r in range(reps + 1):
                torch.cuda.synchronize()
                with P.Context(xy, wl.sigma, wl.cell, wl.rc, rings, wl.box) as c:
                    st = c.setup_times()
                    if r > 0:
                        ts.append(st["rasm"])
                    if r == reps:
                        g = torch.Generator(device="cpu").manual_seed(7)
                        u = torch.randn(c.n_local, dtype=torch.float64, generator=g).cuda()
                        z = c.rasm_apply(u)
                        info, lu = c.info(), c.lu_stats()
            out[v] = z
            print(f"{case} {name}={v}: rasm setup {statistics.median(ts):.2f} ms (all {[round(t, 2) for t in ts]}) "
                  f"n_lu {info['n_lu']} max_ov {info['max_ov']} lu {lu}", flush=True)
        base = out[vals[0]]
        for v in vals[1:]:
            d = (out[v] - base).abs().max().item() / base.abs().max().item()
            print(f"{case}: apply max rel diff {name}={v} vs {vals[0]}: {d:.3e} "
                  f"bitwise={bool(torch.equal(out[v], base))}", flush=True)


if __name__ == "__main__":
    main()
