"""Multi-rank host logic on CPU (world_size 2, gloo): the strip/halo plan the
library uses (rbf_plan_strips / rbf_plan_halo) exchanged over torch.distributed,
the deterministic scalar reduction rule (all-gather of per-rank partials summed in
rank order, reading Q14), and the bench's rank plumbing (id broadcast, max-over-
ranks timing).  NCCL kernels themselves need GPUs; these cover everything around
them."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_0909_5413_b200 as P

        rng = np.random.default_rng(7)
        counts = rng.integers(10, 40, size=24)  # points per cell row
        rs = np.concatenate([[0], np.cumsum(counts)])
        N = int(rs[-1])
        glob = rng.standard_normal(N)  # a global vector in sorted order
        b = P.plan_strips(counts, world, 2)
        h = P.plan_halo(rs, b, rank, 2, 1)
        own = glob[h["own_lo"]:h["own_hi"]].copy()
        ext = np.full(h["ext_hi"] - h["ext_lo"], np.nan)
        ext[h["own_lo"] - h["ext_lo"]:h["own_hi"] - h["ext_lo"]] = own
        # the halo exchange of comm.cu, with gloo point-to-point instead of NCCL
        reqs = []
        for side, peer in (("below", rank - 1), ("above", rank + 1)):
            if 0 <= peer < world:
                so, sc = h[f"{side}_send_off"], h[f"{side}_send_cnt"]
                reqs.append(dist.isend(torch.from_numpy(own[so:so + sc].copy()), peer))
        recv = {}
        for side, peer in (("below", rank - 1), ("above", rank + 1)):
            if 0 <= peer < world:
                rc = h[f"{side}_recv_cnt"]
                buf = torch.empty(rc, dtype=torch.float64)
                dist.recv(buf, peer)
                recv[side] = buf.numpy()
        for r in reqs:
            r.wait()
        for side, arr in recv.items():
            ro = h[f"{side}_recv_off"]
            ext[ro:ro + len(arr)] = arr
        ok_halo = bool(np.array_equal(ext, glob[h["ext_lo"]:h["ext_hi"]]))
        # deterministic reduction: all-gather of partials, summed in rank order
        part = torch.tensor([float(np.dot(own, own))], dtype=torch.float64)
        parts = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, part)
        tot = 0.0
        for p_ in parts:
            tot += float(p_.item())
        # id broadcast + max-over-ranks timing, as in bench.py
        obj = [b"x" * 128 if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        t = torch.tensor([float(rank + 1)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        q.put((rank, ok_halo, tot, obj[0] == b"x" * 128, float(t.item()),
               int(h["own_hi"] - h["own_lo"]), N))
    finally:
        dist.destroy_process_group()


def test_two_rank_halo_and_reductions():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(r[1] for r in res), "halo exchange did not reproduce the global slice"
    assert res[0][2] == res[1][2], "ranks must hold bit-identical reduced scalars"
    assert all(r[3] for r in res) and all(r[4] == world for r in res)
    assert sum(r[5] for r in res) == res[0][6]  # strips partition the points
