#!/usr/bin/env python
"""Benchmark of the PetRBF hot path on B200 (contract: README/DESIGN.md "Bench").

One step = one full interpolation solve of the largest single-GPU configuration in
BASELINE.json: configs[3], cfg4 (the paper-scale case north_star's strong scaling is
quoted on: 7072^2 = 50,013,184 lattice points, h/sigma = 0.8, rc = 6 sigma, cell =
4 sigma, GMRES(30) + RASM, tol 1e-15): rbf_setup (cell list + RASM setup) +
rbf_solve, inputs resident in HBM.  metric/unit follow BASELINE.json: solve time (s,
lower is better) plus the matvec Gpairs/s and the FP64-peak fractions.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl reference]

Multi-GPU: one rank per GPU (torchrun; `--gpus N` without a torchrun environment
re-launches itself under torch.distributed.run with N ranks), strips of cell rows with
NCCL halos/all-gathers (strong scaling: total work fixed).  --impl reference times the
oracle (plain C, host cores): its matvec on the full workload, its RASM setup and
per-iteration preconditioner + orthogonalisation cost on a bounded sample of the same
recipe scaled per point.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import rbf_workloads as W  # noqa: E402

METRIC = "fp64 GMRES+RASM solve time and matvec Gpairs/s at 1/2/4/8 B200, % FP64 peak"
FP64_PEAK_TFLOPS = 36.86  # measured DFMA peak on this pool's B200 (profiles/r01_fp64_peak.json, tools/clock_under_load.cu)
FLOP_PER_PAIR = 38        # algorithmic flops per in-cutoff pair
DMMA_PEAK_TFLOPS = 37.13  # measured fp64 tensor-core (DMMA) peak, profiles/r01_fp64_peak.json
SAMPLE_SIDE = 512         # oracle sample: 512^2 points of the same recipe


def _ncu_entry(kernel_prefix: str, workload: str):
    """The committed ncu --set full summary of one kernel on one workload
    (profiles/ncu_traffic.json: {workload: {kernel: {...}}}), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            d = json.load(f)[workload]
        for k, v in d.items():
            if k == kernel_prefix or k.startswith(kernel_prefix + "<"):
                return v
    except Exception:
        pass
    return None


def ncu_traffic(kernel_prefix: str, workload: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch, or None."""
    e = _ncu_entry(kernel_prefix, workload)
    return float(e["dram_bytes_per_launch"]) if e and "dram_bytes_per_launch" in e else None


def ncu_fp64(kernel_prefix: str, workload: str, key: str, scale: float = 1.0):
    """Executed FP64 fraction from the same capture: ALU flops (dadd + dmul + 2 dfma)
    over the DFMA peak ('fp64_alu_frac_of_peak') or the fp64 tensor pipe's % of peak
    ('fp64_tensor_pct_of_peak'), or None."""
    e = _ncu_entry(kernel_prefix, workload)
    return float(e[key]) * scale if e and key in e else None


def setup_flops(wl) -> float:
    """Algorithmic flops of the RASM setup: per subdomain with n = |Omega_c|,
    n1 = |own(c)|, n0 = n - n1: Cholesky n^3/3, W = L21 L11^-1 n1 n0^2, S^-1 n1^3,
    X = S^-1 [-W, I] 2 n1^2 n0 (multiply-add = 2 flops).  Whole-ring overlap only."""
    x0, y0, x1, y1 = wl.box
    ncx, ncy = int(np.ceil((x1 - x0) / wl.cell)), int(np.ceil((y1 - y0) / wl.cell))
    cx = np.clip(np.floor((wl.xy[:, 0] - x0) / wl.cell), 0, ncx - 1).astype(np.int64)
    cy = np.clip(np.floor((wl.xy[:, 1] - y0) / wl.cell), 0, ncy - 1).astype(np.int64)
    cnt = np.zeros((ncy + 2 * wl.rings, ncx + 2 * wl.rings))
    np.add.at(cnt, (cy + wl.rings, cx + wl.rings), 1.0)
    r = wl.rings
    n = sum(cnt[r + dy:r + dy + ncy, r + dx:r + dx + ncx] for dy in range(-r, r + 1) for dx in range(-r, r + 1))
    n1 = cnt[r:r + ncy, r:r + ncx]
    n0 = n - n1
    m = n1 > 0
    return float(np.sum((n ** 3 / 3 + n1 * n0 ** 2 + n1 ** 3 + 2 * n1 ** 2 * n0)[m]))


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# --------------------------------------------------------------------------- clocks
class Clocks:
    def __init__(self, gpu_index: int):
        self.path = f"/tmp/rbf_clocks_{os.getpid()}.csv"
        q = ("timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(gpu_index), f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def mark(self):
        """Start of the timed window (the sampler is started earlier, so its start-up
        does not fall into the timed steps).  nvidia-smi's first query (NVML start-up)
        stalls this process's CUDA calls for tens of ms: wait for its first samples so
        that the stall falls before the timed steps on short configs."""
        if self.p is not None:
            t_end = time.time() + 10.0
            while time.time() < t_end:
                try:
                    if sum(1 for _ in open(self.path)) >= 2:
                        break
                except OSError:
                    pass
                time.sleep(0.05)
        self.t0 = time.time()

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        t1 = time.time()
        self.p.terminate()
        self.p.wait()
        rows = []
        import datetime

        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 8:
                try:
                    ts = datetime.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                except ValueError:
                    ts = None
                if ts is None or getattr(self, "t0", None) is None or self.t0 - 0.5 <= ts <= t1 + 0.5:
                    rows.append(parts[1:])
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        load = [x for x in sm if mx and x > 0.5 * max(mx)] or sm
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[3 + k] == "Active"})
        return {"sm_mhz": statistics.median(load) if load else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


# --------------------------------------------------------------------------- reference arm
def sample_workload(cfg: int, full):
    """A bounded sample of the same recipe: SAMPLE_SIDE^2 points with the same h/sigma,
    cell/sigma, rc/sigma, jitter/rhs kind and tolerance (cfg5: the clustered recipe at
    SAMPLE_SIDE^2 points)."""
    n = SAMPLE_SIDE
    if cfg == 1:
        return full
    if cfg == 2:
        return W.make_lattice(n, jitter_frac=0.1, seed=2, rhs="gauss", s2=0.02, tol=full.tol)
    if cfg == 3:
        return W.make_lattice(n, seed=3, rhs="blobs", tol=full.tol)
    if cfg == 5:
        return W.make_clustered(n * n, seed=5, tol=full.tol)
    return W.make_lattice(n, rhs="gauss", s2=0.02, tol=full.tol)


def oracle_estimate(cfg: int, full=None):
    """The oracle (plain C + OpenMP on the host cores, as it stands) timed on this
    workload.  cfg1: the whole solve.  Larger configs (the oracle's RASM blocks for cfg4
    need 90 GB of host RAM): the oracle's matvec is timed on the FULL
    workload; the RASM setup and the per-iteration preconditioner apply +
    orthogonalisation are timed in a full oracle solve of a SAMPLE_SIDE^2 sample of the
    same recipe and scaled by the point count (both are O(N): per-cell work is the same,
    P:322, 465); the iteration count is the sample's (mesh-independent at fixed h/sigma,
    P:346).  Returns (seconds, description)."""
    import oracle as O

    full = full or W.config(cfg)
    wl = sample_workload(cfg, full)
    t0 = time.perf_counter()
    P = O.Rasm(wl.xy, wl.sigma, wl.rc, wl.box, wl.cell, wl.rings, wl.overlap_width)
    t_su = time.perf_counter() - t0
    opA = O.op_rbf(wl.xy, wl.sigma, wl.rc, wl.box, wl.cell)
    t0 = time.perf_counter()
    res = O.gmres(opA, O.op_rasm(P), wl.f, rtol=full.tol)
    t_sol = time.perf_counter() - t0
    w_s = np.random.default_rng(0).standard_normal(wl.n)
    t0 = time.perf_counter()
    O.matvec_cells(wl.xy, w_s, wl.sigma, wl.rc, wl.box, wl.cell)
    t_mv_s = time.perf_counter() - t0
    P.close()
    n_mv = res.iterations + res.restarts + 1   # one per iteration, per restart residual, final check
    if wl is full:
        return t_su + t_sol, (f"oracle setup + solve of {full.name} itself ({full.n} points, "
                              f"{res.iterations} it): setup {t_su:.2f} s, solve {t_sol:.2f} s")
    w = np.random.default_rng(0).standard_normal(full.n)
    t0 = time.perf_counter()
    O.matvec_cells(full.xy, w, full.sigma, full.rc, full.box, full.cell)
    t_mv = time.perf_counter() - t0
    scale = full.n / wl.n
    rest = max(t_sol - n_mv * t_mv_s, 0.0) / max(res.iterations, 1)  # PC apply + orth per iteration
    est = t_su * scale + n_mv * t_mv + res.iterations * rest * scale
    desc = (f"matvec timed on {full.name} itself ({full.n} points): {t_mv:.2f} s; RASM setup "
            f"{t_su:.2f} s and PC apply + orthogonalisation {rest * 1e3:.1f} ms/iteration timed in "
            f"a full oracle solve of a {wl.n}-point sample of the same recipe ({wl.name}, "
            f"{res.iterations} it, {res.restarts} restarts), x{scale:.1f} per point; "
            f"estimate = setup + {n_mv} matvecs + {res.iterations} iterations x (PC + orth)")
    return est, desc


def run_reference(args, rank, world):
    if rank != 0:
        return
    # all host cores (torchrun exports OMP_NUM_THREADS=1 to every rank: override it
    # before the oracle's OpenMP runtime is loaded)
    cores = os.cpu_count() or 1
    os.environ["OMP_NUM_THREADS"] = str(cores)
    full = W.config(args.config)
    times = []
    desc = ""
    for i in range(args.warmup + args.steps):
        v, desc = oracle_estimate(args.config, full)
        if i >= args.warmup:
            times.append(v)
    v = statistics.mean(times)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": v * 1e3,
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": full.name, "N": full.n},
            "cpu_baseline": {"value": v, "unit": "s", "cores": cores, "kind": "oracle",
                             "sample": desc, **host_info()},
            "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def host_info():
    """CPU model and host RAM of the box the oracle runs on (recorded with
    the oracle timing)."""
    model, ram = None, None
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
        with open("/proc/meminfo") as fh:
            for ln in fh:
                if ln.startswith("MemTotal"):
                    ram = round(int(ln.split()[1]) / 2**20, 1)
                    break
    except OSError:
        pass
    return {"cpu_model": model, "host_ram_gib": ram}


# --------------------------------------------------------------------------- our arm
def run_ours(args, rank, world):
    import torch
    import torch.distributed as dist

    import paper_0909_5413_b200 as P

    if os.environ.get("RBF_BENCH_NO_GRAPH"):  # profiling only: host-driven GMRES loop
        P.set_option("solve_graph", 0)
    if os.environ.get("RBF_BENCH_LOG_ALLOC"):  # diagnostics: slow device allocations
        P.set_option("log_slow_alloc", int(os.environ["RBF_BENCH_LOG_ALLOC"]))
    dev = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream()
    weak = args.scaling == "weak"
    wl = W.weak(world) if weak else W.config(args.config)
    xy_h = torch.from_numpy(wl.xy)
    f_h = torch.from_numpy(wl.f)
    xy = xy_h.cuda()
    f = f_h.cuda()
    nccl_id = None
    if world > 1:
        obj = [P.get_nccl_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    kw = dict(rank=rank, nranks=world, comm="nccl", nccl_id=nccl_id) if world > 1 else {}
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")

    # Arnoldi orthogonalisation: MGS (BJ:5 "modified Gram-Schmidt", reading Q12) for every
    # GPU count, so a strong-scaling series runs one algorithm; --orth dcgs2 selects the
    # one-reduction variant (reading Q27)
    orth = args.orth or "mgs"

    def step(timing=False):
        c = P.Context(xy, wl.sigma, wl.cell, wl.rc, wl.rings, wl.box, **kw)
        fl = c.to_local(f)
        lam, rep = c.solve(fl, rtol=wl.tol, timing=timing, orth=orth)
        return c, lam, rep

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # the clock sampler starts before the warm-up (nvidia-smi's start-up stays out of the
    # timed steps); only its samples inside the timed window are kept
    clocks = Clocks(dev) if not os.environ.get("RBF_BENCH_NO_CLOCKS") else None
    # warm-up (also: facts for the roofline)
    for _ in range(args.warmup):
        c, lam, rep = step()
        info = c.info()
        c.close()
    barrier()
    # timed region: K steps, each bracketed by CUDA events; L2 flushed between steps
    if clocks:
        clocks.mark()
    launches0 = P.launch_count()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    reps, setups = [], []
    barrier()
    for k in range(args.steps):
        flush.fill_(float(k))
        ev[k][0].record(stream)
        c, lam, rep = step()  # graph-driven solve (no per-phase events in the timed steps)
        ev[k][1].record(stream)
        reps.append(rep)
        setups.append(c.setup_times())
        c.close()
    barrier()
    launches = P.launch_count() - launches0
    clk = clocks.stop() if clocks else {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["not sampled"]}
    ms = [a.elapsed_time(b) for a, b in ev]
    t_local = sum(ms)
    t = torch.tensor([t_local], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_per_step = float(t.item()) / args.steps

    # ---- phase breakdown: one more step with per-phase CUDA events (the host-driven
    # loop records events between the phases of every iteration), after the timed region
    c, lam, rep_t = step(timing=True)
    c.close()
    # ---- per-kernel measurements for the roofline (same stream, after the timed region)
    c = P.Context(xy, wl.sigma, wl.cell, wl.rc, wl.rings, wl.box, **kw)
    info = c.info()
    n_pairs_local = c.count_pairs()
    mstats = c.matvec_stats()  # executed (target, entry) slots vs in-cutoff pairs
    w = torch.randn(c.n_local, dtype=torch.float64, device="cuda")
    y = torch.empty_like(w)

    def time_op(fn, reps_=20):
        fn()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps_):
            fn()
        e1.record(stream)
        e1.synchronize()
        return e0.elapsed_time(e1) / reps_

    mv_ms = time_op(lambda: c.matvec(w, y))
    pc_ms = time_op(lambda: c.rasm_apply(w, y))
    # interpolant evaluation (the paper's application): the weights
    # evaluated on the interior corner lattice of the data's lattice (2048^2 for cfg5)
    ev = None
    if not weak:
        nq = wl.meta.get("n_side", 2048)
        cq = -1.0 + (np.arange(nq - 1) + 1) * (2.0 / nq)
        QX, QY = np.meshgrid(cq, cq)
        qd = torch.from_numpy(np.stack([QX.ravel(), QY.ravel()], 1).copy()).cuda()
        sd = torch.empty(qd.shape[0], dtype=torch.float64, device="cuda")
        ev_pairs = c.evaluate_count_pairs(qd)
        ev_ms = time_op(lambda: c.evaluate(qd, w, sd), reps_=5)
        ev = {"queries": int(qd.shape[0]), "query_set": f"interior corners of the {nq}^2 lattice",
              "pairs": int(ev_pairs), "ms": ev_ms, "gpairs_s": ev_pairs / (ev_ms * 1e-3) / 1e9,
              "fp64_frac_useful": ev_pairs * FLOP_PER_PAIR / (ev_ms * 1e-3) / (FP64_PEAK_TFLOPS * 1e12),
              "includes": "query keys + radix sort + weight pack + evaluation kernel"}
        del qd, sd
    c.close()
    n_loc = c.n_local
    iters = statistics.mean(r.iterations for r in reps)
    # phase shares inside the timed steps (library CUDA events on the launching stream)
    mv_live = rep_t.ms_matmult
    pc_live = rep_t.ms_pcapply
    orth_live = rep_t.ms_orth
    # launches inside the timing step's phases: the matvec once per iteration and once per
    # restart residual; the PC once more (beta0).  The report's final residuals are
    # computed outside the timed phases.
    mv_launches = rep_t.iterations + rep_t.restarts
    pc_launches = rep_t.iterations + rep_t.restarts + 1
    x_bytes = 8 * info["x_doubles"]
    pc_alg_bytes = x_bytes + 16 * n_loc          # X streamed once + u read + z written
    mv_alg_flops = FLOP_PER_PAIR * n_pairs_local
    hbm_peak, hbm_src = peaks()
    pc_per_launch_ms = pc_live / max(pc_launches, 1)   # live: phase time / launches in the phase
    mv_per_launch_ms = mv_live / max(mv_launches, 1)
    pc_gbs = pc_alg_bytes / (pc_per_launch_ms * 1e-3) / 1e9
    mv_tflops = mv_alg_flops / (mv_per_launch_ms * 1e-3) / 1e12
    # Arnoldi (MGS) vector traffic: step k of a cycle reads w and v_0..v_k and writes the
    # new basis vector: (k + 3) x 8 B per point (algorithmic)
    orth_bytes = 8.0 * n_loc * sum((i % 30) + 3 for i in range(rep_t.iterations))
    orth_gbs = orth_bytes / (orth_live * 1e-3) / 1e9 if orth_live > 0 else None
    rasm_ms = statistics.mean(sd["rasm"] for sd in setups)
    sflops = setup_flops(wl) / world if wl.overlap_width == 0.0 else None
    su_tflops = sflops / (rasm_ms * 1e-3) / 1e12 if sflops else None
    tr_src = f"profiles/ncu_traffic.json ({wl.name} capture)"
    roof_all = {
        "k_matvec": {"kernel": "k_matvec", "bound": "alu", "achieved": mv_tflops,
                     "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s", "frac": mv_tflops / FP64_PEAK_TFLOPS,
                     "traffic": ncu_traffic("k_matvec", wl.name),
                     "peak_source": "measured DFMA, tools/clock_under_load.cu (profiles/r01_fp64_peak.json)",
                     "alg_flops_per_launch": mv_alg_flops, "ms_per_launch": mv_per_launch_ms,
                     "ms_per_step": mv_live,
                     "fp64_pipe_active_ncu": ncu_fp64("k_matvec", wl.name, "fp64_pipe_pct_of_peak", 0.01)},
        "k_rasm_apply": {"kernel": "k_rasm_apply", "bound": "hbm", "achieved": pc_gbs, "peak": hbm_peak,
                         "unit": "GB/s", "frac": pc_gbs / hbm_peak, "peak_source": hbm_src,
                         "traffic": ncu_traffic("k_rasm_apply", wl.name),
                         "alg_bytes_per_launch": pc_alg_bytes, "ms_per_launch": pc_per_launch_ms,
                         "ms_per_step": pc_live},
        "k_rasm_setup_tc": {"kernel": "k_rasm_setup_tc", "bound": "tensor", "achieved": su_tflops,
                            "peak": DMMA_PEAK_TFLOPS, "unit": "TFLOP/s",
                            "frac": su_tflops / DMMA_PEAK_TFLOPS if su_tflops else None,
                            "peak_source": "measured fp64 DMMA (profiles/r01_fp64_peak.json); nominal "
                                           "148 SM x 128 flop/clk x 1.965 GHz = 37.2",
                            "traffic": ncu_traffic("k_rasm_setup_tc", wl.name),
                            "ms_per_launch": rasm_ms, "ms_per_step": rasm_ms,
                            "alg_flops_per_launch": sflops,
                            "executed_frac_ncu": ncu_fp64("k_rasm_setup_tc", wl.name,
                                                          "fp64_tensor_pct_of_peak", 0.01),
                            "flops_model": "per subdomain n^3/3 + n1 n0^2 + n1^3 + 2 n1^2 n0 "
                                           "(Cholesky, W, S^-1, X)"},
        "arnoldi": {"kernel": "MGS vector kernels (k_arnoldi_* / k_axpy_dot)", "bound": "hbm",
                    "achieved": orth_gbs, "peak": hbm_peak, "unit": "GB/s",
                    "frac": orth_gbs / hbm_peak if orth_gbs else None, "peak_source": hbm_src,
                    "alg_bytes_per_step": orth_bytes, "ms_per_step": orth_live,
                    "bytes_model": "(k + 3) x 8 B per point for Arnoldi step k of a cycle"},
    }
    for r_ in roof_all.values():
        if r_.get("traffic") is not None:
            r_["traffic_source"] = tr_src
            r_["traffic_unit"] = "DRAM bytes read + written per launch"
    # the contract's `roofline`: the kernel with the largest share of the step
    dom = max(("k_matvec", "k_rasm_apply", "k_rasm_setup_tc", "arnoldi"),
              key=lambda k: roof_all[k]["ms_per_step"] or 0.0)
    roof = dict(roof_all[dom])
    roof["share_of_step"] = roof["ms_per_step"] / ms_per_step
    roof_all = list(roof_all.values())
    gpairs = n_pairs_local / (mv_ms * 1e-3) / 1e9
    if world > 1:
        tot = torch.tensor([float(n_pairs_local)], dtype=torch.float64, device="cuda")
        dist.all_reduce(tot)
        mvt = torch.tensor([mv_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(mvt, op=dist.ReduceOp.MAX)
        gpairs = float(tot.item()) / (float(mvt.item()) * 1e-3) / 1e9

    # ---- e2e: host buffers through the public API.  N=1: rbf_interpolate_host (one
    # C call); N>1: per rank pinned xy, f -> device, Context (strip setup) + to_local +
    # solve, this rank's weights -> host; max over ranks of the wall time.
    e2e = None
    if world > 1:
        xy_pin = xy_h.pin_memory()
        f_pin = f_h.pin_memory()
        e2e_ms, d2h = [], 0
        for k in range(max(1, min(args.steps, 3)) + 1):
            flush.fill_(float(k))
            barrier()
            t0 = time.perf_counter()
            xy_d = xy_pin.cuda(non_blocking=True)
            f_d = f_pin.cuda(non_blocking=True)
            c = P.Context(xy_d, wl.sigma, wl.cell, wl.rc, wl.rings, wl.box, **kw)
            lam, rep_h = c.solve(c.to_local(f_d), rtol=wl.tol, orth=orth)
            if k == 0:  # the rank's result buffer, pinned (allocated in the untimed first pass)
                lam_pin = torch.empty(lam.shape[0], dtype=torch.float64).pin_memory()
            lam_pin.copy_(lam, non_blocking=True)
            lam_h = lam_pin
            torch.cuda.synchronize()
            dt = torch.tensor([(time.perf_counter() - t0) * 1e3], dtype=torch.float64, device="cuda")
            c.close()
            dist.all_reduce(dt, op=dist.ReduceOp.MAX)
            if k > 0:
                e2e_ms.append(float(dt.item()))
            d2h = int(lam_h.numel() * 8)
        e2e = {"value": statistics.mean(e2e_ms) / 1e3, "unit": "s",
               "h2d_bytes_per_step": int(xy_pin.numel() * 8 + f_pin.numel() * 8),
               "d2h_bytes_per_step": d2h,
               "api": "per rank: Context + to_local + solve (pinned host xy, f -> this rank's "
                      "lambda in pinned host memory); bytes per rank; max over ranks"}
    if world == 1:
        xy_pin = xy_h.pin_memory().numpy()
        f_pin = f_h.pin_memory().numpy()
        lam_pin = torch.empty(f_h.shape[0], dtype=torch.float64).pin_memory().numpy()  # the result, pinned
        e2e_ms = []
        for k in range(max(1, min(args.steps, 3)) + 1):
            flush.fill_(float(k))
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            lam_h, rep_h = P.interpolate_host(xy_pin, f_pin, wl.sigma, wl.cell, wl.rc, wl.rings,
                                              wl.box, rtol=wl.tol, out=lam_pin)
            torch.cuda.synchronize()
            if k > 0:
                e2e_ms.append((time.perf_counter() - t0) * 1e3)
        e2e = {"value": statistics.mean(e2e_ms) / 1e3, "unit": "s",
               "h2d_bytes_per_step": int(xy_pin.nbytes + f_pin.nbytes),
               "d2h_bytes_per_step": int(lam_h.nbytes),
               "api": "rbf_interpolate_host (pinned host xy, f -> pinned host lambda)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = os.cpu_count() or 1
        os.environ["OMP_NUM_THREADS"] = str(cores)
        v, desc = oracle_estimate(args.config, None if weak else wl)
        cpu = {"value": v, "unit": "s", "cores": cores, "kind": "oracle", "sample": desc, **host_info()}

    if rank == 0:
        r0 = reps[0]
        line = {
            "metric": METRIC, "value": ms_per_step / 1e3, "unit": "s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": False, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": wl.name, "N": wl.n,
                       "desc": (W.CONFIG_DESCRIPTIONS[2] + f"; {world} copies stacked in y, one per GPU"
                                if weak else W.CONFIG_DESCRIPTIONS[args.config]),
                       "orth": orth,
                       "parallelism": f"strips{world}", "l2": "flushed (256 MiB write) between steps",
                       "step": "rbf_setup (cell list + RASM setup) + rbf_solve, inputs in HBM"},
            "iterations": iters, "restarts": r0.restarts,
            "converged": all(r.converged for r in reps),
            "status": sorted({int(r.status) for r in reps}), "resid_est": r0.resid_est,
            "resid_true": r0.resid_true, "resid_precond": r0.resid_precond,
            "setup_ms": {k: statistics.mean(sd[k] for sd in setups) for k in setups[0]},
            "phase_ms": {"matvec": mv_live, "rasm_apply": pc_live, "orth": orth_live,
                         "solve_host_loop": rep_t.ms_total,
                         "source": "one extra step with per-phase events (host-driven loop)"},
            "solve_ms": statistics.mean(r.ms_total for r in reps),
            "solve_path": ("one CUDA graph per solve (device-side while loops)" if world == 1 else
                           "host-driven loop, NCCL halos + all-gathers"),
            "orth": orth,
            "other_ms": ms_per_step - statistics.mean(r.ms_total for r in reps)
                        - statistics.mean(sd["total"] for sd in setups),
            "matvec_gpairs_s": gpairs,
            "matvec_ms": mv_ms, "rasm_apply_ms": pc_ms,
            "matvec_slots_per_pair": 2.0 * mstats["ell_entries"] / max(n_pairs_local, 1),
            "matvec_fp64_frac_useful": gpairs * 1e9 * FLOP_PER_PAIR / (FP64_PEAK_TFLOPS * 1e12),
            "rasm_apply_gbs": pc_alg_bytes / (pc_ms * 1e-3) / 1e9,
            "evaluate": ev,
            "step_ms": [round(x, 3) for x in ms],
            "step_setup_solve_ms": [[round(sd["cell_list"], 2), round(sd["nlist"], 2), round(sd["rasm"], 2),
                                     round(r.ms_total, 2)] for sd, r in zip(setups, reps)],
            "roofline": roof, "roofline_all": roof_all, "clocks": clk, "gpu_launches": int(launches),
            "e2e": e2e, "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4,
                    help="BASELINE.json config (default 4: the largest single-GPU case, 50M points)")
    ap.add_argument("--dry-run-ranks", action="store_true",
                    help="print this rank's launch environment as JSON and exit (launcher test)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--scaling", choices=["strong", "weak"], default="strong",
                    help="strong: one BASELINE config on all GPUs (default); weak: one cfg2-sized "
                         "block per GPU (rbf_workloads.weak)")
    ap.add_argument("--orth", choices=["mgs", "cgs2", "dcgs2"], default=None,
                    help="GMRES orthogonalisation (default: mgs for every GPU count, BJ:5)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch this script under torch.distributed.run
        import socket

        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
               os.path.abspath(__file__), *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != args.gpus:
        print(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}; using WORLD_SIZE",
              file=sys.stderr)
    if args.dry_run_ranks:
        print(json.dumps({k: os.environ.get(k) for k in
                          ("RANK", "LOCAL_RANK", "WORLD_SIZE", "MASTER_ADDR", "MASTER_PORT")}),
              flush=True)
        return
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        dist.init_process_group("nccl")
    run_ours(args, rank, world)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
