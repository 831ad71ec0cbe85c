"""Uninitialised-memory checks: every SM's shared memory filled with NaN right before
each setup (rbf_debug_poison_shared) and every library buffer allocated NaN-filled
(option "poison"), then the same parity bars as tests/test_gpu_parity.py.  A kernel
that reads shared memory or scratch it never wrote -- even multiplied by zero --
turns the result into NaN here.  (Found: the LU path's 32x32 shared L11/U block was
filled only up to the last panel's width; 0 * stale shared memory gave NaN.)"""
import numpy as np
import pytest

import oracle as O
import rbf_workloads as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_0909_5413_b200 as P  # noqa: E402


@pytest.fixture(autouse=True)
def poisoned_allocations(lib_options):
    lib_options(poison=1)


def ctx_for(wl, rings=None, **kw):
    xy = torch.from_numpy(wl.xy).cuda()
    kw.setdefault("overlap_width", wl.overlap_width)
    P.poison_shared()
    return P.Context(xy, wl.sigma, wl.cell, wl.rc, wl.rings if rings is None else rings, wl.box, **kw)


def to_caller(ctx, v_loc):
    out = np.zeros(ctx.n)
    out[ctx.local_index().cpu().numpy()] = v_loc.cpu().numpy()
    return out


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def test_poison_hook_fills_shared_memory_and_buffers():
    P.poison_shared()  # must run and synchronise without error
    wl = W.make_lattice(24)
    with ctx_for(wl) as c:
        assert c.info()["bytes_device"] > 0


APPLY = [("tc-ragged24", W.make_lattice(24), 1, {}),
         ("tc-jitter37", W.make_lattice(37, jitter_frac=0.3, seed=3), 1, {}),
         ("lu-2rings", W.make_lattice(48, jitter_frac=0.1, seed=5), 2, {}),
         ("lu-3rings", W.make_lattice(48, seed=5), 3, {}),
         ("box-lu", W.make_lattice(48, jitter_frac=0.1, seed=5), 2, {"overlap_width": "1.5"}),
         ("asm-rings0", W.make_lattice(30, jitter_frac=0.1, seed=2), 0, {"schwarz": "asm"}),
         ("asm-jitter40", W.make_lattice(40, jitter_frac=0.1, seed=7), 1, {"schwarz": "asm"})]


@pytest.mark.parametrize("name,wl,rings,kw", APPLY, ids=[a[0] for a in APPLY])
def test_rasm_apply_poisoned(name, wl, rings, kw):
    kw = dict(kw)
    d = float(kw.pop("overlap_width")) * wl.cell if "overlap_width" in kw else 0.0
    schwarz = kw.get("schwarz", "rasm")
    r = np.random.default_rng(7).standard_normal(wl.n)
    Pc = O.Rasm(wl.xy, wl.sigma, wl.rc, wl.box, wl.cell, rings, overlap_width=d)
    ref = Pc.apply(r, schwarz)
    Pc.close()
    with ctx_for(wl, rings=rings, overlap_width=d, **kw) as c:
        z = to_caller(c, c.rasm_apply(c.to_local(torch.from_numpy(r).cuda())))
    assert np.all(np.isfinite(z))
    assert rel(z, ref) <= 1e-10


@pytest.mark.parametrize("kern", [1, 2], ids=["two-per-sm", "pipelined"])
@pytest.mark.parametrize("wl", [W.make_lattice(24), W.make_lattice(37, jitter_frac=0.3, seed=3)],
                         ids=["ragged24", "jitter37"])
def test_rasm_apply_poisoned_other_setup_kernels(wl, kern, lib_options):
    """The two-per-SM and pipelined setup kernels (option setup_kernel) with NaN-filled
    shared memory, workspace and buffers: every tile, retired row and ring slot they read
    was written first."""
    lib_options(setup_kernel=kern)
    r = np.random.default_rng(7).standard_normal(wl.n)
    Pc = O.Rasm(wl.xy, wl.sigma, wl.rc, wl.box, wl.cell, 1)
    ref = Pc.apply(r)
    Pc.close()
    with ctx_for(wl) as c:
        z = to_caller(c, c.rasm_apply(c.to_local(torch.from_numpy(r).cuda())))
    assert np.all(np.isfinite(z))
    assert rel(z, ref) <= 1e-10


@pytest.mark.parametrize("wl", [W.config(1), W.make_lattice(37, jitter_frac=0.3, seed=3)],
                         ids=["cfg1", "jitter37"])
def test_matvec_poisoned(wl):
    w = np.random.default_rng(12).standard_normal(wl.n)
    ref = O.matvec_brute(wl.xy, w, wl.sigma, wl.rc)
    with ctx_for(wl, rings=0) as c:
        got = to_caller(c, c.matvec(c.to_local(torch.from_numpy(w).cuda())))
    assert rel(got, ref) <= 1e-12


@pytest.mark.parametrize("orth", ["mgs", "cgs2", "dcgs2"])
def test_solve_poisoned(orth):
    wl = W.make_lattice(40, jitter_frac=0.1, seed=7)
    ref = O.solve(wl.xy, wl.f, wl.sigma, wl.rc, wl.box, wl.cell, wl.rings, rtol=wl.tol, orth=orth)
    with ctx_for(wl) as c:
        P.poison_shared()
        lam, rep = c.solve(c.to_local(torch.from_numpy(wl.f).cuda()), rtol=wl.tol, orth=orth)
        lam = to_caller(c, lam)
    assert rep.converged and ref.converged
    assert abs(rep.iterations - ref.iterations) <= 2
    assert rep.resid_true <= 1e-10
    assert rel(lam, ref.x) <= 1e-8


@pytest.mark.parametrize("tbox", [False, True], ids=["rc", "tbox"])
def test_matvec_and_evaluate_poisoned(tbox):
    wl = W.make_lattice(37, jitter_frac=0.3, seed=3)
    tau = 5.0 * wl.sigma
    rng = np.random.default_rng(44)
    w = rng.standard_normal(wl.n)
    q = np.column_stack([rng.uniform(-1, 1, 600), rng.uniform(-1, 1, 600)])
    if tbox:
        ref_y = O.matvec_tbox(wl.xy, w, wl.sigma, wl.box, wl.cell, tau)
        ref_s = O.evaluate_tbox(q, wl.xy, w, wl.sigma, wl.box, wl.cell, tau)
    else:
        ref_y = O.matvec_brute(wl.xy, w, wl.sigma, wl.rc)
        ref_s = O.evaluate(q, wl.xy, w, wl.sigma, wl.rc)
    with ctx_for(wl, rings=0, trunc_width=tau if tbox else 0.0) as c:
        wl_ = c.to_local(torch.from_numpy(w).cuda())
        P.poison_shared()
        y = to_caller(c, c.matvec(wl_))
        P.poison_shared()
        s = c.evaluate(torch.from_numpy(q).cuda(), wl_).cpu().numpy()
    assert rel(y, ref_y) <= 1e-12
    assert rel(s, ref_s) <= 1e-12


@pytest.mark.parametrize("orth", ["mgs", "dcgs2"])
def test_threads_strips_solve_poisoned(orth):
    """The multi-strip path (halo plans and exchange, rank-ordered reductions) on the
    in-process transport, every buffer NaN-filled, against the single-strip solve."""
    import os
    import threading

    wl = W.make_lattice(60, jitter_frac=0.1, seed=5)
    xy = torch.from_numpy(wl.xy).cuda()
    f = torch.from_numpy(wl.f).cuda()
    with ctx_for(wl) as c1:
        lam1, rep1 = c1.solve(c1.to_local(f), rtol=1e-13, orth=orth)
        lam1 = c1.from_local(lam1).cpu().numpy()
    nranks, key = 2, os.urandom(128)
    out, err = [None] * nranks, [None] * nranks

    def run(r):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                with P.Context(xy, wl.sigma, wl.cell, wl.rc, 1, wl.box, rank=r, nranks=nranks,
                               comm="threads", nccl_id=key, stream=st) as c:
                    lam, rep = c.solve(c.to_local(f), rtol=1e-13, orth=orth)
                    out[r] = (c.from_local(lam).cpu().numpy(), rep)
            st.synchronize()
        except BaseException as e:  # noqa: BLE001 - reported below
            err[r] = e

    P.poison_shared()
    ths = [threading.Thread(target=run, args=(r,), daemon=True) for r in range(nranks)]
    for t in ths:
        t.start()
    for t in ths:
        t.join(300)
    assert not any(t.is_alive() for t in ths)
    for e in err:
        if e is not None:
            raise e
    assert rep1.converged
    assert len({o[1].iterations for o in out}) == 1
    for lam, rep in out:
        assert rep.converged and abs(rep.iterations - rep1.iterations) <= 1
        assert rep.resid_true <= 1e-10
        assert np.all(np.isfinite(lam))
    # the strips' owned entries, summed over ranks, are the single-strip solution
    got = sum(o[0] for o in out)
    assert rel(got, lam1) <= 1e-8
