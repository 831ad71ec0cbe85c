"""Pins for the oracle's RASM preconditioner, dense factorizations, GMRES and
full solve (CPU only).

The RASM pin builds Eq.(11) M^-1 = sum_i R~_i^T A_i^-1 R_i literally from 0/1
restriction matrices found by a brute-force membership scan in numpy
(SPEC S:392); the solve pins are the dense direct solve and the deconvolution
closed form G_sigma * G_tau = G_s ([D3]).
"""
import json
import math
import os

import numpy as np
import pytest

import oracle as O
import rbf_workloads as W

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "lattice_constants.json")))


def _cells(xy, box, cell):
    ncx, ncy = O.grid_dims(box, cell)
    cx = np.clip(np.floor((xy[:, 0] - box[0]) / cell), 0, ncx - 1).astype(np.int64)
    cy = np.clip(np.floor((xy[:, 1] - box[1]) / cell), 0, ncy - 1).astype(np.int64)
    return cx, cy, ncx, ncy


def _explicit_minv(xy, sigma, rc, box, cell, rings, variant="rasm", overlap_width=0.0):
    """Eq.(5),(9),(11) with explicit 0/1 matrices (N small); overlap_width > 0: the
    block's points inside the cell box grown by overlap_width (reading Q24)."""
    n = xy.shape[0]
    d = xy[:, None, :] - xy[None, :, :]
    r2 = d[..., 0] ** 2 + d[..., 1] ** 2
    A = np.where(r2 < rc * rc, np.exp(-r2 / (2 * sigma * sigma)) / (2 * math.pi * sigma * sigma), 0.0)
    cx, cy, ncx, ncy = _cells(xy, box, cell)
    Minv = np.zeros((n, n))
    for c in range(ncx * ncy):
        ccx, ccy = c % ncx, c // ncx
        own = np.nonzero((cx == ccx) & (cy == ccy))[0]
        if own.size == 0:
            continue
        inblock = (np.abs(cx - ccx) <= rings) & (np.abs(cy - ccy) <= rings)
        if overlap_width > 0:
            lx, hx = box[0] + float(ccx) * cell, box[0] + float(ccx + 1) * cell
            ly, hy = box[1] + float(ccy) * cell, box[1] + float(ccy + 1) * cell
            d = overlap_width
            inbox = ((xy[:, 0] >= lx - d) & (xy[:, 0] <= hx + d) & (xy[:, 1] >= ly - d)
                     & (xy[:, 1] <= hy + d))
            inblock &= inbox | ((cx == ccx) & (cy == ccy))
        ov = np.nonzero(inblock)[0]
        R = np.zeros((ov.size, n)); R[np.arange(ov.size), ov] = 1.0
        Ai = R @ A @ R.T
        if variant == "rasm":
            Rt = np.zeros((ov.size, n))
            for q, j in enumerate(ov):
                if j in set(own.tolist()):
                    Rt[q, j] = 1.0
        else:
            Rt = R
        Minv += Rt.T @ np.linalg.inv(Ai) @ R
    return Minv, A


@pytest.mark.parametrize("wl,rings", [(W.make_lattice(14, jitter_frac=0.1, seed=3), 1),
                                      (W.make_lattice(17), 1),
                                      (W.make_lattice(15, jitter_frac=0.3, seed=2), 1),
                                      (W.make_lattice(14), 0)])
def test_rasm_equals_explicit_eq11(wl, rings):
    Minv, _ = _explicit_minv(wl.xy, wl.sigma, wl.rc, wl.box, wl.cell, rings)
    P = O.Rasm(wl.xy, wl.sigma, wl.rc, wl.box, wl.cell, rings)
    assert P.status == 0
    rng = np.random.default_rng(4)
    for _ in range(3):
        r = rng.standard_normal(wl.n)
        z = P.apply(r)
        ref = Minv @ r
        assert np.linalg.norm(z - ref) / np.linalg.norm(ref) < 1e-11
    P.close()


def test_asm_equals_explicit_eq8():
    wl = W.make_lattice(14, jitter_frac=0.1, seed=8)
    Minv, _ = _explicit_minv(wl.xy, wl.sigma, wl.rc, wl.box, wl.cell, 1, variant="asm")
    P = O.Rasm(wl.xy, wl.sigma, wl.rc, wl.box, wl.cell, 1)
    r = np.random.default_rng(5).standard_normal(wl.n)
    ref = Minv @ r
    assert np.linalg.norm(P.apply(r, "asm") - ref) / np.linalg.norm(ref) < 1e-11


def test_single_subdomain_is_exact_inverse():
    # Eq.(11) with p = 1, R = R~ = I: M^-1 = A_rc^-1
    wl = W.make_lattice(12, jitter_frac=0.1, seed=6)
    P = O.Rasm(wl.xy, wl.sigma, wl.rc, wl.box, 4.0, 0)
    assert P.nsub == 1
    A = O.assemble_dense(wl.xy, wl.sigma, wl.rc)
    r = np.random.default_rng(7).standard_normal(wl.n)
    ref = np.linalg.solve(A, r)
    assert np.linalg.norm(P.apply(r) - ref) / np.linalg.norm(ref) < 1e-10


def test_rasm_partition_property_and_index_sets():
    wl = W.make_lattice(30, jitter_frac=0.1, seed=1)
    P = O.Rasm(wl.xy, wl.sigma, wl.rc, wl.box, wl.cell, 1)
    cx, cy, ncx, ncy = _cells(wl.xy, wl.box, wl.cell)
    rng = np.random.default_rng(2)
    r = rng.standard_normal(wl.n)
    z = P.apply(r)
    nonempty = [c for c in range(ncx * ncy) if np.any((cx == c % ncx) & (cy == c // ncx))]
    assert P.nsub == len(nonempty)
    for s in (0, 7, P.nsub - 1):
        c = nonempty[s]
        ov, own_pos = P.subdomain(s)
        # R_c: 3x3 block row-major, ascending caller index within each cell
        expect = []
        for by in range(c // ncx - 1, c // ncx + 2):
            for bx in range(c % ncx - 1, c % ncx + 2):
                if 0 <= bx < ncx and 0 <= by < ncy:
                    expect += list(np.nonzero((cx == bx) & (cy == by))[0])
        assert list(ov) == expect
        own = ov[own_pos]
        assert set(own.tolist()) == set(np.nonzero((cx == c % ncx) & (cy == c // ncx))[0].tolist())
        # z on own(c) depends only on r on Omega_c: perturb the rest
        r2 = r + rng.standard_normal(wl.n)
        r2[ov] = r[ov]
        z2 = P.apply(r2)
        assert np.array_equal(z[own], z2[own])
    P.close()


# ----------------------------------------------------------------- box overlap (Q24)

@pytest.mark.parametrize("wl,frac", [(W.make_lattice(14, jitter_frac=0.1, seed=3), 0.45),
                                     (W.make_lattice(16, jitter_frac=0.3, seed=4), 0.25),
                                     (W.make_lattice(13), 0.45)])
def test_rasm_box_overlap_equals_explicit_eq11(wl, frac):
    """The paper's D = (1 + 2 frac) B overlap box (D = 1.9 B at frac 0.45)."""
    d = frac * wl.cell
    Minv, _ = _explicit_minv(wl.xy, wl.sigma, wl.rc, wl.box, wl.cell, 1, overlap_width=d)
    P = O.Rasm(wl.xy, wl.sigma, wl.rc, wl.box, wl.cell, 1, overlap_width=d)
    r = np.random.default_rng(9).standard_normal(wl.n)
    ref = Minv @ r
    assert np.linalg.norm(P.apply(r) - ref) / np.linalg.norm(ref) < 1e-10
    P.close()


def test_rasm_box_overlap_index_sets_and_limits():
    wl = W.make_lattice(30, jitter_frac=0.2, seed=6)
    cx, cy, ncx, ncy = _cells(wl.xy, wl.box, wl.cell)
    d = 0.45 * wl.cell
    P = O.Rasm(wl.xy, wl.sigma, wl.rc, wl.box, wl.cell, 1, overlap_width=d)
    Pr = O.Rasm(wl.xy, wl.sigma, wl.rc, wl.box, wl.cell, 1)
    nonempty = [c for c in range(ncx * ncy) if np.any((cx == c % ncx) & (cy == c // ncx))]
    for s in (0, 5, 17, P.nsub - 1):
        c = nonempty[s]
        ov, own_pos = P.subdomain(s)
        ovr, _ = Pr.subdomain(s)
        # brute force over ALL points: inside the grown box (closed) or in the cell
        lx, ly = wl.box[0] + float(c % ncx) * wl.cell, wl.box[1] + float(c // ncx) * wl.cell
        hx, hy = wl.box[0] + float(c % ncx + 1) * wl.cell, wl.box[1] + float(c // ncx + 1) * wl.cell
        x, y = wl.xy[:, 0], wl.xy[:, 1]
        mine = (cx == c % ncx) & (cy == c // ncx)
        inside = mine | ((x >= lx - d) & (x <= hx + d) & (y >= ly - d) & (y <= hy + d))
        assert set(ov.tolist()) == set(np.nonzero(inside)[0].tolist())
        # block order preserved: the box set is the one-ring set filtered
        assert list(ov) == [j for j in ovr if inside[j]]
        assert set(ov[own_pos].tolist()) == set(np.nonzero(mine)[0].tolist())
    # a box wider than the block keeps the whole block: the one-ring preconditioner
    Pw = O.Rasm(wl.xy, wl.sigma, wl.rc, wl.box, wl.cell, 1, overlap_width=10 * wl.cell)
    r = np.random.default_rng(1).standard_normal(wl.n)
    assert np.array_equal(Pw.apply(r), Pr.apply(r))
    P.close(), Pr.close(), Pw.close()


def test_solve_box_overlap_vs_dense(cfg1_solution):
    wl, res, lam = cfg1_solution
    r = O.solve(wl.xy, wl.f, wl.sigma, wl.rc, wl.box, wl.cell, rtol=wl.tol,
                overlap_width=0.45 * wl.cell)
    assert r.converged and np.linalg.norm(r.x - lam) / np.linalg.norm(lam) < 1e-8
    assert r.iterations > res.iterations  # a smaller overlap converges more slowly


def test_dense_factor_examples_and_lu_fallback():
    x, lu = O.dense_factor_solve(np.diag([2.0, 3.0]), np.array([2.0, 3.0]))
    assert not lu and np.allclose(x, [1.0, 1.0], rtol=0, atol=1e-15)
    x, lu = O.dense_factor_solve(np.eye(3), np.array([1.0, -2.0, 5.0]))
    assert np.array_equal(x, [1.0, -2.0, 5.0])
    # symmetric indefinite -> Cholesky breaks down -> LU with partial pivoting
    A = np.array([[1.0, 2.0, 0.0], [2.0, 1.0, 1.0], [0.0, 1.0, 3.0]])
    b = np.array([1.0, 0.0, -1.0])
    x, lu = O.dense_factor_solve(A, b)
    assert lu and np.allclose(A @ x, b, rtol=0, atol=1e-14)
    rng = np.random.default_rng(3)
    G = rng.standard_normal((20, 20))
    A = G @ G.T + 20 * np.eye(20)
    b = rng.standard_normal(20)
    x, lu = O.dense_factor_solve(A, b)
    assert not lu and np.linalg.norm(A @ x - b) / np.linalg.norm(b) < 1e-12
    with pytest.raises(ArithmeticError):
        O.dense_factor_solve(np.zeros((2, 2)), np.ones(2))


# ----------------------------------------------------------------- GMRES (Q12)

def test_gmres_identity_one_iteration():
    b = np.random.default_rng(0).standard_normal(40)
    res = O.gmres(O.op_identity(40), O.op_identity(40), b)
    assert res.iterations == 1 and res.converged
    assert np.allclose(res.x, b, rtol=1e-15, atol=0)


def test_gmres_zero_rhs():
    res = O.gmres(O.op_identity(10), O.op_identity(10), np.zeros(10))
    assert res.iterations == 0 and res.converged and np.all(res.x == 0)


def test_gmres_spd_vs_dense_and_invariants():
    rng = np.random.default_rng(1)
    G = rng.standard_normal((50, 50))
    A = G @ G.T + 5 * np.eye(50)
    b = rng.standard_normal(50)
    res = O.gmres(O.op_dense(A), O.op_identity(50), b, restart=60, rtol=1e-14)
    ref = np.linalg.solve(A, b)
    assert res.converged
    assert np.linalg.norm(res.x - ref) / np.linalg.norm(ref) < 1e-10
    # recurrence residual non-increasing inside a cycle
    assert np.all(np.diff(res.history) <= 1e-15)
    # restarted run: orthonormal Krylov basis of the last cycle
    res = O.gmres(O.op_dense(A), O.op_identity(50), b, restart=12, rtol=1e-12, keep_basis=True)
    V = res.basis
    G2 = V @ V.T
    assert np.max(np.abs(G2 - np.eye(V.shape[0]))) < 1e-8
    assert res.restarts >= 1 and res.converged
    assert np.linalg.norm(A @ res.x - b) / np.linalg.norm(b) < 1e-9


def test_gmres_exact_inverse_pc_two_iterations():
    # Q19: with M = A^-1, M^-1 A = I up to eps*kappa -> <= 2 iterations
    rng = np.random.default_rng(2)
    G = rng.standard_normal((30, 30))
    A = G @ G.T + np.eye(30)
    res = O.gmres(O.op_dense(A), O.op_dense(np.linalg.inv(A)), rng.standard_normal(30), rtol=1e-13)
    assert res.converged and res.iterations <= 2


def test_gmres_not_converged_status():
    rng = np.random.default_rng(3)
    A = np.diag(np.linspace(1.0, 1e4, 200))
    res = O.gmres(O.op_dense(A), O.op_identity(200), rng.standard_normal(200), restart=5,
                  max_iters=7, rtol=1e-14)
    assert not res.converged and res.status == O.ORC_NOT_CONVERGED and res.iterations == 7


# ----------------------------------------------------------------- CGS2 (reading Q23)

def _krylov_qr(A, b, k):
    """Orthonormal basis of span{b, Ab, ..., A^k b} by Householder QR (LAPACK), signs
    fixed so R has a positive diagonal -- the Arnoldi basis (h_{j+1,j} > 0)."""
    K = np.empty((len(b), k + 1))
    K[:, 0] = b / np.linalg.norm(b)
    for j in range(k):
        K[:, j + 1] = A @ K[:, j]
        K[:, j + 1] /= np.linalg.norm(K[:, j + 1])
    Q, R = np.linalg.qr(K)
    return (Q * np.sign(np.diag(R))).T


@pytest.mark.parametrize("orth", ["mgs", "cgs2", "dcgs2"])
def test_gmres_basis_is_the_krylov_qr(orth):
    # implicit-Q theorem: any exact Arnoldi process yields the QR factor of the Krylov
    # matrix; a dropped pass, wrong sign or wrong coefficient breaks the match
    rng = np.random.default_rng(5)
    G = rng.standard_normal((60, 60))
    A = G @ G.T / 60 + np.eye(60)
    b = rng.standard_normal(60)
    res = O.gmres(O.op_dense(A), O.op_identity(60), b, restart=6, max_iters=6, rtol=0.0,
                  keep_basis=True, orth=orth)
    assert res.basis.shape == (7, 60)
    assert np.max(np.abs(res.basis - _krylov_qr(A, b, 6))) < 1e-9


@pytest.mark.parametrize("orth", ["cgs2", "dcgs2"])
def test_gmres_cgs2_same_solution_and_history_as_mgs(orth):
    rng = np.random.default_rng(6)
    G = rng.standard_normal((80, 80))
    A = G @ G.T + 2 * np.eye(80)
    b = rng.standard_normal(80)
    r1 = O.gmres(O.op_dense(A), O.op_identity(80), b, restart=15, rtol=1e-13)
    r2 = O.gmres(O.op_dense(A), O.op_identity(80), b, restart=15, rtol=1e-13, orth=orth)
    assert r1.converged and r2.converged
    assert abs(r1.iterations - r2.iterations) <= 1
    ref = np.linalg.solve(A, b)
    assert np.linalg.norm(r2.x - ref) / np.linalg.norm(ref) < 1e-10
    k = min(r1.iterations, r2.iterations)
    big = r1.history[:k] > 1e-9
    assert np.allclose(r1.history[:k][big], r2.history[:k][big], rtol=1e-6)


@pytest.mark.parametrize("orth", ["cgs2", "dcgs2"])
def test_gmres_cgs2_orthogonal_where_one_pass_is_not(orth):
    # "twice is enough": on an ill-conditioned Krylov sequence CGS2 (and its delayed
    # one-reduction form, reading Q27) keeps ||I - V V^T|| at rounding level; MGS loses
    # orthogonality in proportion to the condition of the Krylov basis
    n = 120
    A = np.diag(np.logspace(0, 10, n))
    b = np.ones(n)
    res = O.gmres(O.op_dense(A), O.op_identity(n), b, restart=40, max_iters=40, rtol=0.0,
                  keep_basis=True, orth=orth)
    V = res.basis
    loss2 = np.max(np.abs(V @ V.T - np.eye(V.shape[0])))
    assert loss2 < 1e-13
    res = O.gmres(O.op_dense(A), O.op_identity(n), b, restart=40, max_iters=40, rtol=0.0,
                  keep_basis=True, orth="mgs")
    V = res.basis
    assert np.max(np.abs(V @ V.T - np.eye(V.shape[0]))) > 100 * loss2  # the contrast (eps kappa)


@pytest.mark.parametrize("orth", ["cgs2", "dcgs2"])
def test_cfg1_solve_cgs2_matches_mgs(cfg1_solution, orth):
    wl, res, lam = cfg1_solution
    r2 = O.solve(wl.xy, wl.f, wl.sigma, wl.rc, wl.box, wl.cell, rtol=wl.tol, orth=orth)
    assert r2.converged and abs(r2.iterations - res.iterations) <= 1
    assert np.linalg.norm(r2.x - lam) / np.linalg.norm(lam) < 1e-8


# ----------------------------------------------------------------- full solve

@pytest.fixture(scope="module")
def cfg1_solution():
    wl = W.config(1)
    res = O.solve(wl.xy, wl.f, wl.sigma, wl.rc, wl.box, wl.cell, rtol=wl.tol)
    lam = O.dense_solve(wl.xy, wl.f, wl.sigma, wl.rc)
    return wl, res, lam


def test_cfg1_solve_vs_dense_direct(cfg1_solution):
    wl, res, lam = cfg1_solution
    assert res.converged
    assert abs(res.iterations - GOLD["cfg1_iterations_model"]) <= 2
    assert np.linalg.norm(res.x - lam) / np.linalg.norm(lam) < 1e-9  # [D3]: 1.6e-10
    assert res.resid_true < 1e-10
    # interpolation conditions at the data (Eq.(2))
    s = O.matvec_brute(wl.xy, res.x, wl.sigma, wl.rc)
    assert np.linalg.norm(s - wl.f) / np.linalg.norm(wl.f) < 1e-10


def test_cfg1_deconvolution_closed_form(cfg1_solution):
    # G_sigma * G_tau = G_s (tau^2 = s^2 - sigma^2): lambda_j ~ h^2 G_tau(x_j) / (1 + alpha - t)
    wl, res, lam = cfg1_solution
    h, s2 = wl.meta["h"], wl.meta["s2"]
    tau2 = s2 - wl.sigma ** 2
    r2 = np.sum(wl.xy ** 2, axis=1)
    closed = h * h * np.exp(-r2 / (2 * tau2)) / (2 * math.pi * tau2)
    closed /= 1.0 + GOLD["alias_alpha"] - GOLD["tail_t"]
    inner = np.max(np.abs(wl.xy), axis=1) <= 0.4
    dev = np.max(np.abs(res.x[inner] - closed[inner])) / np.max(np.abs(res.x))
    assert dev < 3 * GOLD["cfg1_closed_form_dev_x04"]


def test_mesh_independent_iterations():
    # the iteration count does not change with N at fixed ratios
    its = []
    for n in (40, 80):
        wl = W.make_lattice(n, rhs="gauss", s2=0.05)
        res = O.solve(wl.xy, wl.f, wl.sigma, wl.rc, wl.box, wl.cell, rtol=1e-13)
        assert res.converged
        its.append(res.iterations)
    assert abs(its[0] - its[1]) <= 3


@pytest.mark.parametrize("case", ["lattice0.8_tau3", "paper1.0_tau2", "paper0.9_tau2_scattered"])
def test_solve_tbox_vs_dense(case):
    # The paper's T-box matvec (reading Q25; T = B + 6 sigma at h/sigma = 0.8,
    # B + 4 sigma at h/sigma >= 0.9): GMRES + RASM on A_T lambda = f reaches
    # the LAPACK solution of the dense (non-symmetric) A_T.
    if case == "lattice0.8_tau3":
        wl = W.make_lattice(26, jitter_frac=0.1, seed=2, s2=0.05)
        tau = 3.0 * wl.sigma
    elif case == "paper1.0_tau2":
        wl = W.make_paper_lattice(27, 1.0, b_over_sigma=5.0, d_over_b=1.9)
        tau = 2.0 * wl.sigma
    else:
        wl = W.make_paper_lattice(25, 0.9, scatter_seed=7, b_over_sigma=6.0, d_over_b=1.9)
        tau = 3.0 * wl.sigma
    n = wl.n
    A = np.stack([O.matvec_tbox(wl.xy, np.eye(n)[j], wl.sigma, wl.box, wl.cell, tau)
                  for j in range(n)], 1)
    lam = np.linalg.solve(A, wl.f)
    r = O.solve(wl.xy, wl.f, wl.sigma, wl.rc, wl.box, wl.cell, rings=wl.rings, rtol=1e-13,
                overlap_width=wl.overlap_width, trunc_width=tau)
    assert r.converged
    assert np.linalg.norm(r.x - lam) / np.linalg.norm(lam) < 1e-8
    assert np.linalg.norm(wl.f - A @ r.x) / np.linalg.norm(wl.f) < 1e-10
    assert r.resid_true < 1e-10


def test_tbox_too_small_at_h_sigma_08_stalls():
    # The paper's reason for T = B + 6 sigma at h/sigma = 0.8: with
    # T = B + 4 sigma the truncated matrix has an eigenvalue of negative real part
    # on this lattice and preconditioned GMRES stalls.
    wl = W.make_lattice(26, jitter_frac=0.1, seed=2, s2=0.05)
    tau = 2.0 * wl.sigma
    n = wl.n
    A = np.stack([O.matvec_tbox(wl.xy, np.eye(n)[j], wl.sigma, wl.box, wl.cell, tau)
                  for j in range(n)], 1)
    assert np.linalg.eigvals(A).real.min() < 0.0
    r = O.solve(wl.xy, wl.f, wl.sigma, wl.rc, wl.box, wl.cell, rtol=1e-13, max_iters=200,
                trunc_width=tau)
    assert not r.converged


def test_solve_asm_same_weights_as_rasm(cfg1_solution):
    # Eq.(8) ASM and Eq.(11) RASM precondition the same system A_rc lambda = f (reading Q26)
    wl, res, lam = cfg1_solution
    r = O.solve(wl.xy, wl.f, wl.sigma, wl.rc, wl.box, wl.cell, rtol=wl.tol, schwarz="asm")
    assert r.converged and r.resid_true < 1e-10
    assert np.linalg.norm(r.x - lam) / np.linalg.norm(lam) < 1e-8


def test_gmres_dcgs2_restarts_breakdown_and_limits():
    # restarts: the same iterates as MGS across cycles (jittered lattice, GMRES(10))
    wl = W.make_lattice(40, jitter_frac=0.1, seed=5)
    r1 = O.solve(wl.xy, wl.f, wl.sigma, wl.rc, wl.box, wl.cell, restart=10, rtol=1e-13)
    r3 = O.solve(wl.xy, wl.f, wl.sigma, wl.rc, wl.box, wl.cell, restart=10, rtol=1e-13, orth="dcgs2")
    assert r1.converged and r3.converged and r1.restarts >= 2
    assert abs(r1.iterations - r3.iterations) <= 2 and r3.restarts == r1.restarts
    assert np.linalg.norm(r3.x - r1.x) / np.linalg.norm(r1.x) < 1e-8
    # happy breakdown: b in a 3-dimensional invariant subspace -> 3 iterations
    A = np.diag([1.0, 2.0, 3.0] + [5.0] * 17)
    b = np.zeros(20)
    b[:3] = 1.0
    r = O.gmres(O.op_dense(A), O.op_identity(20), b, restart=10, rtol=0.0, orth="dcgs2")
    assert r.converged and r.iterations == 3
    assert np.allclose(r.x[:3], [1.0, 0.5, 1.0 / 3.0], rtol=1e-12) and not r.x[3:].any()
    # max_iters and the identity operator
    r = O.gmres(O.op_identity(5), O.op_identity(5), np.arange(1.0, 6.0), orth="dcgs2")
    assert r.converged and r.iterations == 1


@pytest.mark.parametrize("orth", ["mgs", "cgs2", "dcgs2"])
def test_gmres_history_is_the_minimal_residual(orth):
    """GMRES's definition (Saad & Schultz): after k steps the iterate minimises ||b - A x||
    over the Krylov space K_k(A, b) (identity preconditioner, x0 = 0).  The residual
    estimates of every orthogonalisation -- including the delayed one-reduction form,
    whose recurrences the GPU restates (reading Q27) -- must equal the least-squares
    minimum computed independently by numpy over an explicit Krylov basis."""
    rng = np.random.default_rng(9)
    n, k = 50, 8
    G = rng.standard_normal((n, n))
    A = G @ G.T / n + np.eye(n)  # SPD, well conditioned: the Krylov basis stays accurate
    b = rng.standard_normal(n)
    res = O.gmres(O.op_dense(A), O.op_identity(n), b, restart=30, max_iters=k, rtol=0.0, orth=orth)
    assert len(res.history) == k
    Q = _krylov_qr(A, b, k).T  # n x (k + 1) orthonormal basis of K_{k+1}
    for j in range(1, k + 1):
        y, *_ = np.linalg.lstsq(A @ Q[:, :j], b, rcond=None)
        rmin = np.linalg.norm(b - A @ Q[:, :j] @ y) / np.linalg.norm(b)
        assert res.history[j - 1] == pytest.approx(rmin, rel=1e-8)
