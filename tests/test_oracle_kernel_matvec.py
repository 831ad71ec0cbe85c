"""Pins for the oracle's kernel entries, cell list and matvec (CPU only).

Each check ties the oracle to something other than itself: SPEC worked
examples, closed forms (Poisson summation of the lattice Gaussian), brute-force
membership scans in numpy, integer lattice counts, and the S:333 tail bound.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle as O
import rbf_workloads as W

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "lattice_constants.json")))


# --------------------------------------------------------------- kernel (Eq.12)

def test_phi_worked_examples():
    # sigma=0.01, r=0 -> 1/(2 pi 1e-4); r = 2 sigma -> phi(0) e^-2
    assert O.phi(0.01, 0.0) == pytest.approx(GOLD["phi_sigma001_r0"], rel=2e-16 * 4)
    assert O.phi(0.01, 4e-4) == pytest.approx(GOLD["phi_sigma001_r2sigma"], rel=1e-11)
    # closed form of the normalisation for other sigma
    for s in (0.3, 1e-3, 7.8125e-4):
        assert O.phi(s, 0.0) == pytest.approx(1.0 / (2.0 * math.pi * s * s), rel=1e-15)


def test_phi_decay_and_cutoff_round_trip():
    s = 0.025
    vals = [O.phi(s, (k * 0.1 * s) ** 2) for k in range(80)]
    assert all(a > b for a, b in zip(vals, vals[1:]))
    for t in (math.exp(-2.0), math.exp(-8.0), 1e-6, 0.5):
        r = O.cutoff_radius(s, t)
        assert O.phi(s, r * r) / O.phi(s, 0.0) == pytest.approx(t, rel=1e-12)
    assert O.cutoff_radius(s, math.exp(-2.0)) == pytest.approx(2 * s, rel=1e-14)
    assert O.cutoff_radius(s, math.exp(-8.0)) == pytest.approx(4 * s, rel=1e-14)


def test_gaussian_integrates_to_one():
    # Riemann sum of phi on a fine lattice (h = sigma/3) = 1 up to the Poisson alias
    s = 1.0
    h = s / 3.0
    m = np.arange(-60, 61) * h
    X, Y = np.meshgrid(m, m)
    total = sum(O.phi(s, float(r2)) for r2 in (X * X + Y * Y).ravel()[::1]) * h * h
    assert total == pytest.approx(1.0, abs=1e-13)


# ----------------------------------------------------------------- cell list

def _brute_cells(xy, box, cell):
    ncx, ncy = O.grid_dims(box, cell)
    cx = np.clip(np.floor((xy[:, 0] - box[0]) / cell), 0, ncx - 1).astype(np.int64)
    cy = np.clip(np.floor((xy[:, 1] - box[1]) / cell), 0, ncy - 1).astype(np.int64)
    return cy * ncx + cx, ncx, ncy


@pytest.mark.parametrize("wl", [W.make_lattice(24), W.make_lattice(40, jitter_frac=0.1, seed=7),
                                W.make_clustered(3000, seed=11)])
def test_cell_list_partition_and_membership(wl):
    key, perm, start = O.cell_list(wl.xy, wl.box, wl.cell)
    bkey, ncx, ncy = _brute_cells(wl.xy, wl.box, wl.cell)
    assert np.array_equal(key, bkey)
    assert start[0] == 0 and start[-1] == wl.n and np.all(np.diff(start) >= 0)
    assert np.array_equal(np.sort(perm), np.arange(wl.n))  # partition: each point once
    for c in range(ncx * ncy):
        members = perm[start[c]:start[c + 1]]
        assert np.all(bkey[members] == c)
        assert np.all(np.diff(members) > 0)  # stable: ascending caller index


def test_cell_counts_cfg1_and_ragged():
    wl = W.config(1)
    _, _, start = O.cell_list(wl.xy, wl.box, wl.cell)
    assert O.grid_dims(wl.box, wl.cell) == (20, 20)
    assert np.all(np.diff(start) == 25)
    # 24x24 lattice: 24/5 = 4.8 -> 5 cells per axis, last column 4 points wide
    wl = W.make_lattice(24)
    _, _, start = O.cell_list(wl.xy, wl.box, wl.cell)
    cnt = np.diff(start).reshape(5, 5)
    assert cnt[0, 0] == 25 and cnt[0, 4] == 20 and cnt[4, 0] == 20 and cnt[4, 4] == 16


# ----------------------------------------------------------------- matvec

def _theta2(h, s):
    """Poisson summation: h^2 sum_{m in Z^2} G_s(mh) = (sum_k exp(-2 pi^2 s^2 k^2/h^2))^2."""
    th = 1.0 + 2.0 * sum(math.exp(-2.0 * math.pi ** 2 * s * s * k * k / (h * h)) for k in range(1, 6))
    return th * th


def test_constant_field_exact_and_cutoff():
    wl = W.config(1)
    h = wl.meta["h"]
    centre = [50 * 100 + 50, 45 * 100 + 55, 60 * 100 + 40]  # >= 0.8 from the edge (32 sigma)
    ones = np.ones(wl.n)
    y_ex = O.matvec_brute(wl.xy, ones, wl.sigma, None, rows=centre)
    y_ct = O.matvec_brute(wl.xy, ones, wl.sigma, wl.rc, rows=centre)
    alpha = _theta2(h, wl.sigma) - 1.0
    assert alpha == pytest.approx(GOLD["alias_alpha"], rel=1e-6)  # two independent derivations
    for v in h * h * y_ex:
        assert v - 1.0 == pytest.approx(alpha, abs=2e-15)
    for v in h * h * y_ct:
        assert v - 1.0 == pytest.approx(alpha - GOLD["tail_t"], abs=2e-15)


def test_pairs_per_point_lattice():
    wl = W.config(1)
    assert O.count_pairs(wl.xy, wl.rc, wl.box, wl.cell) == GOLD["cfg1_pairs"]
    m = np.arange(-10, 11)
    M1, M2 = np.meshgrid(m, m)
    assert int(np.sum(M1 ** 2 + M2 ** 2 < 56.25)) == GOLD["interior_pairs_per_point"]
    # exact count for an n x n lattice: sum over offsets m with |m|^2 < 56.25 of
    # (n - |m1|)(n - |m2|) ordered pairs; pairs per point -> 177 as n grows (O(N))
    inside = (M1 ** 2 + M2 ** 2) < 56.25
    for n in (100, 200):
        wl2 = W.make_lattice(n)
        expect = int(np.sum(((n - np.abs(M1)) * (n - np.abs(M2)))[inside]))
        assert O.count_pairs(wl2.xy, wl2.rc, wl2.box, wl2.cell) == expect


def test_unit_vector_column():
    # x = e_j -> y_i = phi(|x_i - x_j|^2) inside the cutoff, exactly 0 outside
    wl = W.make_lattice(30, jitter_frac=0.1, seed=3)
    j = 437
    e = np.zeros(wl.n)
    e[j] = 1.0
    y = O.matvec_brute(wl.xy, e, wl.sigma, wl.rc)
    d = wl.xy - wl.xy[j]
    r2 = d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]
    inside = r2 < wl.rc ** 2
    assert np.all(y[~inside] == 0.0)
    expect = np.exp(-r2[inside] / (2 * wl.sigma ** 2)) / (2 * math.pi * wl.sigma ** 2)
    assert np.allclose(y[inside], expect, rtol=1e-14, atol=0)


@pytest.mark.parametrize("wl", [W.make_lattice(33, jitter_frac=0.1, seed=5),
                                W.make_clustered(2500, seed=9)])
def test_cells_matches_brute_symmetry_linearity(wl):
    rng = np.random.default_rng(0)
    u, w = rng.standard_normal(wl.n), rng.standard_normal(wl.n)
    yb = O.matvec_brute(wl.xy, w, wl.sigma, wl.rc)
    yc = O.matvec_cells(wl.xy, w, wl.sigma, wl.rc, wl.box, wl.cell)
    assert np.linalg.norm(yb - yc) / np.linalg.norm(yb) < 1e-14
    Au = O.matvec_brute(wl.xy, u, wl.sigma, wl.rc)
    assert np.dot(u, yb) == pytest.approx(np.dot(Au, w), rel=1e-12)
    ylin = O.matvec_brute(wl.xy, 2.0 * u - 3.0 * w, wl.sigma, wl.rc)
    assert np.linalg.norm(ylin - (2.0 * Au - 3.0 * yb)) / np.linalg.norm(ylin) < 1e-13
    assert np.all(O.matvec_brute(wl.xy, np.zeros(wl.n), wl.sigma, wl.rc) == 0.0)


def test_truncation_tail_bound():
    # |y_exact - y_cut|_i <= ||w||_inf * neglected_row_mass(i)
    wl = W.make_clustered(1500, seed=4)
    rng = np.random.default_rng(1)
    w = rng.uniform(-1, 1, wl.n)
    rows = np.arange(wl.n)
    ye = O.matvec_brute(wl.xy, w, wl.sigma, None)
    yc = O.matvec_brute(wl.xy, w, wl.sigma, wl.rc)
    mass = O.neglected_row_mass(wl.xy, wl.sigma, wl.rc, rows)
    assert np.all(np.abs(ye - yc) <= np.max(np.abs(w)) * mass * (1 + 1e-12) + 1e-300)
    # and the mass is below the continuum tail exp(-rc^2/2sigma^2) times the point density bound
    assert np.all(mass >= 0.0)


def test_dense_assembly_symmetric_spd():
    wl = W.make_lattice(12, jitter_frac=0.1, seed=1)
    A = O.assemble_dense(wl.xy, wl.sigma, wl.rc)
    assert np.array_equal(A, A.T)
    np.linalg.cholesky(A)
    Ae = O.assemble_dense(wl.xy, wl.sigma, None)
    assert np.array_equal(Ae, Ae.T)
    assert np.all(Ae >= A)


# ------------------------------------------------------------------ interpolant evaluation (§8.f1)

def _theta_shift(h, s, d):
    """h sum_m G_s,1D(mh - d) = 1 + 2 sum_k exp(-2 pi^2 s^2 k^2 / h^2) cos(2 pi k d / h)
    (Poisson summation of a 1-D normalised Gaussian sampled on a shifted lattice)."""
    return 1.0 + 2.0 * sum(math.exp(-2.0 * math.pi ** 2 * s * s * k * k / (h * h)) *
                           math.cos(2.0 * math.pi * k * d / h) for k in range(1, 8))


def test_evaluate_at_data_points_is_matvec_row():
    wl = W.make_lattice(30, jitter_frac=0.2, seed=4)
    lam = np.random.default_rng(5).standard_normal(wl.n)
    rows = np.array([0, 17, 450, wl.n - 1])
    s = O.evaluate(wl.xy[rows], wl.xy, lam, wl.sigma, wl.rc)
    assert np.array_equal(s, O.matvec_brute(wl.xy, lam, wl.sigma, wl.rc, rows=rows))
    s_ex = O.evaluate(wl.xy[rows], wl.xy, lam, wl.sigma, None)
    assert np.array_equal(s_ex, O.matvec_brute(wl.xy, lam, wl.sigma, None, rows=rows))


def test_evaluate_constant_weights_poisson_off_lattice():
    """lambda_j = h^2 on the cfg1 lattice: s(q) = theta(dx) theta(dy) (exact sum) at
    interior queries off the lattice, the truncated sum below it by at most the tail."""
    wl = W.config(1)
    h = wl.meta["h"]
    lam = np.full(wl.n, h * h)
    rng = np.random.default_rng(6)
    q = rng.uniform(-0.3, 0.3, size=(40, 2))
    s_ex = O.evaluate(q, wl.xy, lam, wl.sigma, None)
    s_ct = O.evaluate(q, wl.xy, lam, wl.sigma, wl.rc)
    # lattice x_i = -1 + (i + 1/2) h: offset of q from the lattice
    d = np.mod(q + 1.0 - 0.5 * h, h)
    expect = np.array([_theta_shift(h, wl.sigma, dx) * _theta_shift(h, wl.sigma, dy) for dx, dy in d])
    assert np.max(np.abs(s_ex - expect)) <= 1e-14  # 10^4-term sum of O(1) values
    gap = s_ex - s_ct
    assert np.all(gap >= 0.0) and np.all(gap <= 3e-8)  # tail e^-18-scale mass


# ------------------------------------------- T-box truncation (reading Q25, §8.f2)
# The paper's matvec rule: row i keeps the sources inside the box T of
# target i's cell, T = B + 2 tau (tau = 2 sigma for h/sigma >= 0.9, 3 sigma at 0.8,
# P:307, 348).

def _tbox_separable(n_side, tau_over_h, ax, by):
    """Closed form on a cell-centred lattice with cell = 5h and separable weights
    w_j = ax[jx] * by[jy]: the box is a product of index intervals, so row i is
    norm * (sum_{jx in Jx} ax[jx] e^{-(ix-jx)^2 h^2/2s^2}) * (same in y), with Jx found
    in exact rational arithmetic from x_j = -1 + (j + 1/2) h and the cell edges
    -1 + 5 cx h (no floating-point membership test)."""
    from fractions import Fraction as F
    q = F(tau_over_h)
    c2 = 0.8 * 0.8 / 2.0  # h^2 / (2 sigma^2) at h/sigma = 0.8
    cells = (n_side + 4) // 5

    def interval(c):
        lo = [j for j in range(n_side) if F(2 * j + 1, 2) >= 5 * c - q]
        hi = [j for j in range(n_side) if F(2 * j + 1, 2) <= 5 * c + 5 + q]
        return range(lo[0], hi[-1] + 1)

    J = [interval(c) for c in range(cells)]
    sx = np.array([sum(ax[j] * math.exp(-c2 * (i - j) ** 2) for j in J[i // 5]) for i in range(n_side)])
    sy = np.array([sum(by[j] * math.exp(-c2 * (i - j) ** 2) for j in J[i // 5]) for i in range(n_side)])
    return np.outer(sy, sx).ravel()  # index iy * n + ix


@pytest.mark.parametrize("n_side,tau_over_h", [(62, "15/4"), (62, "2"), (40, "6/5")])
def test_tbox_separable_closed_form(n_side, tau_over_h):
    from fractions import Fraction as F
    wl = W.make_lattice(n_side)
    h = wl.meta["h"]
    rng = np.random.default_rng(25)
    ax, by = rng.uniform(0.5, 1.5, n_side), rng.uniform(-1.0, 1.0, n_side)
    w = np.outer(by, ax).ravel()
    tau = float(F(tau_over_h)) * h
    y = O.matvec_tbox(wl.xy, w, wl.sigma, wl.box, wl.cell, tau)
    ref = _tbox_separable(n_side, tau_over_h, ax, by) / (2.0 * math.pi * wl.sigma ** 2)
    assert np.abs(y - ref).max() <= 1e-13 * np.abs(ref).max()


def test_tbox_covering_everything_is_the_exact_operator():
    wl = W.make_lattice(24, jitter_frac=0.1, seed=2)
    w = np.random.default_rng(3).standard_normal(wl.n)
    y = O.matvec_tbox(wl.xy, w, wl.sigma, wl.box, wl.cell, 2.5)
    ref = O.matvec_brute(wl.xy, w, wl.sigma, None)
    assert np.abs(y - ref).max() <= 1e-14 * np.abs(ref).max()


@pytest.mark.parametrize("kind", ["jitter", "clustered"])
def test_tbox_pattern_and_cells_form(kind):
    wl = (W.make_lattice(21, jitter_frac=0.1, seed=4) if kind == "jitter"
          else W.make_clustered(500, seed=5))
    n, box, c = wl.n, wl.box, wl.cell
    for tau in (2 * wl.sigma, 3 * wl.sigma, c, 2 * c):
        # the dense matrix column by column vs a numpy membership scan
        A = np.stack([O.matvec_tbox(wl.xy, np.eye(n)[j], wl.sigma, box, c, tau) for j in range(n)], 1)
        key, _, _ = O.cell_list(wl.xy, box, c)
        ncx, _ = O.grid_dims(box, c)
        cx, cy = key % ncx, key // ncx
        lx, ly = box[0] + cx * c, box[1] + cy * c
        hx, hy = box[0] + (cx + 1) * c, box[1] + (cy + 1) * c
        X, Y = wl.xy[:, 0][None, :], wl.xy[:, 1][None, :]
        M = ((X >= (lx - tau)[:, None]) & (X <= (hx + tau)[:, None]) &
             (Y >= (ly - tau)[:, None]) & (Y <= (hy + tau)[:, None]))
        assert np.array_equal(A != 0.0, M)
        d2 = ((wl.xy[:, None, :] - wl.xy[None, :, :]) ** 2).sum(-1)
        ref = np.exp(-d2 / (2 * wl.sigma ** 2)) / (2 * math.pi * wl.sigma ** 2)
        assert np.allclose(A[M], ref[M], rtol=1e-13, atol=0)
        if tau < c:
            assert not np.array_equal(M, M.T)  # one box per target cell: not symmetric
        w = np.random.default_rng(6).standard_normal(n)
        y1 = O.matvec_tbox(wl.xy, w, wl.sigma, box, c, tau)
        y2 = O.matvec_tbox(wl.xy, w, wl.sigma, box, c, tau, cells=True)
        assert np.abs(y1 - y2).max() <= 1e-14 * np.abs(y1).max()
        rows = np.array([0, n // 3, n - 1])
        assert np.array_equal(O.matvec_tbox(wl.xy, w, wl.sigma, box, c, tau, rows=rows), y1[rows])


def test_tbox_evaluate_at_data_points_is_matvec_row():
    wl = W.make_lattice(20, jitter_frac=0.1, seed=9)
    lam = np.random.default_rng(10).standard_normal(wl.n)
    tau = 3 * wl.sigma
    s = O.evaluate_tbox(wl.xy, wl.xy, lam, wl.sigma, wl.box, wl.cell, tau)
    y = O.matvec_tbox(wl.xy, lam, wl.sigma, wl.box, wl.cell, tau)
    assert np.array_equal(s, y)
    # a query keeps the sources of ITS cell's box: two queries in one cell see one set
    q = np.array([[wl.box[0] + 0.2 * wl.cell, wl.box[1] + 0.3 * wl.cell],
                  [wl.box[0] + 0.9 * wl.cell, wl.box[1] + 0.8 * wl.cell]])
    one = np.ones(wl.n)
    big = O.evaluate_tbox(q, wl.xy, one, 1e6, wl.box, wl.cell, tau)  # phi ~ constant
    assert big[0] == pytest.approx(big[1], rel=1e-9)
