"""Seeded synthetic inputs for the PetRBF hot path (shared by oracle tests and
the CUDA path).  This module holds NO arithmetic of the method: it only draws
point sets and right-hand sides.  Recipes restate BASELINE.json configs 1-5
(BJ:7-11) with the readings Q3, Q6, Q7, Q8, Q16 of DESIGN.md.

The paper itself measured Franke data on [0,1]^2 lattices;
BASELINE.json replaces that by Gaussian right-hand sides on [-1,1]^2 at the
paper's hardest ratio h/sigma = 0.8.  No public dataset is
involved.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

BOX = (-1.0, -1.0, 1.0, 1.0)


@dataclass
class Workload:
    name: str
    xy: np.ndarray          # (N, 2) float64, caller order
    f: np.ndarray           # (N,) float64 right-hand side
    sigma: float
    rc: float
    cell: float
    rings: int = 1
    tol: float = 1e-13
    box: tuple = BOX
    meta: dict = field(default_factory=dict)
    overlap_width: float = 0.0  # box overlap delta (reading Q24); 0 = whole rings

    @property
    def n(self) -> int:
        return int(self.xy.shape[0])


def lattice(n_side: int) -> np.ndarray:
    """Cell-centred n x n lattice over [-1,1]^2 (reading Q3): x_i = -1 + (i + 1/2) h,
    h = 2/n, point index = iy*n + ix (x fastest)."""
    h = 2.0 / n_side
    c = -1.0 + (np.arange(n_side, dtype=np.float64) + 0.5) * h
    X, Y = np.meshgrid(c, c, indexing="xy")
    return np.stack([X.ravel(), Y.ravel()], axis=1).copy()


def jitter(xy: np.ndarray, h: float, frac: float, seed: int) -> np.ndarray:
    """Add independent U[-frac*h, +frac*h] to each coordinate, drawn with
    numpy PCG64(seed) in point-index order (reading Q6)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    d = rng.uniform(-frac * h, frac * h, size=xy.shape)
    return xy + d


def clustered(n: int, seed: int, frac_uniform: float = 0.7, std: float = 0.1) -> np.ndarray:
    """round(0.7 N) uniform points in [-1,1]^2, then N - round(0.7 N) points from
    N(0, std^2 I) rejection-resampled into [-1,1]^2, PCG64(seed) (reading Q8)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    n_u = int(round(frac_uniform * n))
    n_c = n - n_u
    u = rng.uniform(-1.0, 1.0, size=(n_u, 2))
    c = rng.normal(0.0, std, size=(n_c, 2))
    bad = np.any(np.abs(c) > 1.0, axis=1)
    while bad.any():
        c[bad] = rng.normal(0.0, std, size=(int(bad.sum()), 2))
        bad = np.any(np.abs(c) > 1.0, axis=1)
    return np.concatenate([u, c], axis=0)


def gauss_rhs(xy: np.ndarray, s2: float) -> np.ndarray:
    """Unit-mass Gaussian f(x) = exp(-|x|^2/(2 s2)) / (2 pi s2) (reading Q16;
    BJ:7 s2 = 0.05, BJ:8/10/11 s2 = 0.02 'Lamb-Oseen' vorticity)."""
    r2 = xy[:, 0] ** 2 + xy[:, 1] ** 2
    return np.exp(-r2 / (2.0 * s2)) / (2.0 * math.pi * s2)


def blob_params(seed: int):
    """Three signed Gaussian blobs (reading Q7), drawn with PCG64(seed) in the order
    centres (3x2) ~ U[-0.5,0.5], widths (3) ~ U[0.05,0.2], |amplitudes| (3) ~ U[0.5,1],
    signs (3) ~ +-1."""
    rng = np.random.Generator(np.random.PCG64(seed))
    centres = rng.uniform(-0.5, 0.5, size=(3, 2))
    widths = rng.uniform(0.05, 0.2, size=3)
    amps = rng.uniform(0.5, 1.0, size=3)
    signs = np.where(rng.integers(0, 2, size=3) == 1, 1.0, -1.0)
    return centres, widths, amps * signs


def blobs_rhs(xy: np.ndarray, seed: int) -> np.ndarray:
    centres, widths, amps = blob_params(seed)
    f = np.zeros(xy.shape[0])
    for c, s, a in zip(centres, widths, amps):
        r2 = (xy[:, 0] - c[0]) ** 2 + (xy[:, 1] - c[1]) ** 2
        f += a * np.exp(-r2 / (2.0 * s * s))
    return f


def lattice_params(n_side: int):
    """h = 2/n, sigma = h/0.8, rc = 6 sigma, cell = 4 sigma (BJ:7-10)."""
    h = 2.0 / n_side
    sigma = h / 0.8
    return h, sigma, 6.0 * sigma, 4.0 * sigma


def make_lattice(n_side: int, *, jitter_frac: float = 0.0, seed: int | None = None,
                 rhs: str = "gauss", s2: float = 0.02, tol: float = 1e-13,
                 name: str | None = None, rings: int = 1) -> Workload:
    h, sigma, rc, cell = lattice_params(n_side)
    xy = lattice(n_side)
    if jitter_frac > 0.0:
        xy = jitter(xy, h, jitter_frac, seed if seed is not None else 0)
    if rhs == "gauss":
        f = gauss_rhs(xy, s2)
    elif rhs == "blobs":
        f = blobs_rhs(xy, seed if seed is not None else 0)
    elif rhs == "ones":
        f = np.ones(xy.shape[0])
    else:
        raise ValueError(rhs)
    return Workload(name or f"lattice{n_side}", xy, f, sigma, rc, cell, rings, tol,
                    meta=dict(h=h, n_side=n_side, jitter=jitter_frac, seed=seed, rhs=rhs, s2=s2))


def make_clustered(n: int, seed: int, *, s2: float = 0.02, tol: float = 1e-13,
                   name: str | None = None) -> Workload:
    """sigma = 0.8 sqrt(4/N) (reading Q8), rc = 6 sigma, cell = 4 sigma."""
    xy = clustered(n, seed)
    sigma = 0.8 * math.sqrt(4.0 / n)
    return Workload(name or f"clustered{n}", xy, gauss_rhs(xy, s2), sigma, 6.0 * sigma,
                    4.0 * sigma, 1, tol, meta=dict(seed=seed, s2=s2))


def franke(xy: np.ndarray) -> np.ndarray:
    """Franke's test function as printed in PAPER.md Eq.(13) at the points.
    (The paper prints (9y+1)^2/10 in the second term where Franke's 1982 function has
    (9y+1)/10; this follows the paper -- reading Q22 of DESIGN.md.  It is input data
    only, no part of the method.)"""
    x, y = xy[:, 0], xy[:, 1]
    return (0.75 * np.exp(-0.25 * ((9 * x - 2) ** 2 + (9 * y - 2) ** 2))
            + 0.75 * np.exp(-((9 * x + 1) ** 2) / 49.0 - ((9 * y + 1) ** 2) / 10.0)
            + 0.5 * np.exp(-0.25 * ((9 * x - 7) ** 2 + (9 * y - 3) ** 2))
            - 0.2 * np.exp(-((9 * x - 4) ** 2) - (9 * y - 7) ** 2))


def make_paper_lattice(n_side: int, h_over_sigma: float, *, scatter_seed: int | None = None,
                       tol: float = 1e-13, name: str | None = None,
                       b_over_sigma: float | None = None, d_over_b: float | None = None) -> Workload:
    """The paper's test problem: Franke data on an n x n lattice of
    [0,1]^2 that includes the boundary (x_i = i h, h = 1/(n-1); N = (1/h + 1)^2 as in
    the paper, reading Q4), sigma = h / (h/sigma); quasi-scattered variant: every
    coordinate shifted by U[0, h/2), PCG64(scatter_seed).  Subdomain geometry:
    this build's by default (rc = 6 sigma, cell = 4 sigma, one ring; readings Q1, Q9);
    with b_over_sigma / d_over_b the paper's boxes: cell B = b sigma,
    overlap box D = d B (overlap_width (D - B)/2, reading Q24), rc = 6 sigma."""
    h = 1.0 / (n_side - 1)
    sigma = h / h_over_sigma
    c = np.arange(n_side, dtype=np.float64) * h
    X, Y = np.meshgrid(c, c, indexing="xy")
    xy = np.stack([X.ravel(), Y.ravel()], axis=1).copy()
    box = (0.0, 0.0, 1.0, 1.0)
    if scatter_seed is not None:
        rng = np.random.Generator(np.random.PCG64(scatter_seed))
        xy = xy + rng.uniform(0.0, 0.5 * h, size=xy.shape)
        box = (0.0, 0.0, 1.0 + 0.5 * h, 1.0 + 0.5 * h)
    cell, ow, rings = 4.0 * sigma, 0.0, 1
    if b_over_sigma is not None:
        cell = b_over_sigma * sigma
        ow = 0.5 * (d_over_b - 1.0) * cell
        rings = max(1, int(math.ceil(ow / cell - 1e-12)))
    return Workload(name or f"franke{n_side}_{h_over_sigma}", xy, franke(xy), sigma, 6.0 * sigma,
                    cell, rings, tol, box=box,
                    meta=dict(h=h, n_side=n_side, h_over_sigma=h_over_sigma, scatter=scatter_seed,
                              b_over_sigma=b_over_sigma, d_over_b=d_over_b),
                    overlap_width=ow)


def weak(world: int) -> Workload:
    """Weak-scaling version of cfg2: `world` copies of the cfg2 block stacked
    in y -- a 1024 x (1024 world) lattice with the same h, jitter recipe (PCG64(2) in point
    order, so the first 1024^2 points ARE cfg2's) and one unit-mass Gaussian (s^2 = 0.02)
    at the centre of every [-1,1] x [2g-1, 2g+1] block; box [-1,1] x [-1, 2 world - 1].
    Strips balanced by point count give every GPU one cfg2-sized block."""
    n = 1024
    h, sigma, rc, cell = lattice_params(n)
    c = -1.0 + (np.arange(n, dtype=np.float64) + 0.5) * h
    cy = -1.0 + (np.arange(n * world, dtype=np.float64) + 0.5) * h
    X, Y = np.meshgrid(c, cy, indexing="xy")
    xy = jitter(np.stack([X.ravel(), Y.ravel()], axis=1).copy(), h, 0.1, 2)
    f = np.zeros(xy.shape[0])
    for g in range(world):
        f += gauss_rhs(xy - np.array([0.0, 2.0 * g]), 0.02)
    return Workload(f"cfg2-weak{world}", xy, f, sigma, rc, cell, 1, 1e-13,
                    box=(-1.0, -1.0, 1.0, 2.0 * world - 1.0), meta=dict(h=h, world=world))


def config(k: int) -> Workload:
    """BASELINE.json configs[k-1] (BJ:7-11) as seeded synthetic input."""
    if k == 1:
        return make_lattice(100, rhs="gauss", s2=0.05, tol=1e-13, name="cfg1")
    if k == 2:
        return make_lattice(1024, jitter_frac=0.1, seed=2, rhs="gauss", s2=0.02, tol=1e-13,
                            name="cfg2")
    if k == 3:
        return make_lattice(4096, seed=3, rhs="blobs", tol=1e-13, name="cfg3")
    if k == 4:
        return make_lattice(7072, rhs="gauss", s2=0.02, tol=1e-15, name="cfg4")
    if k == 5:
        return make_clustered(4194304, seed=5, tol=1e-13, name="cfg5")
    raise ValueError(k)


CONFIG_DESCRIPTIONS = {
    1: "100x100 cell-centred lattice on [-1,1]^2, h/sigma=0.8, rc=6 sigma, cell=4 sigma, "
       "f=G_s s2=0.05, tol 1e-13",
    2: "1024x1024 lattice + U[+-0.1h] jitter (PCG64(2)), f=G_s s2=0.02, tol 1e-13",
    3: "4096x4096 lattice, 3 seeded Gaussian blobs (PCG64(3)), tol 1e-13",
    4: "7072x7072 lattice (N=50,013,184), f=G_s s2=0.02, tol 1e-15",
    5: "4,194,304 points: 70% U[-1,1]^2 + 30% N(0,0.1^2) (PCG64(5)), sigma=0.8 sqrt(4/N)",
}
