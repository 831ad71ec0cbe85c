"""Oracle for the PetRBF hot path -- TEST INFRASTRUCTURE, NOT THE PRODUCT.

Plain, slow, obviously-correct CPU reference (C in ``rbf_oracle.c`` via ctypes,
plus numpy/scipy for the dense direct solve).  It shares no code with the CUDA
path in ``paper_0909_5413_b200/`` and neither imports the other.  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.

Every function cites the passage of /root/reference/PAPER.md (``P:<line>``) it
follows; the readings Q1..Q20 are listed in DESIGN.md (and SURVEY.md §8.c.2).

Parity status: every function here is pinned by a
``-m "not gpu"`` test in tests/test_oracle_*.py, except ``solve`` on clustered
scattered data (config 5), whose solve is "parity unpinned" (reading Q8).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "rbf_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

ORC_OK, ORC_NOT_CONVERGED, ORC_EINVAL, ORC_ENOMEM, ORC_EFACTOR, ORC_ENUMERIC = 0, 2, -1, -2, -5, -6


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no CUDA).  -ffp-contract=off keeps every
    fused multiply-add explicit (reading Q1)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fPIC", "-shared",
               "-std=c11", "-D_GNU_SOURCE", "-o", _LIB, _SRC, "-lm"]
        subprocess.run(cmd, check=True)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        i64, dbl, ptr = C.c_int64, C.c_double, C.c_void_p
        L.orc_phi.restype = dbl
        L.orc_phi.argtypes = [dbl, dbl]
        L.orc_cutoff_radius.restype = dbl
        L.orc_cutoff_radius.argtypes = [dbl, dbl]
        L.orc_assemble_dense.argtypes = [i64, ptr, dbl, dbl, ptr]
        L.orc_matvec_brute.argtypes = [i64, ptr, ptr, dbl, dbl, C.c_int, i64, ptr, ptr]
        L.orc_neglected_row_mass.argtypes = [i64, ptr, dbl, dbl, i64, ptr, ptr]
        L.orc_evaluate.argtypes = [i64, ptr, i64, ptr, ptr, dbl, dbl, C.c_int, ptr]
        L.orc_evaluate.restype = None
        L.orc_grid_dims.argtypes = [dbl, dbl, dbl, dbl, dbl, ptr, ptr]
        L.orc_cell_list.argtypes = [i64, ptr, dbl, dbl, dbl, dbl, dbl, ptr, ptr, ptr]
        L.orc_matvec_cells.restype = C.c_int
        L.orc_matvec_cells.argtypes = [i64, ptr, ptr, dbl, dbl, dbl, dbl, dbl, dbl, dbl, ptr]
        L.orc_matvec_tbox.argtypes = [i64, ptr, ptr, dbl, dbl, dbl, dbl, dbl, dbl, dbl, i64, ptr,
                                      ptr]
        L.orc_matvec_tbox.restype = None
        L.orc_matvec_tbox_cells.restype = C.c_int
        L.orc_matvec_tbox_cells.argtypes = [i64, ptr, ptr, dbl, dbl, dbl, dbl, dbl, dbl, dbl, ptr]
        L.orc_evaluate_tbox.argtypes = [i64, ptr, i64, ptr, ptr, dbl, dbl, dbl, dbl, dbl, dbl,
                                        dbl, ptr]
        L.orc_evaluate_tbox.restype = None
        L.orc_op_rbf_tbox.argtypes = [ptr, i64, ptr, dbl, dbl, dbl, dbl, dbl, dbl, dbl]
        L.orc_count_pairs.restype = i64
        L.orc_count_pairs.argtypes = [i64, ptr, dbl, dbl, dbl, dbl, dbl, dbl]
        L.orc_dense_factor_solve.restype = C.c_int
        L.orc_dense_factor_solve.argtypes = [i64, ptr, ptr, ptr, ptr]
        L.orc_rasm_setup.restype = ptr
        L.orc_rasm_setup.argtypes = [i64, ptr, dbl, dbl, dbl, dbl, dbl, dbl, dbl, i64]
        L.orc_rasm_setup_box.restype = ptr
        L.orc_rasm_setup_box.argtypes = [i64, ptr, dbl, dbl, dbl, dbl, dbl, dbl, dbl, i64, dbl]
        L.orc_rasm_status.restype = C.c_int
        L.orc_rasm_status.argtypes = [ptr, ptr, ptr, ptr]
        L.orc_rasm_sub_info.argtypes = [ptr, i64, ptr, ptr]
        L.orc_rasm_sub_sets.argtypes = [ptr, i64, ptr, ptr]
        L.orc_rasm_apply.argtypes = [ptr, ptr, ptr, C.c_int]
        L.orc_rasm_free.argtypes = [ptr]
        L.orc_gmres.restype = C.c_int
        L.orc_gmres.argtypes = [ptr, ptr, ptr, i64, i64, dbl, dbl, ptr, ptr, i64, ptr, ptr, ptr]
        L.orc_gmres_orth.restype = C.c_int
        L.orc_gmres_orth.argtypes = [ptr, ptr, ptr, i64, i64, dbl, dbl, C.c_int, ptr, ptr, i64, ptr,
                                     ptr, ptr]
        L.orc_op_identity.argtypes = [ptr, i64]
        L.orc_op_dense.argtypes = [ptr, i64, ptr]
        L.orc_op_rbf.argtypes = [ptr, i64, ptr, dbl, dbl, dbl, dbl, dbl, dbl, dbl, C.c_int]
        L.orc_op_rasm.argtypes = [ptr, ptr, C.c_int]
        L.orc_op_size.restype = i64
        L.orc_report_size.restype = i64
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


# --------------------------------------------------------------------------
# Kernel, Eq.(12)
# --------------------------------------------------------------------------

def phi(sigma: float, r2: float) -> float:
    """Normalised Gaussian entry exp(-r^2/2 sigma^2)/(2 pi sigma^2), Eq.(12) P:244-246."""
    return lib().orc_phi(float(sigma), float(r2))


def cutoff_radius(sigma: float, rel_tol: float) -> float:
    """Radius where exp(-r^2/2sigma^2) = rel_tol."""
    return lib().orc_cutoff_radius(float(sigma), float(rel_tol))


def assemble_dense(xy, sigma: float, rc: float | None) -> np.ndarray:
    """Dense A (rc=None: exact Eq.(4) Phi block) or A_rc (reading Q1)."""
    xy = _f64(xy)
    n = xy.shape[0]
    A = np.empty((n, n), dtype=np.float64)
    lib().orc_assemble_dense(n, _p(xy), float(sigma), -1.0 if rc is None else float(rc), _p(A))
    return A


# --------------------------------------------------------------------------
# Matvec, P:248 and reading Q1
# --------------------------------------------------------------------------

def matvec_brute(xy, w, sigma: float, rc: float | None, rows=None) -> np.ndarray:
    """y_i = sum_j [r2_ij < rc^2] w_j phi(r2_ij), brute force over all j (the
    plain definition).  rc=None: exact (untruncated) product.  rows
    selects a subset of target rows (sampled parity at full sizes)."""
    xy, w = _f64(xy), _f64(w)
    n = xy.shape[0]
    exact = rc is None
    if rows is None:
        y = np.empty(n, dtype=np.float64)
        lib().orc_matvec_brute(n, _p(xy), _p(w), float(sigma), 0.0 if exact else float(rc),
                               int(exact), 0, None, _p(y))
    else:
        rows = _i64(rows)
        y = np.empty(rows.shape[0], dtype=np.float64)
        lib().orc_matvec_brute(n, _p(xy), _p(w), float(sigma), 0.0 if exact else float(rc),
                               int(exact), rows.shape[0], _p(rows), _p(y))
    return y


def evaluate(q, xy, lam, sigma: float, rc: float | None) -> np.ndarray:
    """Interpolant s(q) = sum_j [|q - x_j| < rc] lambda_j phi(|q - x_j|^2) at query
    points q (Eq.(1), Eq.(12)), brute force.  rc=None: the
    untruncated sum.  Pinned by tests/test_oracle_kernel_matvec.py (queries at the
    data points reproduce matvec_brute rows; Poisson summation for constant weights)."""
    q, xy, lam = _f64(q), _f64(xy), _f64(lam)
    s = np.empty(q.shape[0], dtype=np.float64)
    exact = rc is None
    lib().orc_evaluate(q.shape[0], _p(q), xy.shape[0], _p(xy), _p(lam), float(sigma),
                       0.0 if exact else float(rc), int(exact), _p(s))
    return s


def evaluate_tbox(q, xy, lam, sigma: float, box, cell: float, tau: float) -> np.ndarray:
    """Interpolant with the T-box of reading Q25: s(q) = sum_j [x_j in T(cell(q))]
    lambda_j phi(|q - x_j|^2), brute force.  Pinned: at the data points it is
    matvec_tbox (tests/test_oracle_kernel_matvec.py)."""
    q, xy, lam = _f64(q), _f64(xy), _f64(lam)
    s = np.empty(q.shape[0], dtype=np.float64)
    lib().orc_evaluate_tbox(q.shape[0], _p(q), xy.shape[0], _p(xy), _p(lam), float(sigma),
                            *map(float, box), float(cell), float(tau), _p(s))
    return s


def neglected_row_mass(xy, sigma: float, rc: float, rows) -> np.ndarray:
    """sum_{j: r_ij >= rc} phi(r2_ij) by brute force."""
    xy, rows = _f64(xy), _i64(rows)
    out = np.empty(rows.shape[0], dtype=np.float64)
    lib().orc_neglected_row_mass(xy.shape[0], _p(xy), float(sigma), float(rc),
                                 rows.shape[0], _p(rows), _p(out))
    return out


def grid_dims(box, cell: float) -> tuple[int, int]:
    """(ncx, ncy) = ceil((x1-x0)/c), ceil((y1-y0)/c) (reading Q5)."""
    ncx, ncy = C.c_int64(), C.c_int64()
    lib().orc_grid_dims(*map(float, box), float(cell), C.byref(ncx), C.byref(ncy))
    return ncx.value, ncy.value


def cell_list(xy, box, cell: float):
    """Cell key per point, stable sort permutation (sorted -> caller index) and
    cell_start offsets (reading Q5; index sets of P:250, 268)."""
    xy = _f64(xy)
    n = xy.shape[0]
    ncx, ncy = grid_dims(box, cell)
    key = np.empty(n, dtype=np.int64)
    perm = np.empty(n, dtype=np.int64)
    start = np.empty(ncx * ncy + 1, dtype=np.int64)
    lib().orc_cell_list(n, _p(xy), *map(float, box), float(cell), _p(key), _p(perm), _p(start))
    return key, perm, start


def matvec_cells(xy, w, sigma: float, rc: float, box, cell: float) -> np.ndarray:
    """orc_matvec_brute restricted to cells within ceil(rc/c) rings (acceleration only)."""
    xy, w = _f64(xy), _f64(w)
    y = np.empty(xy.shape[0], dtype=np.float64)
    st = lib().orc_matvec_cells(xy.shape[0], _p(xy), _p(w), float(sigma), float(rc),
                                *map(float, box), float(cell), _p(y))
    if st != ORC_OK:
        raise MemoryError("orc_matvec_cells")
    return y


def matvec_tbox(xy, w, sigma: float, box, cell: float, tau: float, rows=None,
                cells: bool = False) -> np.ndarray:
    """The paper's T-box truncation (reading Q25): y_i = sum_j
    [x_j in T(cell(i))] w_j phi(r2_ij), T(c) = cell c's box grown by tau on every side
    (closed), brute force over all j (cells=True: the cell-list form, all rows)."""
    xy, w = _f64(xy), _f64(w)
    n = xy.shape[0]
    if cells:
        y = np.empty(n, dtype=np.float64)
        st = lib().orc_matvec_tbox_cells(n, _p(xy), _p(w), float(sigma), *map(float, box),
                                         float(cell), float(tau), _p(y))
        if st != ORC_OK:
            raise MemoryError("orc_matvec_tbox_cells")
        return y
    if rows is None:
        y = np.empty(n, dtype=np.float64)
        lib().orc_matvec_tbox(n, _p(xy), _p(w), float(sigma), *map(float, box), float(cell),
                              float(tau), 0, None, _p(y))
    else:
        rows = _i64(rows)
        y = np.empty(rows.shape[0], dtype=np.float64)
        lib().orc_matvec_tbox(n, _p(xy), _p(w), float(sigma), *map(float, box), float(cell),
                              float(tau), rows.shape[0], _p(rows), _p(y))
    return y


def count_pairs(xy, rc: float, box, cell: float) -> int:
    """Number of ordered pairs (i, j), i == j included, with r2_ij < rc^2."""
    xy = _f64(xy)
    return int(lib().orc_count_pairs(xy.shape[0], _p(xy), float(rc), *map(float, box), float(cell)))


def dense_factor_solve(A, b) -> tuple[np.ndarray, bool]:
    """Cholesky solve, LU-with-partial-pivoting fallback (reading Q11)."""
    A, b = _f64(A), _f64(b)
    x = np.empty_like(b)
    used = C.c_int()
    st = lib().orc_dense_factor_solve(A.shape[0], _p(A), _p(b), _p(x), C.byref(used))
    if st != ORC_OK:
        raise ArithmeticError("singular matrix")
    return x, bool(used.value)


# --------------------------------------------------------------------------
# RASM preconditioner, Eqs.(5),(9)-(11) P:180-226
# --------------------------------------------------------------------------

class Rasm:
    """M^-1 = sum_c R~_c^T A_c^-1 R_c (Eq.(11)); one subdomain per
    non-empty cell, overlap `rings` cell rings (Q9) -- or, with overlap_width > 0,
    the points of that block inside the cell's box grown by overlap_width (the
    paper's D box, reading Q24) -- A_c the principal submatrix of A_rc (Q10),
    Cholesky with LU fallback (Q11)."""

    def __init__(self, xy, sigma: float, rc: float, box, cell: float, rings: int = 1,
                 overlap_width: float = 0.0):
        self.xy = _f64(xy)
        self.n = self.xy.shape[0]
        self._h = lib().orc_rasm_setup_box(self.n, _p(self.xy), float(sigma), float(rc),
                                           *map(float, box), float(cell), int(rings),
                                           float(overlap_width))
        bad, nsub, nlu = C.c_int64(), C.c_int64(), C.c_int64()
        self.status = lib().orc_rasm_status(self._h, C.byref(bad), C.byref(nsub), C.byref(nlu))
        self.bad_cell, self.nsub, self.n_lu = bad.value, nsub.value, nlu.value

    def apply(self, r, variant: str = "rasm") -> np.ndarray:
        """z = M^-1 r, Eq.(10) (variant 'rasm') or Eq.(8) (variant 'asm')."""
        r = _f64(r)
        z = np.empty(self.n, dtype=np.float64)
        lib().orc_rasm_apply(self._h, _p(r), _p(z), int(variant == "asm"))
        return z

    def subdomain(self, s: int):
        """(overlap caller indices R_c, local positions of own(c)) of subdomain s."""
        n_own, n_ov = C.c_int64(), C.c_int64()
        lib().orc_rasm_sub_info(self._h, s, C.byref(n_own), C.byref(n_ov))
        ov = np.empty(n_ov.value, dtype=np.int64)
        own = np.empty(n_own.value, dtype=np.int64)
        lib().orc_rasm_sub_sets(self._h, s, _p(ov), _p(own))
        return ov, own

    def close(self):
        if self._h:
            lib().orc_rasm_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# --------------------------------------------------------------------------
# GMRES, P:226 / SPEC S:264-284 / reading Q12
# --------------------------------------------------------------------------

class _Report(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("restarts", C.c_int64), ("converged", C.c_int),
                ("status", C.c_int), ("resid_est", C.c_double), ("resid_precond", C.c_double),
                ("resid_true", C.c_double), ("beta0", C.c_double)]


@dataclass
class GmresResult:
    x: np.ndarray
    iterations: int
    restarts: int
    converged: bool
    status: int
    resid_est: float
    resid_precond: float
    resid_true: float
    beta0: float
    history: np.ndarray
    basis: np.ndarray | None = None


def _op_buf():
    return C.create_string_buffer(int(lib().orc_op_size()))


def _addr(buf) -> C.c_void_p:
    return C.c_void_p(C.addressof(buf))


def op_identity(n):
    b = _op_buf(); lib().orc_op_identity(_addr(b), int(n)); return (b, None)


def op_dense(A):
    A = _f64(A)
    b = _op_buf(); lib().orc_op_dense(_addr(b), A.shape[0], _p(A)); return (b, A)


def op_rbf(xy, sigma, rc, box, cell, brute=False):
    xy = _f64(xy)
    b = _op_buf()
    lib().orc_op_rbf(_addr(b), xy.shape[0], _p(xy), float(sigma), float(rc), *map(float, box),
                     float(cell), int(brute))
    return (b, xy)


def op_rbf_tbox(xy, sigma, box, cell, tau):
    xy = _f64(xy)
    b = _op_buf()
    lib().orc_op_rbf_tbox(_addr(b), xy.shape[0], _p(xy), float(sigma), *map(float, box),
                          float(cell), float(tau))
    return (b, xy)


def op_rasm(P: Rasm, variant: str = "rasm"):
    b = _op_buf(); lib().orc_op_rasm(_addr(b), P._h, int(variant == "asm")); return (b, P)


def gmres(opA, opM, b, restart=30, max_iters=1000, rtol=1e-13, atol=0.0,
          keep_basis=False, orth="mgs") -> GmresResult:
    """Left-preconditioned restarted GMRES(m), Givens, x0 = 0 (Q12); Arnoldi by
    modified Gram-Schmidt (orth="mgs", Q12) or classical Gram-Schmidt twice
    (orth="cgs2", reading Q23)."""
    b = _f64(b)
    n = b.shape[0]
    x = np.empty(n, dtype=np.float64)
    hist = np.zeros(max_iters, dtype=np.float64)
    rep = _Report()
    V = np.empty((restart + 1, n), dtype=np.float64) if keep_basis else None
    nv = C.c_int64(0)
    st = lib().orc_gmres_orth(_addr(opA[0]), _addr(opM[0]), _p(b), int(restart), int(max_iters),
                         float(rtol), float(atol), {"mgs": 0, "cgs2": 1, "dcgs2": 2}[orth], _p(x), _p(hist),
                         int(max_iters), C.byref(rep),
                         _p(V) if V is not None else None, C.byref(nv))
    if st == ORC_EINVAL:
        raise ValueError("invalid GMRES parameters")
    return GmresResult(x=x, iterations=rep.iterations, restarts=rep.restarts,
                       converged=bool(rep.converged), status=st, resid_est=rep.resid_est,
                       resid_precond=rep.resid_precond, resid_true=rep.resid_true,
                       beta0=rep.beta0, history=hist[: rep.iterations].copy(),
                       basis=None if V is None else V[: nv.value].copy())


def solve(xy, f, sigma, rc, box, cell, rings=1, restart=30, max_iters=1000, rtol=1e-13,
          atol=0.0, brute=False, orth="mgs", overlap_width=0.0,
          trunc_width=0.0, schwarz="rasm") -> GmresResult:
    """Solve A_rc lambda = f by GMRES(restart) left-preconditioned with RASM
    (the paper's KSPSolve).  trunc_width > 0 solves with the
    paper's T-box matvec instead (reading Q25; the local matrices stay A_rc's);
    schwarz="asm" preconditions with Eq.(8) instead of Eq.(11) (reading Q26)."""
    P = Rasm(xy, sigma, rc, box, cell, rings, overlap_width)
    if P.status != ORC_OK:
        raise ArithmeticError(f"RASM setup failed in cell {P.bad_cell}")
    try:
        opA = (op_rbf_tbox(xy, sigma, box, cell, trunc_width) if trunc_width > 0
               else op_rbf(xy, sigma, rc, box, cell, brute))
        return gmres(opA, op_rasm(P, schwarz), f, restart,
                     max_iters, rtol, atol, orth=orth)
    finally:
        P.close()


def dense_solve(xy, f, sigma, rc) -> np.ndarray:
    """Direct solve of A_rc lambda = f (Cholesky via scipy/LAPACK) -- the exact
    answer GMRES approximates, for N <= ~1e4 (Eq.(4))."""
    import scipy.linalg as sla

    A = assemble_dense(xy, sigma, rc)
    c = sla.cho_factor(A, lower=True, check_finite=False)
    return sla.cho_solve(c, _f64(f), check_finite=False)
