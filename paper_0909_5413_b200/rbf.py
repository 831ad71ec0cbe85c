"""Thin Python binding of librbf.so (include/rbf.h).  Argument marshalling only:
every step of the hot path runs in the library's CUDA kernels.  PyTorch provides
device memory and streams.  There is no fallback: if the library is missing or no
GPU is present, calls raise."""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "librbf.so")

RBF_OK, RBF_NOT_CONVERGED = 0, 2
RBF_COMM_NONE, RBF_COMM_NCCL, RBF_COMM_THREADS = 0, 1, 2
RBF_DIST_NO_OVERLAP = 1
_ERRORS = {-1: "EINVAL", -2: "ENOMEM", -3: "ECUDA", -4: "ENCCL", -5: "EFACTOR", -6: "ENUMERIC",
           -7: "EUNSUPPORTED"}


class RbfError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"rbf error {code} ({_ERRORS.get(code, '?')}): {msg}")
        self.code = code


class Params(C.Structure):
    _fields_ = [("sigma", C.c_double), ("cell", C.c_double), ("rc", C.c_double),
                ("overlap_rings", C.c_int32), ("schwarz", C.c_int32),
                ("x0", C.c_double), ("y0", C.c_double), ("x1", C.c_double), ("y1", C.c_double),
                ("overlap_width", C.c_double), ("trunc_width", C.c_double)]


class Dist(C.Structure):
    _fields_ = [("rank", C.c_int32), ("nranks", C.c_int32), ("comm", C.c_int32),
                ("flags", C.c_int32), ("nccl_id", C.c_ubyte * 128)]


class GmresParams(C.Structure):
    _fields_ = [("restart", C.c_int32), ("max_iters", C.c_int32), ("rtol", C.c_double),
                ("atol", C.c_double), ("timing", C.c_int32), ("orth", C.c_int32)]


class Report(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("converged", C.c_int32), ("restarts", C.c_int32),
                ("status", C.c_int32), ("resid_est", C.c_double), ("resid_precond", C.c_double),
                ("resid_true", C.c_double), ("beta0", C.c_double), ("ms_setup", C.c_double),
                ("ms_matmult", C.c_double), ("ms_pcapply", C.c_double), ("ms_orth", C.c_double),
                ("ms_total", C.c_double), ("n_pairs", C.c_int64), ("n_cells", C.c_int64),
                ("bytes_device", C.c_int64), ("history", C.POINTER(C.c_double)),
                ("history_cap", C.c_int32), ("history_len", C.c_int32)]


EXPORTS = ["rbf_get_nccl_id", "rbf_setup", "rbf_local_count", "rbf_ext_count", "rbf_ranges",
           "rbf_local_index", "rbf_cell_list", "rbf_to_local", "rbf_from_local", "rbf_matvec",
           "rbf_rasm_apply", "rbf_matvec_ext", "rbf_rasm_apply_ext", "rbf_solve",
           "rbf_interpolate_host", "rbf_count_pairs", "rbf_dot", "rbf_plan_strips",
           "rbf_last_error", "rbf_destroy", "rbf_info", "rbf_launch_count", "rbf_setup_times",
           "rbf_plan_halo", "rbf_evaluate", "rbf_matvec_stats", "rbf_lu_stats",
           "rbf_debug_poison_shared", "rbf_debug_krylov_basis", "rbf_evaluate_count_pairs", "rbf_set_option", "rbf_get_option", "rbf_trim_memory"]

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                               "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        p, i64, i32 = C.c_void_p, C.c_int64, C.c_int32
        sigs = {
            "rbf_get_nccl_id": (C.c_int, [p]),
            "rbf_setup": (C.c_int, [C.POINTER(p), p, i64, C.POINTER(Params), C.POINTER(Dist), p]),
            "rbf_local_count": (i64, [p]),
            "rbf_ext_count": (i64, [p]),
            "rbf_ranges": (C.c_int, [p, p]),
            "rbf_local_index": (C.c_int, [p, p, p]),
            "rbf_cell_list": (C.c_int, [p, p, p, p, p]),
            "rbf_to_local": (C.c_int, [p, p, p, p]),
            "rbf_from_local": (C.c_int, [p, p, p, p]),
            "rbf_matvec": (C.c_int, [p, p, p, p]),
            "rbf_rasm_apply": (C.c_int, [p, p, p, p]),
            "rbf_matvec_ext": (C.c_int, [p, p, p, p]),
            "rbf_rasm_apply_ext": (C.c_int, [p, p, p, p]),
            "rbf_solve": (C.c_int, [p, p, C.POINTER(GmresParams), p, C.POINTER(Report), p]),
            "rbf_interpolate_host": (C.c_int, [p, p, i64, C.POINTER(Params), C.POINTER(GmresParams),
                                               p, C.POINTER(Report), p]),
            "rbf_count_pairs": (C.c_int, [p, p, p]),
            "rbf_evaluate": (C.c_int, [p, p, i64, p, p, p]),
            "rbf_evaluate_count_pairs": (C.c_int, [p, p, i64, C.POINTER(i64), p]),
            "rbf_matvec_stats": (C.c_int, [p, p]),
            "rbf_lu_stats": (C.c_int, [p, p]),
            "rbf_debug_poison_shared": (C.c_int, []),
            "rbf_set_option": (C.c_int, [C.c_char_p, i64]),
            "rbf_trim_memory": (C.c_int, []),
            "rbf_get_option": (C.c_int, [C.c_char_p, C.POINTER(i64)]),
            "rbf_debug_krylov_basis": (C.c_int, [p, p, i32, p]),
            "rbf_dot": (C.c_int, [p, p, p, p, p]),
            "rbf_plan_strips": (C.c_int, [p, i64, i32, i64, p]),
            "rbf_last_error": (C.c_char_p, []),
            "rbf_info": (C.c_int, [p, p]),
            "rbf_launch_count": (i64, []),
            "rbf_setup_times": (C.c_int, [p, p]),
            "rbf_plan_halo": (C.c_int, [p, i64, p, i32, i32, i32, i32, p]),
            "rbf_destroy": (None, [p]),
        }
        for name, (res, args) in sigs.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(code: int) -> int:
    if code < 0:
        raise RbfError(code, lib().rbf_last_error().decode())
    return code


def _ptr(t) -> C.c_void_p:
    return C.c_void_p(t.data_ptr())


def _stream(stream):
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


SCHWARZ = {"rasm": 0, "asm": 1}


def make_params(sigma, cell, rc, rings=1, box=(-1.0, -1.0, 1.0, 1.0), overlap_width=0.0,
                trunc_width=0.0, schwarz="rasm") -> Params:
    return Params(float(sigma), float(cell), float(rc), int(rings), SCHWARZ[schwarz],
                  *map(float, box), float(overlap_width), float(trunc_width))


def poison_shared() -> None:
    """Test hook: NaN-fill every SM's shared memory (rbf_debug_poison_shared)."""
    _check(lib().rbf_debug_poison_shared())


def set_option(name: str, value: int) -> None:
    """rbf_set_option: a process-wide test / A/B switch (include/rbf.h)."""
    _check(lib().rbf_set_option(name.encode(), int(value)))


def trim_memory() -> None:
    """rbf_trim_memory: release the library's kept buffers and trim the memory pool."""
    _check(lib().rbf_trim_memory())


def get_option(name: str) -> int:
    v = C.c_int64()
    _check(lib().rbf_get_option(name.encode(), C.byref(v)))
    return v.value


class options:
    """Context manager: set library options, restore them on exit (tests, tools)."""

    def __init__(self, **kw):
        self.kw = kw
        self.old = {}

    def __enter__(self):
        for k, v in self.kw.items():
            self.old[k] = get_option(k)
            set_option(k, v)
        return self

    def __exit__(self, *a):
        for k, v in self.old.items():
            set_option(k, v)


def launch_count() -> int:
    """Kernel launches issued by librbf.so so far (process-wide)."""
    return int(lib().rbf_launch_count())


def get_nccl_id() -> bytes:
    buf = (C.c_ubyte * 128)()
    _check(lib().rbf_get_nccl_id(buf))
    return bytes(buf)


def plan_strips(row_counts, nranks: int, min_rows: int) -> np.ndarray:
    """Host-only strip planner (no GPU needed)."""
    rc = np.ascontiguousarray(row_counts, dtype=np.int64)
    out = np.zeros(nranks + 1, dtype=np.int64)
    _check(lib().rbf_plan_strips(rc.ctypes.data_as(C.c_void_p), rc.shape[0], int(nranks),
                                 int(min_rows), out.ctypes.data_as(C.c_void_p)))
    return out


def plan_halo(row_start, row_bounds, rank: int, kh: int, rings: int) -> dict:
    """Host-only halo plan of strip `rank` (the one rbf_setup uses)."""
    rs = np.ascontiguousarray(row_start, dtype=np.int64)
    rb = np.ascontiguousarray(row_bounds, dtype=np.int64)
    out = np.zeros(12, dtype=np.int64)
    _check(lib().rbf_plan_halo(rs.ctypes.data_as(C.c_void_p), rs.shape[0] - 1,
                               rb.ctypes.data_as(C.c_void_p), rb.shape[0] - 1, int(rank), int(kh),
                               int(rings), out.ctypes.data_as(C.c_void_p)))
    keys = ["ext_lo", "own_lo", "own_hi", "ext_hi",
            "below_send_off", "below_send_cnt", "below_recv_off", "below_recv_cnt",
            "above_send_off", "above_send_cnt", "above_recv_off", "above_recv_cnt"]
    return {k: int(v) for k, v in zip(keys, out)}


@dataclass
class SolveReport:
    iterations: int
    converged: bool
    restarts: int
    status: int
    resid_est: float
    resid_precond: float
    resid_true: float
    beta0: float
    ms_matmult: float
    ms_pcapply: float
    ms_orth: float
    ms_total: float
    n_cells: int
    bytes_device: int
    history: np.ndarray = field(default_factory=lambda: np.zeros(0))


def _report(rep: Report, hist: np.ndarray) -> SolveReport:
    return SolveReport(rep.iterations, bool(rep.converged), rep.restarts, rep.status, rep.resid_est,
                       rep.resid_precond, rep.resid_true, rep.beta0, rep.ms_matmult, rep.ms_pcapply,
                       rep.ms_orth, rep.ms_total, rep.n_cells, rep.bytes_device,
                       hist[: rep.history_len].copy())


class Context:
    """rbf_setup / rbf_matvec / rbf_rasm_apply / rbf_solve on one strip (one GPU)."""

    def __init__(self, xy, sigma, cell, rc, rings=1, box=(-1.0, -1.0, 1.0, 1.0), *, rank=0,
                 nranks=1, comm="none", nccl_id: bytes | None = None, stream=None,
                 overlap_width=0.0, trunc_width=0.0, schwarz="rasm", overlap=True):
        import torch

        if not (isinstance(xy, torch.Tensor) and xy.is_cuda and xy.dtype == torch.float64):
            raise TypeError("xy must be a CUDA float64 tensor of shape (N, 2)")
        xy = xy.contiguous()
        self.n = int(xy.shape[0])
        self.params = make_params(sigma, cell, rc, rings, box, overlap_width, trunc_width, schwarz)
        dist = None
        if nranks > 1 or comm == "nccl":
            mode = {"nccl": RBF_COMM_NCCL, "threads": RBF_COMM_THREADS, "none": RBF_COMM_NONE}[comm]
            dist = Dist(int(rank), int(nranks), mode, 0 if overlap else RBF_DIST_NO_OVERLAP)
            if nccl_id is not None:
                C.memmove(dist.nccl_id, nccl_id, 128)
        self._h = C.c_void_p()
        self._stream = stream
        _check(lib().rbf_setup(C.byref(self._h), _ptr(xy), self.n, C.byref(self.params),
                               C.byref(dist) if dist is not None else None, _stream(stream)))
        self.n_local = int(lib().rbf_local_count(self._h))
        self.n_ext = int(lib().rbf_ext_count(self._h))
        r = np.zeros(4, dtype=np.int64)
        _check(lib().rbf_ranges(self._h, r.ctypes.data_as(C.c_void_p)))
        self.ext_lo, self.own_lo, self.own_hi, self.ext_hi = map(int, r)

    # ------------------------------------------------------------------ helpers
    def _new(self, n):
        import torch

        return torch.empty(n, dtype=torch.float64, device="cuda")

    def local_index(self):
        import torch

        idx = torch.empty(self.n_local, dtype=torch.int64, device="cuda")
        _check(lib().rbf_local_index(self._h, _ptr(idx), _stream(self._stream)))
        return idx

    def cell_list(self):
        import torch

        dims = np.zeros(2, dtype=np.int64)
        _check(lib().rbf_cell_list(self._h, None, None, dims.ctypes.data_as(C.c_void_p),
                                   _stream(self._stream)))
        perm = torch.empty(self.n, dtype=torch.int64, device="cuda")
        cs = torch.empty(int(dims[0] * dims[1] + 1), dtype=torch.int64, device="cuda")
        _check(lib().rbf_cell_list(self._h, _ptr(perm), _ptr(cs), dims.ctypes.data_as(C.c_void_p),
                                   _stream(self._stream)))
        return perm, cs, (int(dims[0]), int(dims[1]))

    def to_local(self, v_caller):
        out = self._new(self.n_local)
        _check(lib().rbf_to_local(self._h, _ptr(v_caller.contiguous()), _ptr(out), _stream(self._stream)))
        return out

    def from_local(self, v_loc, out=None):
        if out is None:
            out = self._new(self.n)
            out.zero_()
        _check(lib().rbf_from_local(self._h, _ptr(v_loc.contiguous()), _ptr(out), _stream(self._stream)))
        return out

    # ------------------------------------------------------------------ operators
    def matvec(self, w, y=None):
        y = self._new(self.n_local) if y is None else y
        _check(lib().rbf_matvec(self._h, _ptr(w), _ptr(y), _stream(self._stream)))
        return y

    def evaluate(self, q_xy, lam, s=None):
        """Interpolant s(q) at query points q_xy (m x 2, device, fp64) from the
        local weights lam (rbf_evaluate, Eq.(1)); returns s in query order."""
        m = int(q_xy.shape[0])
        s = self._new(m) if s is None else s
        _check(lib().rbf_evaluate(self._h, _ptr(q_xy.contiguous()), m, _ptr(lam), _ptr(s),
                                  _stream(self._stream)))
        return s

    def evaluate_count_pairs(self, q_xy) -> int:
        """In-cutoff (query, source) pairs of an evaluation at q_xy (rbf_evaluate_count_pairs)."""
        v = C.c_int64()
        _check(lib().rbf_evaluate_count_pairs(self._h, _ptr(q_xy.contiguous()), int(q_xy.shape[0]),
                                              C.byref(v), _stream(self._stream)))
        return v.value

    def rasm_apply(self, r, z=None):
        z = self._new(self.n_local) if z is None else z
        _check(lib().rbf_rasm_apply(self._h, _ptr(r), _ptr(z), _stream(self._stream)))
        return z

    def matvec_ext(self, w_ext, y=None):
        y = self._new(self.n_local) if y is None else y
        _check(lib().rbf_matvec_ext(self._h, _ptr(w_ext), _ptr(y), _stream(self._stream)))
        return y

    def rasm_apply_ext(self, r_ext, z=None):
        z = self._new(self.n_local) if z is None else z
        _check(lib().rbf_rasm_apply_ext(self._h, _ptr(r_ext), _ptr(z), _stream(self._stream)))
        return z

    def solve(self, f_loc, restart=30, max_iters=1000, rtol=1e-13, atol=0.0, timing=False,
              lam=None, orth="mgs"):
        lam = self._new(self.n_local) if lam is None else lam
        gp = GmresParams(int(restart), int(max_iters), float(rtol), float(atol), int(timing),
                         {"mgs": 0, "cgs2": 1, "dcgs2": 2}[orth])
        hist = np.zeros(max_iters, dtype=np.float64)
        rep = Report()
        rep.history = hist.ctypes.data_as(C.POINTER(C.c_double))
        rep.history_cap = max_iters
        code = _check(lib().rbf_solve(self._h, _ptr(f_loc), C.byref(gp), _ptr(lam), C.byref(rep),
                                      _stream(self._stream)))
        r = _report(rep, hist)
        r.status = code
        return lam, r

    def info(self) -> dict:
        o = np.zeros(8, dtype=np.int64)
        _check(lib().rbf_info(self._h, o.ctypes.data_as(C.c_void_p)))
        keys = ["x_doubles", "nsub", "max_ov", "max_own", "n_lu", "ncx", "ncy", "bytes_device"]
        return {k: int(v) for k, v in zip(keys, o)}

    def setup_times(self) -> dict:
        o = np.zeros(4, dtype=np.float64)
        _check(lib().rbf_setup_times(self._h, o.ctypes.data_as(C.c_void_p)))
        return dict(zip(["cell_list", "nlist", "rasm", "total"], map(float, o)))

    def matvec_stats(self) -> dict:
        o = (C.c_int64 * 4)()
        _check(lib().rbf_matvec_stats(self._h, o))
        return dict(zip(["lanes", "chunks", "ell_entries", "union_entries"], map(int, o)))

    def lu_stats(self) -> dict:
        o = (C.c_int64 * 2)()
        _check(lib().rbf_lu_stats(self._h, o))
        return {"n_lu": int(o[0]), "n_lu_pivot": int(o[1])}

    def krylov_basis(self, nvec: int):
        """Test hook: the first nvec GMRES basis vectors of the last solve's last cycle
        (rbf_debug_krylov_basis), an (nvec, n_local) device tensor."""
        import torch

        V = torch.empty((int(nvec), self.n_local), dtype=torch.float64, device="cuda")
        _check(lib().rbf_debug_krylov_basis(self._h, _ptr(V), int(nvec), _stream(self._stream)))
        return V

    def count_pairs(self) -> int:
        v = C.c_int64()
        _check(lib().rbf_count_pairs(self._h, C.byref(v), _stream(self._stream)))
        return v.value

    def dot(self, a, b) -> float:
        v = C.c_double()
        _check(lib().rbf_dot(self._h, _ptr(a), _ptr(b), C.byref(v), _stream(self._stream)))
        return v.value

    def close(self):
        if self._h:
            lib().rbf_destroy(self._h)
            self._h = C.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def interpolate_host(xy: np.ndarray, f: np.ndarray, sigma, cell, rc, rings=1,
                     box=(-1.0, -1.0, 1.0, 1.0), restart=30, max_iters=1000, rtol=1e-13,
                     atol=0.0, stream=None, overlap_width=0.0, orth="mgs", trunc_width=0.0,
                     out=None):
    """rbf_interpolate_host: host buffers in caller order -> weights lambda (host).  `out`:
    optional float64 host array for lambda (e.g. pinned memory, reused across calls)."""
    xy = np.ascontiguousarray(xy, dtype=np.float64)
    f = np.ascontiguousarray(f, dtype=np.float64)
    if out is not None:
        if (not isinstance(out, np.ndarray) or out.dtype != np.float64 or out.shape != f.shape
                or not out.flags.c_contiguous):
            raise ValueError("interpolate_host: out must be a contiguous float64 array shaped like f")
        lam = out
    else:
        lam = np.empty_like(f)
    prm = make_params(sigma, cell, rc, rings, box, overlap_width, trunc_width)
    gp = GmresParams(int(restart), int(max_iters), float(rtol), float(atol), 0,
                     {"mgs": 0, "cgs2": 1, "dcgs2": 2}[orth])
    hist = np.zeros(max_iters, dtype=np.float64)
    rep = Report()
    rep.history = hist.ctypes.data_as(C.POINTER(C.c_double))
    rep.history_cap = max_iters
    code = _check(lib().rbf_interpolate_host(xy.ctypes.data_as(C.c_void_p),
                                             f.ctypes.data_as(C.c_void_p), xy.shape[0],
                                             C.byref(prm), C.byref(gp),
                                             lam.ctypes.data_as(C.c_void_p), C.byref(rep),
                                             _stream(stream)))
    r = _report(rep, hist)
    r.status = code
    return lam, r
