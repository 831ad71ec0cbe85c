"""CPU-only checks of the C-ABI library: it loads, exports every entry point that
include/rbf.h declares, its host-only planners are right, and compute calls fail
loudly (no CPU fallback) when there is no GPU."""
import ctypes as C
import os
import re
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rbf.h")


def _lib():
    from paper_0909_5413_b200 import build as B

    if not os.path.exists(B.LIB):
        B.build()
    import paper_0909_5413_b200 as P

    return P


def header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(rbf_[a-z_0-9]+)\s*\(", text)))


def test_header_symbols_exported():
    P = _lib()
    L = P.lib()
    names = header_functions()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    assert set(names) <= set(P.EXPORTS) | {"rbf_debug_probe"}


def test_library_is_sm100a_native():
    P = _lib()
    out = subprocess.run(["cuobjdump", "--list-elf", P.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_plan_strips_balanced_and_minimum():
    P = _lib()
    counts = np.full(41, 25)
    counts[-1] = 10  # ragged last row
    b = P.plan_strips(counts, 4, 2)
    assert b[0] == 0 and b[-1] == 41 and np.all(np.diff(b) >= 2)
    sizes = [counts[b[g]:b[g + 1]].sum() for g in range(4)]
    assert max(sizes) - min(sizes) <= 2 * 25
    # clustered rows: balanced by points, not by rows
    counts = np.array([1] * 30 + [100] * 10 + [1] * 30)
    b = P.plan_strips(counts, 2, 2)
    s = [counts[b[0]:b[1]].sum(), counts[b[1]:b[2]].sum()]
    assert abs(s[0] - s[1]) <= 100
    with pytest.raises(P.RbfError):
        P.plan_strips(np.full(5, 10), 4, 2)  # 4 strips x 2 rows > 5 rows


def test_plan_halo_partition():
    P = _lib()
    rng = np.random.default_rng(0)
    counts = rng.integers(0, 40, size=30)
    rs = np.concatenate([[0], np.cumsum(counts)])
    for nr in (1, 2, 3, 5):
        b = P.plan_strips(counts, nr, 2)
        own = []
        for g in range(nr):
            h = P.plan_halo(rs, b, g, 2, 1)
            assert h["own_lo"] == rs[b[g]] and h["own_hi"] == rs[b[g + 1]]
            assert h["ext_lo"] == rs[max(b[g] - 2, 0)] and h["ext_hi"] == rs[min(b[g + 1] + 2, 30)]
            own.append((h["own_lo"], h["own_hi"]))
            if g > 0:  # what I receive from below is what rank g-1 sends up
                hb = P.plan_halo(rs, b, g - 1, 2, 1)
                assert h["below_recv_cnt"] == hb["above_send_cnt"]
                assert h["ext_lo"] + h["below_recv_off"] == hb["own_lo"] + hb["above_send_off"]
        assert own[0][0] == 0 and own[-1][1] == rs[-1]
        assert all(own[i][1] == own[i + 1][0] for i in range(nr - 1))


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="checks the no-GPU failure path")
def test_compute_calls_fail_without_gpu():
    P = _lib()
    L = P.lib()
    xy = np.zeros((4, 2))
    prm = P.rbf.make_params(0.1, 0.5, 0.6)
    h = C.c_void_p()
    code = L.rbf_setup(C.byref(h), xy.ctypes.data_as(C.c_void_p), 4, C.byref(prm), None, None)
    assert code == -3  # RBF_ECUDA
    assert b"no CPU fallback" in L.rbf_last_error()
    # argument validation happens before the device check
    bad = P.rbf.make_params(-1.0, 0.5, 0.6)
    assert L.rbf_setup(C.byref(h), xy.ctypes.data_as(C.c_void_p), 4, C.byref(bad), None, None) == -1
    far = P.rbf.make_params(0.01, 0.5, 1.0)  # rc > 37 sigma
    assert L.rbf_setup(C.byref(h), xy.ctypes.data_as(C.c_void_p), 4, C.byref(far), None, None) == -1


def test_binding_fails_loudly_without_library(tmp_path):
    code = ("import paper_0909_5413_b200.rbf as R; R.LIB_PATH='/nonexistent/librbf.so'\n"
            "try:\n    R.lib()\nexcept RuntimeError as e:\n    print('RAISED', e)\n")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT)
    assert "RAISED" in out.stdout and "no CPU fallback" in out.stdout


def test_product_does_not_import_oracle():
    """The product path never imports oracle/ (DESIGN.md 'Boundary')."""
    for dirpath, _, files in os.walk(os.path.join(ROOT, "paper_0909_5413_b200")):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text
                assert "rbf_oracle" not in text


def test_weak_scaling_workload_and_strips():
    """bench.py --scaling weak: world copies of cfg2 stacked in y; one copy per strip."""
    import rbf_workloads as W
    import oracle as O

    P = _lib()
    a, b = W.weak(1), W.config(2)
    assert np.array_equal(a.xy, b.xy) and np.array_equal(a.f, b.f) and a.box == b.box
    c = W.weak(4)
    assert c.n == 4 * b.n and np.array_equal(c.xy[:b.n], b.xy)
    assert np.max(np.abs(c.f[:b.n] - b.f)) < 1e-9 * np.max(np.abs(b.f))
    # strips balanced by point count give each rank one block (+- one cell row)
    key, _, start = O.cell_list(c.xy, c.box, c.cell)
    ncx, ncy = O.grid_dims(c.box, c.cell)
    rows = np.array([start[(r + 1) * ncx] - start[r * ncx] for r in range(ncy)])
    bnd = P.plan_strips(rows, 4, 2)
    own = [int(rows[bnd[g]:bnd[g + 1]].sum()) for g in range(4)]
    assert sum(own) == c.n and max(abs(o - b.n) for o in own) <= 2 * rows.max()


def test_options_api_without_gpu():
    """rbf_set_option / rbf_get_option (include/rbf.h): the library's only switches (it
    reads no environment variables); range-checked, restorable, no GPU needed."""
    import paper_0909_5413_b200 as P

    assert P.get_option("lu_nopiv") == 1 and P.get_option("solve_graph") == 1
    with P.options(lu_nopiv=0, mv_targets_per_lane=3):
        assert P.get_option("lu_nopiv") == 0 and P.get_option("mv_targets_per_lane") == 3
    assert P.get_option("lu_nopiv") == 1 and P.get_option("mv_targets_per_lane") == 2
    with pytest.raises(P.RbfError):
        P.set_option("mv_targets_per_lane", 4)
    with pytest.raises(P.RbfError):
        P.set_option("no_such_option", 1)


def test_library_reads_no_environment():
    import glob

    for f in glob.glob(os.path.join(ROOT, "paper_0909_5413_b200", "csrc", "*.cu*")):
        assert "getenv" not in open(f).read(), f
