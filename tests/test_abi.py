"""C-ABI library checks that need no GPU: it loads, exports every symbol include/grf.h
declares, validates arguments, and its host-side plan matches the oracle's."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from oracle import quadrature


@pytest.fixture(scope="module")
def lib(repo_root):
    from paper_2605_02670_b200 import build
    build.build()
    from paper_2605_02670_b200 import _lib
    return _lib.load()


def _header_functions(repo_root):
    src = open(os.path.join(repo_root, "include", "grf.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(grf_[a-z_0-9]+)\s*\(", src)))


def test_exports_every_declared_symbol(lib, repo_root):
    names = _header_functions(repo_root)
    assert len(names) >= 18
    for n in names:
        assert hasattr(lib, n), f"libgrf.so does not export {n}"
    from paper_2605_02670_b200 import EXPORTS
    assert sorted(EXPORTS) == names


def test_sm100a_code_in_library(repo_root):
    import subprocess
    from paper_2605_02670_b200 import LIB_PATH
    out = subprocess.run(["cuobjdump", "--list-elf", LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_plan_info_matches_oracle(lib):
    from paper_2605_02670_b200 import plan_info
    for beta, k in [(0.75, 0.5), (0.6, 0.2), (0.75, 0.25), (0.55, 0.3), (0.9, 0.2)]:
        km, kp, cI, cL = plan_info(beta, k)
        p = quadrature.plan(beta, k)
        assert (km, kp) == (p.K_minus, p.K_plus)
        assert np.allclose(cI, p.c_I, rtol=1e-15, atol=0) and np.allclose(cL, p.c_L, rtol=1e-15, atol=0)


def test_plan_info_rejects_bad_beta(lib):
    km = C.c_int64()
    for beta in (0.25, 1.0, -1.0, float("nan")):
        assert lib.grf_plan_info(beta, 0.2, C.byref(km), None, None, None) == 1  # GRF_EINVAL
    assert lib.grf_plan_info(0.5, 0.0, C.byref(km), None, None, None) == 1
    assert b"beta" in lib.grf_last_error() or b"k must" in lib.grf_last_error()


def _create(lib, nv, eu, ev, ln, h):
    eu = np.asarray(eu, dtype=np.int64)
    ev = np.asarray(ev, dtype=np.int64)
    ln = np.asarray(ln, dtype=np.float64)
    out = C.c_void_p()
    p = C.POINTER(C.c_int64)
    return lib.grf_graph_create(nv, len(eu), eu.ctypes.data_as(p), ev.ctypes.data_as(p),
                                ln.ctypes.data_as(C.POINTER(C.c_double)), h, None, C.byref(out))


def test_graph_create_validation(lib):
    assert _create(lib, 2, [0], [1], [-2.0], 0.1) == 1          # non-positive length (S46)
    assert b"length" in lib.grf_last_error()
    assert _create(lib, 2, [0], [2], [1.0], 0.1) == 1           # endpoint out of range
    assert _create(lib, 3, [0], [1], [1.0], 0.1) == 1           # isolated vertex
    assert b"isolated" in lib.grf_last_error()
    assert _create(lib, 2, [0], [1], [1.0], 0.0) == 1           # h <= 0
    assert _create(lib, 2, [0], [1], [float("inf")], 0.1) == 1  # non-finite length
    assert _create(lib, 0, [0], [0], [1.0], 0.1) == 1
