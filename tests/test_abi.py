"""CPU-side checks of the C-ABI boundary: libcvx.so loads, exports every symbol include/cvx.h declares,
the binding declares a signature for each, and host-side argument validation works without a GPU."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "cvx.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cvx_[a-z_]+)\s*\(", src)))


def test_header_declares_the_four_calls():
    d = _declared()
    for name in ("cvx_create_submap", "cvx_integrate_pointcloud", "cvx_finalize_esdf", "cvx_query_distance"):
        assert name in d


def test_library_exports_every_declared_symbol():
    import paper_2410_21149_b200 as p
    L = p.lib()
    for name in _declared():
        assert hasattr(L, name), name
    assert set(_declared()) == set(p.SIGNATURES), set(_declared()) ^ set(p.SIGNATURES)
    assert b"sm_100a" in L.cvx_version()


def test_library_is_sm100a_cubin():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", os.path.join(ROOT, "paper_2410_21149_b200", "libcvx.so")],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_host_validation_without_gpu():
    import paper_2410_21149_b200.cvx as cv
    L = cv.lib()
    h = C.c_void_p()
    T = np.eye(4)
    bad = cv.GridConfig(0.1, 16, 0.3, 0, 0.1, 1, 0.1, 1024)        # block_side != 8
    assert L.cvx_create_submap(C.byref(bad), T.ctypes.data_as(C.c_void_p), 0, C.byref(h)) == cv.E_INVALID
    assert b"block_side" in L.cvx_last_error()
    bad = cv.GridConfig(-0.1, 8, 0.3, 0, 0.1, 1, 0.1, 1024)
    assert L.cvx_create_submap(C.byref(bad), T.ctypes.data_as(C.c_void_p), 0, C.byref(h)) == cv.E_INVALID
    ok = cv.GridConfig(0.1, 8, 0.3, 0, 0.1, 1, 0.1, 1024)
    T2 = T.copy()
    T2[0, 1] = 0.5                                                  # not a rotation
    assert L.cvx_create_submap(C.byref(ok), T2.ctypes.data_as(C.c_void_p), 0, C.byref(h)) == cv.E_INVALID
    assert L.cvx_destroy_submap(None) == cv.OK
    assert L.cvx_integrate_pointcloud(None, None, 0, None, None, None, None) == cv.E_INVALID
    assert L.cvx_finalize_esdf(None, None) == cv.E_INVALID
    assert L.cvx_query_distance(None, None, 0, None, None, None) == cv.E_INVALID


def test_no_cpu_fallback_in_product_package():
    """The product package never imports the oracle or computes the method in Python."""
    pkg = os.path.join(ROOT, "paper_2410_21149_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            src = open(os.path.join(pkg, fn)).read()
            assert "import oracle" not in src and "from oracle" not in src, fn
