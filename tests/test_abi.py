"""CPU-side checks of the C-ABI boundary (no compute calls without a GPU): libmhd.so loads,
exports every symbol include/mhd.h declares, and argument validation happens before any CUDA
call.  Also: the product package never imports the oracle."""
import ast
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2510_24175_b200 import build, mhd
    build.build()
    return mhd.load()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "mhd.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mhd_[a-z_]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    syms = declared_symbols()
    for s in ("mhd_create", "mhd_set_state", "mhd_compute_dt", "mhd_step", "mhd_get_state", "mhd_destroy"):
        assert s in syms


def test_library_exports_every_declared_symbol(lib):
    from paper_2510_24175_b200 import mhd
    syms = declared_symbols()
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(mhd.EXPORTS)


def test_version(lib):
    from paper_2510_24175_b200 import mhd
    assert "sm_100a" in mhd.version()


def test_create_rejects_bad_arguments_without_gpu(lib):
    from paper_2510_24175_b200 import mhd
    from paper_2510_24175_b200 import inputs as I
    g, bc = mhd.Grid(), mhd.BC()
    for d in range(3):
        g.n[d], g.lo[d], g.hi[d] = 16, 0.0, 1.0
    h = C.c_void_p()
    # cfl out of (0,1), gamma <= 1, inactive-axis gap, n < 4, lo >= hi
    assert lib.mhd_create(C.byref(g), 5 / 3, 1.2, C.byref(bc), None, None, C.byref(h)) == mhd.MHD_E_ARG
    assert lib.mhd_create(C.byref(g), 1.0, 0.4, C.byref(bc), None, None, C.byref(h)) == mhd.MHD_E_ARG
    g2 = mhd.Grid()
    for d, n in enumerate((16, 1, 16)):
        g2.n[d], g2.lo[d], g2.hi[d] = n, 0.0, 1.0
    assert lib.mhd_create(C.byref(g2), 5 / 3, 0.4, C.byref(bc), None, None, C.byref(h)) == mhd.MHD_E_ARG
    g3 = mhd.Grid()
    for d, n in enumerate((3, 1, 1)):
        g3.n[d], g3.lo[d], g3.hi[d] = n, 0.0, 1.0
    assert lib.mhd_create(C.byref(g3), 5 / 3, 0.4, C.byref(bc), None, None, C.byref(h)) == mhd.MHD_E_ARG
    g.hi[1] = 0.0
    assert lib.mhd_create(C.byref(g), 5 / 3, 0.4, C.byref(bc), None, None, C.byref(h)) == mhd.MHD_E_ARG
    g.hi[1] = 1.0
    sc = mhd.Scheme(1, 1, 0, 0, 0.1, 1e-12, 0, 0)  # no GLM in 3D
    assert lib.mhd_create(C.byref(g), 5 / 3, 0.4, C.byref(bc), C.byref(sc), None, C.byref(h)) == mhd.MHD_E_ARG
    sc = mhd.Scheme(1, 1, 1, 0, 0.1, 1e-12, 1, 0)  # CT together with GLM
    assert lib.mhd_create(C.byref(g), 5 / 3, 0.4, C.byref(bc), C.byref(sc), None, C.byref(h)) == mhd.MHD_E_ARG
    d = mhd.Dist(0, 3, -1, 0)                # 3 ranks do not divide nz = 16
    assert lib.mhd_create(C.byref(g), 5 / 3, 0.4, C.byref(bc), None, C.byref(d), C.byref(h)) == mhd.MHD_E_ARG
    g4 = mhd.Grid()                          # nx * ny * 9 >= 2^31 (32-bit in-plane offsets)
    for dd, n in enumerate((16384, 16384, 8)):
        g4.n[dd], g4.lo[dd], g4.hi[dd] = n, 0.0, 1.0
    assert lib.mhd_create(C.byref(g4), 5 / 3, 0.4, C.byref(bc), None, None, C.byref(h)) == mhd.MHD_E_ARG
    bc.lo[0] = 1                             # periodic on one side only
    assert lib.mhd_create(C.byref(g), 5 / 3, 0.4, C.byref(bc), None, None, C.byref(h)) == mhd.MHD_E_ARG
    assert h.value is None
    assert lib.mhd_create(None, 5 / 3, 0.4, None, None, None, C.byref(h)) == mhd.MHD_E_ARG
    lib.mhd_destroy(None)  # NULL-safe
    lib.mhd_halo_push.argtypes = [C.c_void_p]
    assert lib.mhd_halo_push(None) == mhd.MHD_E_ARG


def test_product_package_does_not_import_the_oracle():
    pkg = os.path.join(ROOT, "paper_2510_24175_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            path = os.path.join(dirpath, fn)
            if fn.endswith(".py"):
                tree = ast.parse(open(path).read())
                for node in ast.walk(tree):
                    if isinstance(node, ast.Import):
                        assert not any(a.name.split(".")[0] == "oracle" for a in node.names), path
                    if isinstance(node, ast.ImportFrom):
                        assert (node.module or "").split(".")[0] != "oracle", path
            if fn.endswith((".cu", ".cuh", ".h", ".cpp")):
                assert "mhd_oracle" not in open(path).read(), path
    # and the oracle does not include the CUDA path
    assert "paper_2510_24175_b200" not in open(os.path.join(ROOT, "oracle", "mhd_oracle.c")).read()
