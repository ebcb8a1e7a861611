"""CPU checks of the boundary: libbsct.so builds/loads and exports every entry point
declared in include/bsct.h (no compute calls without a GPU), the Python binding
mirrors the C names, and argument validation that needs no device."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "bsct.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(bsct_[a-z_]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    import paper_2005_13471_b200 as bsct
    from paper_2005_13471_b200 import build
    if not os.path.exists(bsct.LIB_PATH):
        build.build()
    return bsct.load()


def test_header_declares_the_hot_path():
    syms = header_symbols()
    for s in ("bsct_gram_build", "bsct_backproject", "bsct_normal_apply", "bsct_cg_solve", "bsct_plan_create"):
        assert s in syms


def test_library_exports_every_symbol(lib):
    import paper_2005_13471_b200 as bsct
    syms = header_symbols()
    assert sorted(bsct.SYMBOLS) == syms
    for s in syms:
        assert hasattr(lib, s), s


def test_no_torch_in_header():
    txt = open(os.path.join(ROOT, "include", "bsct.h")).read()
    assert "torch" not in txt.replace("torch tensors", "") and "at::" not in txt


def test_host_only_calls(lib):
    import paper_2005_13471_b200 as bsct
    assert bsct.version() >= 100
    assert [bsct.fft_size(n) for n in (1, 2, 5, 64, 256, 512, 1024)] == [2, 4, 16, 128, 512, 1024, 2048]


def test_validation_without_device(lib):
    """Invalid geometries fail with BSCT_EINVAL before touching the device."""
    import paper_2005_13471_b200 as bsct
    ang = np.zeros(4)
    for bad in (dict(N=0), dict(lambda_x=0.0), dict(lambda_y=-1.0), dict(zeta=-0.5), dict(n_det=0)):
        g = dict(N=4, lambda_x=1.0, angles=ang, lambda_y=1.0, n_det=9, zeta=0.0)
        g.update(bad)
        s, keep = bsct._geom(g)
        st = lib.bsct_gram_build(ctypes.byref(s), bsct.F32, 0, 4, ctypes.c_void_p(1), None)
        assert st == bsct.EINVAL
        assert lib.bsct_last_error()
    g = dict(N=4, lambda_x=1.0, angles=np.array([0.0, np.nan]), lambda_y=1.0, n_det=9, zeta=0.0)
    s, keep = bsct._geom(g)
    assert lib.bsct_gram_build(ctypes.byref(s), bsct.F32, 0, 2, ctypes.c_void_p(1), None) == bsct.EINVAL
    g = dict(N=4, lambda_x=1.0, angles=ang, lambda_y=1.0, n_det=9, zeta=0.0)
    s, keep = bsct._geom(g)
    assert lib.bsct_gram_build(ctypes.byref(s), bsct.F32, 3, 2, ctypes.c_void_p(1), None) == bsct.EINVAL
    assert lib.bsct_gram_build(ctypes.byref(s), bsct.F32, 0, 5, ctypes.c_void_p(1), None) == bsct.EINVAL
    assert lib.bsct_gram_build(ctypes.byref(s), bsct.F32, 0, 4, None, None) == bsct.EINVAL
    assert lib.bsct_plan_destroy(None) == bsct.OK
    assert lib.bsct_backproject(None, None, None, 1, None) == bsct.EINVAL


def test_null_plan_rejected_everywhere(lib):
    """Every plan-taking entry point rejects a NULL plan with BSCT_EINVAL (no device work)."""
    import paper_2005_13471_b200 as bsct
    vp = ctypes.c_void_p
    calls = [
        lambda: lib.bsct_correction_filter(None, vp(1), vp(1), 1, None),
        lambda: lib.bsct_normal_apply(None, vp(1), vp(1), 1, None),
        lambda: lib.bsct_cg_solve(None, vp(1), vp(1), 1, 3, 0, None, None, None),
        lambda: lib.bsct_forward_project(None, vp(1), vp(1), 1, None),
        lambda: lib.bsct_reconstruct(None, vp(1), vp(1), 1, 3, 0, None, None, None),
        lambda: lib.bsct_reconstruct_host(None, vp(1), vp(1), 1, 3, 0, None),
        lambda: lib.bsct_adjoint_project(None, vp(1), vp(1), 1, None),
        lambda: lib.bsct_sirt_solve(None, vp(1), vp(1), 1, 3, None),
        lambda: lib.bsct_chebyshev_solve(None, vp(1), vp(1), 1, 3, 0.1, 1.0, None, None),
        lambda: lib.bsct_plan_set_filter(None, vp(1), None),
        lambda: lib.bsct_plan_profile(None, 1),
    ]
    for c in calls:
        assert c() == bsct.EINVAL
        assert b"plan" in lib.bsct_last_error()


def test_plan_create_rejects_oversized_batch(lib):
    """max_batch > 65535 (the batched kernels' grid limit) fails with BSCT_EINVAL before any
    device work; so does a negative one."""
    import paper_2005_13471_b200 as bsct
    g = dict(N=4, lambda_x=1.0, angles=np.zeros(4), lambda_y=1.0, n_det=9, zeta=0.0)
    s, keep = bsct._geom(g)
    out = ctypes.c_void_p()
    for mb in (70000, -1):
        assert lib.bsct_plan_create(ctypes.byref(s), bsct.F32, ctypes.c_void_p(1), mb, ctypes.byref(out), None) == bsct.EINVAL
        assert b"max_batch" in lib.bsct_last_error()
