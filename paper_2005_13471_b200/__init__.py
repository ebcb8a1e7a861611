"""paper_2005_13471_b200 -- B200-native box-spline parallel-beam CT hot path.

Thin ctypes binding of the C ABI in include/bsct.h (libbsct.so, built in-tree by
paper_2005_13471_b200/build.py).  Names mirror the C entry points without the
``bsct_`` prefix.  This module only marshals arguments: torch tensors are passed as
raw device pointers together with torch's current CUDA stream; every computation
runs in the library's sm_100a kernels.  There is no CPU fallback: if libbsct.so
cannot be loaded, every call raises.

    import paper_2005_13471_b200 as bsct
    geom = dict(N=512, lambda_x=1.0, angles=angles, lambda_y=1.0, n_det=725, zeta=1.0)
    taps = torch.empty((2*512-1, 2*512-1), device="cuda")
    bsct.gram_build(geom, taps)                       # (a) Gram filter
    plan = bsct.plan_create(geom, taps, max_batch=B)  # spectrum + tables + workspace
    bsct.backproject(plan, sino, b)                   # (b) H^T g^
    bsct.cg_solve(plan, b, x, iters=50)               # (c) CG on G x = b
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libbsct.so")

OK, EINVAL, ECUDA, ENOMEM, EBREAKDOWN, ESHAPE = 0, -1, -2, -3, -4, -5
F32, F64 = 0, 1
CG, SD, LANDWEBER = 0, 1, 2
SOLVERS = {"cg": CG, "sd": SD, "landweber": LANDWEBER}
H_CORR = 25

# exported symbols of include/bsct.h (checked by tests/test_abi.py)
SYMBOLS = ("bsct_version", "bsct_last_error", "bsct_fft_size", "bsct_gram_build", "bsct_plan_create",
           "bsct_plan_destroy", "bsct_plan_set_filter", "bsct_plan_spectrum", "bsct_correction_filter", "bsct_backproject",
           "bsct_normal_apply", "bsct_cg_solve", "bsct_cg_resume", "bsct_forward_project", "bsct_reconstruct", "bsct_reconstruct_host",
           "bsct_adjoint_project", "bsct_sirt_solve", "bsct_chebyshev_solve",
           "bsct_plan_launch_count", "bsct_plan_profile", "bsct_plan_profile_read")

# bsct_kernel_class
KERNEL_CLASSES = ("tables", "spectrum", "correction", "backproject", "pass_a", "pass_b", "pass_c",
                  "solver_init", "solver_update", "solver_finish", "forward", "fused_cg")


class BsctError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"bsct status {status}: {msg}")
        self.status = status


class Geometry(ctypes.Structure):
    _fields_ = [("N", ctypes.c_int32), ("lambda_x", ctypes.c_double), ("n_angles", ctypes.c_int32),
                ("angles", ctypes.POINTER(ctypes.c_double)), ("lambda_y", ctypes.c_double),
                ("n_det", ctypes.c_int32), ("zeta_blur", ctypes.c_double)]


_lib = None


def load(path: str | None = None):
    """Load libbsct.so (raises if it is missing: there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    p = path or os.environ.get("BSCT_LIB") or LIB_PATH  # BSCT_LIB: A/B builds (tools/)
    if not os.path.exists(p):
        raise ImportError(f"{p} not found -- build it with `python -m paper_2005_13471_b200.build`")
    lib = ctypes.CDLL(p)
    vp, i32, i64, dp = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    G = ctypes.POINTER(Geometry)
    sig = {
        "bsct_version": (i32, []),
        "bsct_last_error": (ctypes.c_char_p, []),
        "bsct_fft_size": (i32, [i32]),
        "bsct_gram_build": (i32, [G, i32, i32, i32, vp, vp]),
        "bsct_plan_create": (i32, [G, i32, vp, i32, ctypes.POINTER(vp), vp]),
        "bsct_plan_destroy": (i32, [vp]),
        "bsct_plan_set_filter": (i32, [vp, vp, vp]),
        "bsct_plan_spectrum": (i32, [vp, vp, vp]),
        "bsct_correction_filter": (i32, [vp, vp, vp, i32, vp]),
        "bsct_backproject": (i32, [vp, vp, vp, i32, vp]),
        "bsct_normal_apply": (i32, [vp, vp, vp, i32, vp]),
        "bsct_cg_solve": (i32, [vp, vp, vp, i32, i32, i32, vp, vp, vp]),
        "bsct_cg_resume": (i32, [vp, vp, vp, vp, i32, i32, i32, vp, vp, vp, vp]),
        "bsct_forward_project": (i32, [vp, vp, vp, i32, vp]),
        "bsct_reconstruct": (i32, [vp, vp, vp, i32, i32, i32, vp, vp, vp]),
        "bsct_adjoint_project": (i32, [vp, vp, vp, i32, vp]),
        "bsct_sirt_solve": (i32, [vp, vp, vp, i32, i32, vp]),
        "bsct_chebyshev_solve": (i32, [vp, vp, vp, i32, i32, dp, dp, vp, vp]),
        "bsct_reconstruct_host": (i32, [vp, vp, vp, i32, i32, i32, vp]),
        "bsct_plan_launch_count": (i64, [vp]),
        "bsct_plan_profile": (i32, [vp, i32]),
        "bsct_plan_profile_read": (i32, [vp, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64), i32]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def _check(st: int):
    if st != OK:
        raise BsctError(st, load().bsct_last_error().decode())


def version() -> int:
    return load().bsct_version()


def fft_size(N: int) -> int:
    return load().bsct_fft_size(N)


def _geom(g: dict):
    ang = np.ascontiguousarray(np.asarray(g["angles"], dtype=np.float64))
    s = Geometry(int(g["N"]), float(g.get("lambda_x", 1.0)), int(ang.size),
                 ang.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), float(g.get("lambda_y", 1.0)),
                 int(g["n_det"]), float(g.get("zeta", g.get("zeta_blur", 0.0))))
    return s, ang  # keep `ang` alive for the call


def _stream(stream=None):
    import torch
    st = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(st.cuda_stream)


def _dt(t) -> int:
    import torch
    if t.dtype == torch.float32:
        return F32
    if t.dtype == torch.float64:
        return F64
    raise TypeError(f"unsupported dtype {t.dtype}")


def _ptr(t, dtype=None, numel=None, name="tensor"):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if dtype is not None and t.dtype != dtype:
        raise TypeError(f"{name} has dtype {t.dtype}, expected {dtype}")
    if numel is not None and t.numel() < numel:
        raise ValueError(f"{name} has {t.numel()} elements, needs {numel}")
    return ctypes.c_void_p(t.data_ptr())


def gram_build(geom: dict, taps, angle_begin: int = 0, angle_end: int | None = None, stream=None):
    """(a) taps[(2N-1),(2N-1)] <- Gram filter over angles [angle_begin, angle_end)."""
    lib = load()
    g, keep = _geom(geom)
    N = g.N
    end = g.n_angles if angle_end is None else angle_end
    _check(lib.bsct_gram_build(ctypes.byref(g), _dt(taps), angle_begin, end,
                               _ptr(taps, numel=(2 * N - 1) ** 2, name="taps"), _stream(stream)))
    return taps


class Plan:
    """Owning handle of a bsct_plan (destroyed with the object)."""

    def __init__(self, handle, geom: dict, dtype, max_batch: int):
        self.handle = handle
        self.geom = dict(geom)
        self.dtype = dtype
        self.N = int(geom["N"])
        self.n_angles = len(geom["angles"])
        self.n_det = int(geom["n_det"])
        self.max_batch = max_batch
        self.L = fft_size(self.N)

    def close(self):
        if self.handle:
            load().bsct_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def launches(self) -> int:
        return int(load().bsct_plan_launch_count(self.handle))

    def profile(self, enable: bool = True):
        """Bracket every launch of this plan with CUDA events (see bsct_plan_profile)."""
        _check(load().bsct_plan_profile(self.handle, int(bool(enable))))

    def profile_read(self) -> dict:
        """{kernel class: (device ms, bracket count)} since the last read (synchronises)."""
        n = len(KERNEL_CLASSES)
        ms = (ctypes.c_double * n)()
        cnt = (ctypes.c_int64 * n)()
        _check(load().bsct_plan_profile_read(self.handle, ms, cnt, n))
        return {k: (ms[i], cnt[i]) for i, k in enumerate(KERNEL_CLASSES) if cnt[i]}


def plan_create(geom: dict, taps, max_batch: int = 1, stream=None) -> Plan:
    lib = load()
    g, keep = _geom(geom)
    h = ctypes.c_void_p()
    _check(lib.bsct_plan_create(ctypes.byref(g), _dt(taps), _ptr(taps, numel=(2 * g.N - 1) ** 2, name="taps"),
                                int(max_batch), ctypes.byref(h), _stream(stream)))
    return Plan(h, geom, taps.dtype, int(max_batch))


def plan_destroy(plan: Plan):
    plan.close()


def _batch(t, per: int, name: str) -> int:
    if t.numel() % per:
        raise ValueError(f"{name}: {t.numel()} elements is not a multiple of {per}")
    return t.numel() // per


def plan_set_filter(plan: Plan, taps, stream=None):
    """Rebuild the plan's tables and filter spectrum from taps (no reallocation, async)."""
    _check(load().bsct_plan_set_filter(plan.handle, _ptr(taps, plan.dtype, (2 * plan.N - 1) ** 2, "taps"),
                                       _stream(stream)))
    return plan


def plan_spectrum(plan: Plan, out, stream=None):
    _check(load().bsct_plan_spectrum(plan.handle, _ptr(out, plan.dtype, (plan.L // 2 + 1) * plan.L, "out"),
                                     _stream(stream)))
    return out


def correction_filter(plan: Plan, sino, g_tilde, stream=None):
    B = _batch(sino, plan.n_angles * plan.n_det, "sino")
    _check(load().bsct_correction_filter(plan.handle, _ptr(sino, plan.dtype, name="sino"),
                                         _ptr(g_tilde, plan.dtype, B * plan.n_angles * (plan.n_det + 2 * H_CORR),
                                              "g_tilde"), B, _stream(stream)))
    return g_tilde


def backproject(plan: Plan, sino, b, stream=None):
    """(b) b[B,N,N] <- H^T g^ of sino[B, n_angles, n_det]."""
    B = _batch(sino, plan.n_angles * plan.n_det, "sino")
    _check(load().bsct_backproject(plan.handle, _ptr(sino, plan.dtype, name="sino"),
                                   _ptr(b, plan.dtype, B * plan.N * plan.N, "b"), B, _stream(stream)))
    return b


def normal_apply(plan: Plan, x, y, stream=None):
    """(c) y <- G x for x[B,N,N]."""
    B = _batch(x, plan.N * plan.N, "x")
    _check(load().bsct_normal_apply(plan.handle, _ptr(x, plan.dtype, name="x"),
                                    _ptr(y, plan.dtype, B * plan.N * plan.N, "y"), B, _stream(stream)))
    return y


def cg_solve(plan: Plan, b, x, iters: int, solver="cg", resid_hist=None, flags=None, stream=None):
    """x[B,N,N] <- `iters` iterations of CG / SD / Landweber on G x = b from x = 0."""
    import torch
    B = _batch(b, plan.N * plan.N, "b")
    sv = SOLVERS[solver] if isinstance(solver, str) else int(solver)
    _check(load().bsct_cg_solve(plan.handle, _ptr(b, plan.dtype, name="b"),
                                _ptr(x, plan.dtype, B * plan.N * plan.N, "x"), B, int(iters), sv,
                                _ptr(resid_hist, torch.float64, B * iters, "resid_hist"),
                                _ptr(flags, torch.int32, B, "flags"), _stream(stream)))
    return x


def cg_resume(plan: Plan, x, r, p, iters: int, solver="cg", alpha_last=None, resid_hist=None, flags=None,
              stream=None):
    """Continue a solve from the state (x_j, r_j, p_j) for `iters` iterations; x, r, p are
    updated in place to the final state (p: CG only, None for SD / Landweber)."""
    import torch
    B = _batch(x, plan.N * plan.N, "x")
    sv = SOLVERS[solver] if isinstance(solver, str) else int(solver)
    n = B * plan.N * plan.N
    _check(load().bsct_cg_resume(plan.handle, _ptr(x, plan.dtype, n, "x"), _ptr(r, plan.dtype, n, "r"),
                                 _ptr(p, plan.dtype, n, "p"), B, int(iters), sv,
                                 _ptr(alpha_last, torch.float64, B, "alpha_last"),
                                 _ptr(resid_hist, torch.float64, B * iters, "resid_hist"),
                                 _ptr(flags, torch.int32, B, "flags"), _stream(stream)))
    return x, r, p


def reconstruct(plan: Plan, sino, x, iters: int, solver="cg", resid_hist=None, flags=None, stream=None):
    """x[B,N,N] <- back projection of sino[B,n_angles,n_det], then `iters` solver iterations
    (device tensors; slice chunks pipelined inside the library)."""
    import torch
    B = _batch(sino, plan.n_angles * plan.n_det, "sino")
    sv = SOLVERS[solver] if isinstance(solver, str) else int(solver)
    _check(load().bsct_reconstruct(plan.handle, _ptr(sino, plan.dtype, name="sino"),
                                   _ptr(x, plan.dtype, B * plan.N * plan.N, "x"), B, int(iters), sv,
                                   _ptr(resid_hist, torch.float64, B * iters, "resid_hist"),
                                   _ptr(flags, torch.int32, B, "flags"), _stream(stream)))
    return x


def chebyshev_solve(plan: Plan, b, x, iters: int, lambda_min: float, lambda_max: float = 0.0,
                    resid_hist=None, stream=None):
    """x[B,N,N] <- `iters` Chebyshev semi-iterations on G x = b (spectrum in [lambda_min,
    lambda_max]; lambda_max <= 0: the plan's embedding-spectrum bound)."""
    import torch
    B = _batch(b, plan.N * plan.N, "b")
    _check(load().bsct_chebyshev_solve(plan.handle, _ptr(b, plan.dtype, name="b"),
                                       _ptr(x, plan.dtype, B * plan.N * plan.N, "x"), B, int(iters),
                                       float(lambda_min), float(lambda_max),
                                       _ptr(resid_hist, torch.float64, B * iters, "resid_hist"), _stream(stream)))
    return x


def adjoint_project(plan: Plan, sino, img, stream=None):
    """img[B,N,N] <- H^T sino (plain adjoint of forward_project; SIRT's back projection)."""
    B = _batch(sino, plan.n_angles * plan.n_det, "sino")
    _check(load().bsct_adjoint_project(plan.handle, _ptr(sino, plan.dtype, name="sino"),
                                       _ptr(img, plan.dtype, B * plan.N * plan.N, "img"), B, _stream(stream)))
    return img


def sirt_solve(plan: Plan, sino, x, iters: int, stream=None):
    """x[B,N,N] <- `iters` SIRT iterations on sino[B,n_angles,n_det] from x = 0."""
    B = _batch(sino, plan.n_angles * plan.n_det, "sino")
    _check(load().bsct_sirt_solve(plan.handle, _ptr(sino, plan.dtype, name="sino"),
                                  _ptr(x, plan.dtype, B * plan.N * plan.N, "x"), B, int(iters), _stream(stream)))
    return x


def forward_project(plan: Plan, c, sino, stream=None):
    """sino[B, n_angles, n_det] <- H c (Eq.(3)/(4))."""
    B = _batch(c, plan.N * plan.N, "c")
    _check(load().bsct_forward_project(plan.handle, _ptr(c, plan.dtype, name="c"),
                                       _ptr(sino, plan.dtype, B * plan.n_angles * plan.n_det, "sino"), B,
                                       _stream(stream)))
    return sino


def reconstruct_host(plan: Plan, sino_host, x_host, iters: int, solver="cg", stream=None):
    """End to end from HOST tensors (pinned preferred): H2D, back projection, solver, D2H."""
    if sino_host.is_cuda or x_host.is_cuda:
        raise ValueError("reconstruct_host takes host tensors")
    if not (sino_host.is_contiguous() and x_host.is_contiguous()):
        raise ValueError("host tensors must be contiguous")
    if sino_host.dtype != plan.dtype or x_host.dtype != plan.dtype:
        raise TypeError("host tensors must have the plan dtype")
    B = _batch(sino_host, plan.n_angles * plan.n_det, "sino_host")
    if x_host.numel() < B * plan.N * plan.N:
        raise ValueError("x_host too small")
    sv = SOLVERS[solver] if isinstance(solver, str) else int(solver)
    _check(load().bsct_reconstruct_host(plan.handle, ctypes.c_void_p(sino_host.data_ptr()),
                                        ctypes.c_void_p(x_host.data_ptr()), B, int(iters), sv, _stream(stream)))
    return x_host
