"""Iterative solvers for G x = b, FP64 (BASELINE.json north_star).

P:34: "execute iterative reconstruction with a single back projection, H^T g^_psi, at the
beginning and apply the filter in every iteration" -- b = H^T g^ once, then each
iteration applies G (normal.py).  All solvers start from x = 0.

cg         conjugate gradients (north_star "CG/Landweber loop"), textbook form:
             r0 = b, p0 = r0; alpha = <r,r>/<p,Gp>; x += alpha p; r -= alpha Gp;
             beta = <r',r'>/<r,r>; p = r' + beta p.
sd         steepest descent with exact line search, the paper's solver:
             q = G r; alpha = <r,r>/<r,q>; x += alpha r; r -= alpha q.
landweber  x += tau r; r -= tau G r, tau = 1/max(embedding spectrum) (DESIGN.md R-LW).
Each returns (x, history) where history[k] = ||r_k|| after iteration k.  A zero
residual stops updating (alpha = 0); <p,Gp> <= 0 with r != 0 raises.
"""
from __future__ import annotations

import numpy as np

from .normal import apply_direct, apply_fft, embed_spectrum


def _apply(taps, x, direct):
    return apply_direct(taps, x) if direct else apply_fft(taps, x)


def cg(taps, b, iters: int, direct: bool = False, record=None):
    b = np.asarray(b, dtype=np.float64)
    x = np.zeros_like(b)
    r = b.copy()
    p = r.copy()
    rr = float(np.vdot(r, r))
    hist = []
    for k in range(iters):
        if rr == 0.0:
            hist.append(0.0)
            continue
        q = _apply(taps, p, direct)
        pq = float(np.vdot(p, q))
        if pq <= 0.0:
            raise FloatingPointError("CG breakdown: <p, Gp> <= 0")
        alpha = rr / pq
        x = x + alpha * p
        r = r - alpha * q
        rr_new = float(np.vdot(r, r))
        p = r + (rr_new / rr) * p
        rr = rr_new
        hist.append(np.sqrt(rr))
        if record is not None:  # state after this iteration (R12 check (ii) resumes from it)
            record.append(dict(alpha=alpha, x=x.copy(), r=r.copy(), p=p.copy(), rr=rr))
    return x, np.array(hist)


def sd(taps, b, iters: int, direct: bool = False):
    b = np.asarray(b, dtype=np.float64)
    x = np.zeros_like(b)
    r = b.copy()
    hist = []
    for k in range(iters):
        rr = float(np.vdot(r, r))
        if rr == 0.0:
            hist.append(0.0)
            continue
        q = _apply(taps, r, direct)
        rq = float(np.vdot(r, q))
        if rq <= 0.0:
            raise FloatingPointError("SD breakdown: <r, Gr> <= 0")
        alpha = rr / rq
        x = x + alpha * r
        r = r - alpha * q
        hist.append(np.sqrt(float(np.vdot(r, r))))
    return x, np.array(hist)


def landweber_tau(taps) -> float:
    return 1.0 / float(embed_spectrum(taps).max())


def landweber(taps, b, iters: int, tau: float | None = None, direct: bool = False):
    b = np.asarray(b, dtype=np.float64)
    tau = landweber_tau(taps) if tau is None else tau
    x = np.zeros_like(b)
    r = b.copy()
    hist = []
    for k in range(iters):
        q = _apply(taps, r, direct)
        x = x + tau * r
        r = r - tau * q
        hist.append(np.sqrt(float(np.vdot(r, r))))
    return x, np.array(hist)


def objective(taps, b, x) -> float:
    """f(x) = 1/2 <x, Gx> - <b, x> (monotone in CG/SD; SURVEY.md R12 guard)."""
    return 0.5 * float(np.vdot(x, apply_fft(taps, x))) - float(np.vdot(b, x))


def chebyshev(taps, b, iters: int, lmin: float, lmax: float, direct: bool = False):
    """Chebyshev semi-iteration for G x = b with spectrum assumed in [lmin, lmax] (SURVEY.md
    8(f) NEXT-4; Saad, Iterative Methods for Sparse Linear Systems, 2nd ed., Alg. 12.1):
        theta = (lmax + lmin)/2, delta = (lmax - lmin)/2, sigma = theta/delta,
        x0 = 0, r0 = b, rho0 = 1/sigma, d0 = r0/theta;
        x_{k+1} = x_k + d_k, r_{k+1} = r_k - G d_k,
        rho_{k+1} = 1/(2 sigma - rho_k), d_{k+1} = rho_{k+1} rho_k d_k + (2 rho_{k+1}/delta) r_{k+1}.
    No inner products: x_k is a fixed polynomial in G applied to b (linear in b)."""
    b = np.asarray(b, dtype=np.float64)
    theta, delta = 0.5 * (lmax + lmin), 0.5 * (lmax - lmin)
    sigma = theta / delta
    x = np.zeros_like(b)
    r = b.copy()
    rho = 1.0 / sigma
    d = r / theta
    hist = []
    for _ in range(iters):
        x = x + d
        r = r - _apply(taps, d, direct)
        rho_n = 1.0 / (2.0 * sigma - rho)
        d = rho_n * rho * d + (2.0 * rho_n / delta) * r
        rho = rho_n
        hist.append(np.sqrt(float(np.vdot(r, r))))
    return x, np.array(hist)
