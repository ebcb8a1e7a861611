"""Geometric pixel footprints: the brute-force side of the oracle's pins.

The X-ray transform of one pixel (indicator of a square of side lambda_x, P:22, P:66
"pixel-basis coincides with two directions bivariate box spline") is computed here
WITHOUT box splines: chord lengths of the line {<theta_perp, x> = y} through the
square by slab clipping (as in Siddon), and the detector blur of
P:24 ((1/zeta) box(./zeta) * P_theta) by exact piecewise integration of the chord
(the chord is linear between the projections of the square's corners, so 2-point
Gauss-Legendre per piece is exact).
"""
from __future__ import annotations

import numpy as np

_GL2 = np.polynomial.legendre.leggauss(2)
_GL3 = np.polynomial.legendre.leggauss(3)


def chord(y, t: float, centre, lam: float) -> np.ndarray:
    """Length of {x in square(centre, lam) : <(-sin t, cos t), x> = y}, vectorised in y."""
    y = np.asarray(y, dtype=np.float64)
    n = np.array([-np.sin(t), np.cos(t)])
    d = np.array([np.cos(t), np.sin(t)])
    tlo = np.full(y.shape, -np.inf)
    thi = np.full(y.shape, np.inf)
    for ax in range(2):
        lo, hi = centre[ax] - 0.5 * lam, centre[ax] + 0.5 * lam
        p = y * n[ax]                      # point of the line at parameter 0
        if abs(d[ax]) < 1e-300:
            inside = (p >= lo) & (p <= hi)
            tlo = np.where(inside, tlo, np.inf)
            thi = np.where(inside, thi, -np.inf)
        else:
            a, b = (lo - p) / d[ax], (hi - p) / d[ax]
            tlo = np.maximum(tlo, np.minimum(a, b))
            thi = np.minimum(thi, np.maximum(a, b))
    return np.maximum(thi - tlo, 0.0)


def corner_projections(t: float, centre, lam: float) -> np.ndarray:
    n = np.array([-np.sin(t), np.cos(t)])
    cs = [(centre[0] + sx * 0.5 * lam, centre[1] + sy * 0.5 * lam) for sx in (-1, 1) for sy in (-1, 1)]
    return np.sort(np.array([n[0] * a + n[1] * b for a, b in cs]))


def chord_integral(lo, hi, t: float, centre, lam: float) -> np.ndarray:
    """int_lo^hi chord(y) dy exactly (chord linear between corner projections)."""
    lo = np.asarray(lo, dtype=np.float64)
    hi = np.asarray(hi, dtype=np.float64)
    cp = corner_projections(t, centre, lam)
    pts = [lo] + [np.clip(c, lo, hi) for c in cp] + [hi]
    total = np.zeros(np.broadcast(lo, hi).shape)
    xg, wg = _GL2
    for a, b in zip(pts[:-1], pts[1:]):
        h = 0.5 * (b - a)
        m = 0.5 * (a + b)
        for xi, wi in zip(xg, wg):
            total = total + wi * h * chord(m + h * xi, t, centre, lam)
    return total


def footprint(y, t: float, centre, lam: float, zeta: float) -> np.ndarray:
    """F(y) = ((1/zeta) box(./zeta) * P_theta 1_square)(y); zeta = 0: the chord."""
    if zeta <= 0:
        return chord(y, t, centre, lam)
    y = np.asarray(y, dtype=np.float64)
    return chord_integral(y - 0.5 * zeta, y + 0.5 * zeta, t, centre, lam) / zeta


def footprint_breakpoints(t: float, centre, lam: float, zeta: float) -> np.ndarray:
    cp = corner_projections(t, centre, lam)
    if zeta <= 0:
        return cp
    return np.sort(np.concatenate([cp - 0.5 * zeta, cp + 0.5 * zeta]))


def footprint_inner(t: float, ci, cj, lam: float, zeta: float) -> float:
    """int F_i(y) F_j(y) dy, exact: both are piecewise polynomials of degree <= 2
    between the merged breakpoints, so 3-point Gauss-Legendre per piece is exact."""
    bi = footprint_breakpoints(t, ci, lam, zeta)
    bj = footprint_breakpoints(t, cj, lam, zeta)
    lo, hi = max(bi[0], bj[0]), min(bi[-1], bj[-1])
    if hi <= lo:
        return 0.0
    br = np.unique(np.concatenate([[lo, hi], bi[(bi > lo) & (bi < hi)], bj[(bj > lo) & (bj < hi)]]))
    a, b = br[:-1], br[1:]
    h = 0.5 * (b - a)
    m = 0.5 * (a + b)
    xg, wg = _GL3
    ys = (m[:, None] + h[:, None] * xg[None, :]).ravel()
    ws = (h[:, None] * wg[None, :]).ravel()
    return float(np.sum(ws * footprint(ys, t, ci, lam, zeta) * footprint(ys, t, cj, lam, zeta)))
