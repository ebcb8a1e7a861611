"""Interpolated back projection H^T g^_psi (section 5).

Algorithm, per angle theta in the given order:
 1. degree d of the interpolating B-spline from the continuity of g_psi:
      no blur: C^0 -> d = 1; axis-aligned C^-1 -> d = 0; blur: C^1 / C^0 -> d = 2 / 1.
    i.e. d = #nonzero{lambda_x|cos|, lambda_x|sin|, zeta} - 1 (R9).
 2. correction filter q (Eq.(5)): Q(z) = 1/sum_m b[m] z^-m with
    b[m] = <delta(y-m), B(y)>; q = delta for d <= 1; for d = 2
    q[m] = sqrt(2)(2 sqrt(2) - 3)^|m| (P:150 with reading R7: the sqrt(2) makes
    q * [1/8, 6/8, 1/8] = delta and reproduces the paper's q[40] = 3.38e-31),
    truncated to |m| <= h = 25 ("truncated"; R8), applied as a zero-extended
    full linear convolution: g~ = g_s * q has M + 2h samples at y_{-h} .. y_{M+h-1}.
 3. interpolant g^(y) = sum_m g~[m] B_d((y - y_m)/lambda_y) (R10 for lambda_y).
 4. H^T: b[k] += int g^(y) F_k(y) dy with the pixel footprint
    F_k(y) = lambda_x^2 M_[lambda_x|c|, lambda_x|s|, zeta](y - k_theta) (Eq.(4), R1, R3).
    Since B_d(u/lambda_y) = lambda_y M_[lambda_y]^(d+1)(u) and box splines are closed
    under convolution (Eq.(1)), the integral is the closed form
      b[k] += lambda_x^2 lambda_y sum_m g~[m] M_[lambda|c|, lambda|s|, zeta] U [lambda_y]^(d+1)(y_m - k_theta)
    (SPEC S:216-218).  backproject_quadrature evaluates step 4 by numerical
    integration of the explicit interpolant instead (pin in tests).
"""
from __future__ import annotations

import numpy as np

from .boxspline import box_spline, kept_widths
from .geometry import as_geometry

H_CORR = 25


def interpolation_degree(geom, t: float) -> int:
    g = as_geometry(geom)
    return len(kept_widths(g.blurred_widths(t))) - 1


def correction_filter(d: int, h: int = H_CORR) -> np.ndarray:
    """q[-h..h] (Eq.(5))."""
    m = np.arange(-h, h + 1)
    if d <= 1:
        return (m == 0).astype(np.float64)
    if d == 2:
        z = 2.0 * np.sqrt(2.0) - 3.0
        return np.sqrt(2.0) * z ** np.abs(m)
    raise ValueError("unsupported B-spline degree")


def corrected_row(g_row: np.ndarray, d: int, h: int = H_CORR) -> np.ndarray:
    """g~ on detector indices -h .. M+h-1 (zero-extended full linear convolution)."""
    M = g_row.shape[-1]
    out = np.zeros(M + 2 * h)
    if d <= 1:
        out[h:h + M] = g_row
        return out
    return np.convolve(g_row, correction_filter(d, h))   # length M + 2h, index 0 <-> m = -h


def bp_widths(geom, t: float) -> list[float]:
    g = as_geometry(geom)
    d = interpolation_degree(g, t)
    return g.blurred_widths(t) + [g.lambda_y] * (d + 1)


def backproject(geom, sino: np.ndarray, pixels=None) -> np.ndarray:
    """b = H^T g^_psi, FP64.  sino: [n_angles, M].  pixels: optional (k1, k2) index arrays
    to evaluate a subset of output pixels (full-size parity sampling)."""
    g = as_geometry(geom)
    N, M = g.N, g.n_det
    xs = g.pixel_centres()
    if pixels is None:
        X1, X2 = np.meshgrid(xs, xs, indexing="ij")
    else:
        X1, X2 = xs[np.asarray(pixels[0])], xs[np.asarray(pixels[1])]
    b = np.zeros(X1.shape)
    for it, t in enumerate(g.angles):
        d = interpolation_degree(g, t)
        gt = corrected_row(np.asarray(sino[it], dtype=np.float64), d)   # index j <-> m = j - h
        w = bp_widths(g, t)
        half = 0.5 * sum(kept_widths(w))
        kt = -np.sin(t) * X1 + np.cos(t) * X2
        # only samples with |y_m - k_theta| < half contribute (M is 0 outside its support):
        # for each pixel the S consecutive detector indices starting at m_first
        S = int(np.floor(2.0 * half / g.lambda_y)) + 2
        m_first = np.floor((kt - half) / g.lambda_y + (M // 2)).astype(np.int64)
        m = m_first[..., None] + np.arange(S)
        arg = g.lambda_y * (m - (M // 2)) - kt[..., None]
        j = m + H_CORR
        ok = (np.abs(arg) < half) & (j >= 0) & (j < M + 2 * H_CORR)
        vals = np.zeros(arg.shape)
        vals[ok] = gt[j[ok]] * box_spline(w, arg[ok])
        b += g.lambda_x ** 2 * g.lambda_y * vals.sum(axis=-1)
    return b


def interpolant(geom, t: float, sino_row: np.ndarray, y: np.ndarray) -> np.ndarray:
    """g^(y) = sum_m g~[m] B_d((y - y_m)/lambda_y), B_d the cardinal B-spline
    = box spline with d+1 unit widths (Eq.(1))."""
    g = as_geometry(geom)
    M = g.n_det
    d = interpolation_degree(g, t)
    gt = corrected_row(sino_row, d)
    ym = g.lambda_y * (np.arange(-H_CORR, M + H_CORR) - (M // 2))
    out = np.zeros_like(y, dtype=np.float64)
    for mi in range(gt.shape[0]):
        if gt[mi] != 0.0:
            out += gt[mi] * box_spline([1.0] * (d + 1), (y - ym[mi]) / g.lambda_y)
    return out


def backproject_quadrature(geom, sino: np.ndarray, k1: int, k2: int, nq: int = 20000) -> float:
    """Step 4 by numerical integration (midpoint rule between all breakpoints) of the
    explicit interpolant times the pixel footprint -- pin for the closed form."""
    g = as_geometry(geom)
    xs = g.pixel_centres()
    total = 0.0
    for it, t in enumerate(g.angles):
        kt = -np.sin(t) * xs[k1] + np.cos(t) * xs[k2]
        wf = g.blurred_widths(t)
        half = 0.5 * sum(kept_widths(wf))
        y = kt + np.linspace(-half, half, nq + 1)
        ymid = 0.5 * (y[1:] + y[:-1])
        dy = y[1] - y[0]
        F = g.lambda_x ** 2 * box_spline(wf, ymid - kt)
        total += float(np.sum(interpolant(g, t, np.asarray(sino[it], float), ymid) * F) * dy)
    return total
