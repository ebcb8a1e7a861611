"""Forward projection H c (Eq.(3), Eq.(4)).

forward: g_psi(y_m) = sum_k c_k lambda_x^2 M_[lambda_x|cos|, lambda_x|sin|, zeta](y_m - k_theta)
  -- Eq.(4) with reading R1 (unit-integral blur, no extra 1/zeta) and R3 (lambda_x^2 mass);
  zeta = 0 gives Eq.(3).  Sampled at y_m = lambda_y (m - floor(M/2)) by S.
forward_geometric: the same sampled sinogram from geometric chord-length footprints
  (footprint.py), i.e. without box splines -- the pin for forward (and for Eq.(2)).
"""
from __future__ import annotations

import numpy as np

from .boxspline import box_spline, kept_widths
from .footprint import footprint
from .geometry import as_geometry


def forward(geom, c: np.ndarray) -> np.ndarray:
    g = as_geometry(geom)
    y = g.detector_positions()
    out = np.zeros((len(g.angles), g.n_det))
    nz = np.nonzero(c)
    cv = c[nz]
    xs = g.pixel_centres()
    x1, x2 = xs[nz[0]], xs[nz[1]]
    for it, t in enumerate(g.angles):
        w = g.blurred_widths(t)
        half = 0.5 * sum(kept_widths(w))
        kt = -np.sin(t) * x1 + np.cos(t) * x2
        for m in range(g.n_det):
            arg = y[m] - kt
            msk = np.abs(arg) < half
            if msk.any():
                out[it, m] = g.lambda_x ** 2 * np.sum(cv[msk] * box_spline(w, arg[msk]))
    return out


def forward_geometric(geom, c: np.ndarray) -> np.ndarray:
    g = as_geometry(geom)
    y = g.detector_positions()
    xs = g.pixel_centres()
    out = np.zeros((len(g.angles), g.n_det))
    for it, t in enumerate(g.angles):
        for k1 in range(g.N):
            for k2 in range(g.N):
                if c[k1, k2] != 0.0:
                    out[it] += c[k1, k2] * footprint(y, t, (xs[k1], xs[k2]), g.lambda_x, g.zeta)
    return out


def adjoint(geom, g: np.ndarray, pixels=None) -> np.ndarray:
    """Plain adjoint of the sampled forward model: (H^T g)[k] = lambda_x^2 sum_t sum_m g[t, m]
    M_[lambda_x|cos t|, lambda_x|sin t|, zeta](y_m - k_t) -- the transpose of `forward` (no
    interpolation of g; contrast backproject.backproject).  Used by SIRT.
    pixels=(k1, k2): only those pixels (same sum, evaluated one by one)."""
    g0 = as_geometry(geom)
    y = g0.detector_positions()
    if pixels is not None:
        xs = g0.pixel_centres()
        p1, p2 = xs[np.asarray(pixels[0])], xs[np.asarray(pixels[1])]
        out = np.zeros(len(p1))
        for it, t in enumerate(g0.angles):
            w = g0.blurred_widths(t)
            half = 0.5 * sum(kept_widths(w))
            kt = -np.sin(t) * p1 + np.cos(t) * p2
            arg = y[:, None] - kt[None, :]                 # [M, P]
            msk = np.abs(arg) < half
            val = np.zeros_like(arg)
            val[msk] = box_spline(w, arg[msk])
            out += g0.lambda_x ** 2 * (g[it][:, None] * val).sum(axis=0)
        return out
    out = np.zeros((g0.N, g0.N))
    for it, t in enumerate(g0.angles):
        w = g0.blurred_widths(t)
        half = 0.5 * sum(kept_widths(w))
        kt = g0.k_theta(t)
        for m in range(g0.n_det):
            if g[it, m] == 0.0:
                continue
            arg = y[m] - kt
            msk = np.abs(arg) < half
            if msk.any():
                out[msk] += g0.lambda_x ** 2 * g[it, m] * box_spline(w, arg[msk])
    return out
