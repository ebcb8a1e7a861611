"""Gram filter of the pixel-basis forward model (section 4).

gram_taps -- the paper's closed form.  Without blur
    g_ij = sum_theta M_[cos t, cos t, sin t, sin t](k_i,theta - k_j,theta)
and with detector blur
    g_ij = (1/zeta)^2 sum_theta M_[cos t, cos t, sin t, sin t, zeta, zeta](k_i,theta - k_j,theta).
Reading R1: every M here is unit-integral, so the blur box (1/zeta)box(./zeta)
IS M_[zeta]; the (1/zeta)^2 prefactor is already inside the two unit-integral blur
widths.  Reading R3: with Lambda_x = lambda_x I the projected widths scale by lambda_x
and the pixel mass by lambda_x^2, so taps carry lambda_x^4.  Reading R2: H maps to a
continuous detector coordinate y (the Gram element is a continuous inner product).

G depends only on k_i - k_j (Toeplitz-block-Toeplitz), so it is returned as the
(2N-1)x(2N-1) filter G[dk1 + N-1, dk2 + N-1].  Angles are summed in the given order.

footprint_gram_dense -- brute force for pins: the dense N^2 x N^2 matrix
    G_ij = sum_theta int F_i(y) F_j(y) dy
with F_k the geometric (chord-length, blurred) footprint of pixel k (footprint.py),
i.e. H^T H of P:96 built without box splines and without assuming Toeplitz structure.
"""
from __future__ import annotations

import numpy as np

from .boxspline import box_spline, kept_widths
from .footprint import footprint_inner
from .geometry import as_geometry


def gram_widths(lambda_x: float, t: float, zeta: float) -> list[float]:
    """[lambda_x|c|, lambda_x|c|, lambda_x|s|, lambda_x|s|, zeta, zeta]."""
    c, s = abs(np.cos(t)), abs(np.sin(t))
    w = [lambda_x * c, lambda_x * c, lambda_x * s, lambda_x * s]
    if zeta > 0:
        w += [zeta, zeta]
    return w


def gram_taps(geom, angle_begin: int = 0, angle_end: int | None = None) -> np.ndarray:
    """(2N-1)^2 Gram filter, FP64.  angle_begin/angle_end select an angle shard
    (BASELINE.json config 4: partial filters are summed by an allreduce)."""
    g = as_geometry(geom)
    N, lam = g.N, g.lambda_x
    d = np.arange(-(N - 1), N, dtype=np.float64)
    a = d[:, None]          # dk1
    b = d[None, :]          # dk2
    G = np.zeros((2 * N - 1, 2 * N - 1), dtype=np.float64)
    end = len(g.angles) if angle_end is None else angle_end
    for t in g.angles[angle_begin:end]:
        w = gram_widths(lam, t, g.zeta)
        half = 0.5 * sum(kept_widths(w))
        u = lam * (-np.sin(t) * a + np.cos(t) * b)     # k_i,theta - k_j,theta
        m = np.abs(u) < half                            # M is exactly 0 outside its support
        G[m] += lam ** 4 * box_spline(w, u[m])
    return G


def gram_taps_at(geom, dk1, dk2) -> np.ndarray:
    """The same sum as gram_taps at selected offsets (dk1[i], dk2[i]) -- for sampling
    full-size filters one tap at a time."""
    g = as_geometry(geom)
    lam = g.lambda_x
    a = np.asarray(dk1, dtype=np.float64)
    b = np.asarray(dk2, dtype=np.float64)
    out = np.zeros(a.shape, dtype=np.float64)
    for t in g.angles:
        w = gram_widths(lam, t, g.zeta)
        half = 0.5 * sum(kept_widths(w))
        u = lam * (-np.sin(t) * a + np.cos(t) * b)
        m = np.abs(u) < half
        out[m] += lam ** 4 * box_spline(w, u[m])
    return out


def toeplitz_matrix(taps: np.ndarray) -> np.ndarray:
    """Dense N^2 x N^2 matrix G[i, j] = taps[k_i - k_j], row-major pixel order."""
    N = (taps.shape[0] + 1) // 2
    k1, k2 = np.meshgrid(np.arange(N), np.arange(N), indexing="ij")
    k1, k2 = k1.ravel(), k2.ravel()
    return taps[(k1[:, None] - k1[None, :]) + N - 1, (k2[:, None] - k2[None, :]) + N - 1]


def footprint_gram_dense(geom) -> np.ndarray:
    """Brute-force H^T H (continuous y) from geometric footprints; N <= 8 intended."""
    g = as_geometry(geom)
    N, lam = g.N, g.lambda_x
    xs = g.pixel_centres()
    centres = [(xs[i], xs[j]) for i in range(N) for j in range(N)]
    n = N * N
    G = np.zeros((n, n))
    for t in g.angles:
        for i in range(n):
            for j in range(i, n):
                v = footprint_inner(t, centres[i], centres[j], lam, g.zeta)
                G[i, j] += v
                if j != i:
                    G[j, i] += v
    return G
