"""Univariate box splines (section 3).

Eq.(1): M_Xi = M_xi1 * M_xi2 * ... * M_xin (convolution of elementary splines).
For univariate directions of length w_i each elementary spline is the unit-integral
box of width w_i, so M_W is the density of a sum of independent U(-w_i/2, w_i/2)
variables.  Its closed form is the truncated-power subset sum:

    M_W(x) = [(n-1)! prod w_i]^-1  sum_{S subset W} (-1)^|S| (x + sum(W)/2 - sum(S))_+^(n-1)

Widths at most 1e-12*max(1, sum W) are dropped (a zero-length elementary spline is the
Dirac, the convolution identity).  For n = 1 the support is
half-open [-w/2, w/2) (R6).
"""
from __future__ import annotations

import itertools
import math

import numpy as np

DROP_REL = 1e-12


def kept_widths(widths) -> list[float]:
    """Drop degenerate widths."""
    w = [abs(float(v)) for v in widths]
    thr = DROP_REL * max(1.0, sum(w))
    return [v for v in w if v > thr]


def box_spline(widths, x) -> np.ndarray:
    """M_W(x), FP64, vectorised over x.  Raises for the Dirac case (no width left)."""
    w = kept_widths(widths)
    n = len(w)
    if n == 0:
        raise ValueError("Dirac box spline cannot be evaluated pointwise")
    x = np.asarray(x, dtype=np.float64)
    W = sum(w)
    if n == 1:
        u = x + 0.5 * W
        return np.where((u >= 0.0) & (u < w[0]), 1.0 / w[0], 0.0)
    # M_W is even (a sum of centred uniforms is symmetric): evaluate on the left half,
    # where fewer truncated powers are active and their magnitudes are smaller.
    u = 0.5 * W - np.abs(x)
    acc = np.zeros_like(u)
    for r in range(n + 1):
        for S in itertools.combinations(range(n), r):
            sigma = sum(w[i] for i in S)
            acc += (-1.0) ** r * np.maximum(u - sigma, 0.0) ** (n - 1)
    val = acc / (math.factorial(n - 1) * math.prod(w))
    return np.where((u > 0.0) & (u < W), val, 0.0)


def support_halfwidth(widths) -> float:
    return 0.5 * sum(kept_widths(widths))
