"""SIRT on the sampled forward model, FP64.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper names forward and back projection as the computational burden of iterative
reconstruction (P:4) and avoids them inside the loop; SIRT is the textbook
projection-based iteration it is contrasted with:
    x_0 = 0,  x_{k+1} = x_k + C H^T R (g - H x_k),
    R = diag(1 / (H 1)) over detector samples, C = diag(1 / (H^T 1)) over pixels
(zero weight where a row or column sum is zero), H = forward.forward, H^T = forward.adjoint.
Returns (x, hist) with hist[k] = ||R^(1/2) (g - H x_{k+1})|| (weighted residual).
"""
from __future__ import annotations

import numpy as np

from .forward import adjoint, forward
from .geometry import as_geometry


def weights(geom):
    g = as_geometry(geom)
    hr = forward(g, np.ones((g.N, g.N)))
    hc = adjoint(g, np.ones((len(g.angles), g.n_det)))
    R = np.where(hr > 0, 1.0 / np.where(hr > 0, hr, 1.0), 0.0)
    C = np.where(hc > 0, 1.0 / np.where(hc > 0, hc, 1.0), 0.0)
    return R, C


def sirt(geom, sino: np.ndarray, iters: int):
    g = as_geometry(geom)
    R, C = weights(g)
    x = np.zeros((g.N, g.N))
    hist = []
    for _ in range(iters):
        res = sino - forward(g, x)
        x = x + C * adjoint(g, R * res)
        r2 = sino - forward(g, x)
        hist.append(float(np.sqrt(np.sum(R * r2 * r2))))
    return x, np.array(hist)
