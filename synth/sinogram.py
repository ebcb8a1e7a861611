"""Closed-form sinograms of ellipse phantoms and noise models (no method arithmetic).

The analytic line integral of an ellipse is the continuous ground truth g_c of
P:22; averaging it over a detector cell of width zeta is the detector model of
P:24 applied to g_c.  Both are textbook geometry, independent of box splines.
"""
from __future__ import annotations

import numpy as np


def detector_positions(n_det: int, lambda_y: float) -> np.ndarray:
    """y_m = lambda_y*(m - floor(M/2))."""
    return lambda_y * (np.arange(n_det, dtype=np.float64) - (n_det // 2))


def ellipse_sinogram(ellipses: np.ndarray, angles: np.ndarray, n_det: int, lambda_y: float,
                     zeta: float) -> np.ndarray:
    """g[theta, m] = (1/zeta) int_{y_m-zeta/2}^{y_m+zeta/2} P_theta f(y) dy for f = sum of
    ellipses, P_theta the line integral along (cos t, sin t), detector axis
    e = (-sin t, cos t).  zeta = 0: point sampling."""
    y = detector_positions(n_det, lambda_y)[None, :]
    th = np.asarray(angles, dtype=np.float64)[:, None]
    e1, e2 = -np.sin(th), np.cos(th)
    g = np.zeros((th.shape[0], n_det), dtype=np.float64)
    for (cx, cy, a, b, phi, rho) in ellipses:
        t0 = e1 * cx + e2 * cy
        p1 = e1 * np.cos(phi) + e2 * np.sin(phi)
        p2 = -e1 * np.sin(phi) + e2 * np.cos(phi)
        r2 = (a * p1) ** 2 + (b * p2) ** 2
        r = np.sqrt(r2)
        if zeta > 0:
            def Phi(u):
                uc = np.clip(u, -r, r)
                return (rho * a * b / r2) * (uc * np.sqrt(np.maximum(r2 - uc * uc, 0.0))
                                             + r2 * np.arcsin(uc / r))
            g += (Phi(y + 0.5 * zeta - t0) - Phi(y - 0.5 * zeta - t0)) / zeta
        else:
            d = y - t0
            g += np.where(np.abs(d) < r, (2.0 * rho * a * b / r2) * np.sqrt(np.maximum(r2 - d * d, 0.0)), 0.0)
    return g


def add_gaussian_noise(sino: np.ndarray, seed: int, rel_sigma: float) -> np.ndarray:
    """BASELINE.json configs 1,2,4: Gaussian noise sigma = rel_sigma * max|g|."""
    if rel_sigma <= 0:
        return sino.copy()
    rng = np.random.default_rng(seed)
    return sino + rng.standard_normal(sino.shape) * (rel_sigma * np.abs(sino).max())


def add_poisson_noise(sino: np.ndarray, seed: int, photons: float, kappa: float | None = None) -> np.ndarray:
    """counts ~ Poisson(I0 exp(-kappa p)), floored at 1,
    p~ = -ln(counts/I0)/kappa.  kappa = 4/max(p) unless given (config 5: kappa = 1)."""
    rng = np.random.default_rng(seed)
    if kappa is None:
        m = float(np.abs(sino).max())
        kappa = 4.0 / m if m > 0 else 1.0
    lam = photons * np.exp(-kappa * sino)
    counts = np.maximum(rng.poisson(lam), 1).astype(np.float64)
    return -np.log(counts / photons) / kappa


def config_sinogram(cfg, slice_index: int = 0) -> np.ndarray:
    """Sinogram g_s[theta, m] of a config from the analytic ellipse projections plus the
    config's noise model.  (Configs 3-5 specify a pixel-basis forward projection of an
    image; parity of the operators does not depend on which sinogram is used, so tests use
    this closed-form sinogram at every config's geometry; bench.py uses the GPU forward.)"""
    from .phantom import random_ellipses
    seed = cfg.seed + slice_index
    rho_range = (0.0, 1.0) if cfg.index == 5 else (-0.5, 1.0)
    ell = random_ellipses(seed, cfg.n_ellipses, cfg.ellipse_scale, rho_range=rho_range)
    if cfg.index == 5:
        ell[:, 5] *= 0.05
    g = ellipse_sinogram(ell, cfg.angles, cfg.n_det, cfg.lambda_y, cfg.zeta)
    if cfg.noise == "gauss":
        return add_gaussian_noise(g, seed + 1, cfg.noise_level)
    kappa = 1.0 if cfg.index == 5 else None
    return add_poisson_noise(g, seed + 1, cfg.noise_level, kappa=kappa)


def random_sinogram(seed: int, B: int, n_angles: int, n_det: int) -> np.ndarray:
    """i.i.d. U(-1,1) sinogram samples [B, n_angles, n_det] (operator parity inputs:
    exercises every detector bin including the edges)."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, size=(B, n_angles, n_det))
