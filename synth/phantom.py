"""Seeded phantoms: random ellipses ("Spots") and a Gaussian random field.

No method arithmetic here: ellipses are rasterised by 4x4 point supersampling of
each pixel (area fractions) and the GRF is white noise filtered in
Fourier space.
"""
from __future__ import annotations

import numpy as np

# one ellipse = (cx, cy, a, b, phi, rho); cx/cy are coordinates along image axes 1/2
ELLIPSE_FIELDS = ("cx", "cy", "a", "b", "phi", "rho")


def random_ellipses(seed: int, count: int, scale: float, rho_range=(-0.5, 1.0)) -> np.ndarray:
    """BASELINE.json configs: centres U(-24,24), semi-axes U(3,20), angle U(0,pi),
    density U(-0.5,1); spatial parameters scaled by `scale` = N/64.
    Draw order per ellipse: cx, cy, a, b, phi, rho from numpy default_rng(seed)."""
    rng = np.random.default_rng(seed)
    out = np.empty((count, 6), dtype=np.float64)
    for i in range(count):
        cx = rng.uniform(-24.0, 24.0) * scale
        cy = rng.uniform(-24.0, 24.0) * scale
        a = rng.uniform(3.0, 20.0) * scale
        b = rng.uniform(3.0, 20.0) * scale
        phi = rng.uniform(0.0, np.pi)
        rho = rng.uniform(*rho_range)
        out[i] = (cx, cy, a, b, phi, rho)
    return out


def pixel_centres(N: int, lambda_x: float) -> np.ndarray:
    """x_k = lambda_x*(k - floor(N/2))."""
    return lambda_x * (np.arange(N, dtype=np.float64) - (N // 2))


def rasterize_ellipses(ellipses: np.ndarray, N: int, lambda_x: float = 1.0, sub: int = 4) -> np.ndarray:
    """Pixel coefficients c[k1,k2] = sum_e rho_e * (area fraction of pixel k inside e),
    estimated by sub x sub point supersampling.  Axis 0 is coordinate 1."""
    xc = pixel_centres(N, lambda_x)
    offs = ((np.arange(sub) + 0.5) / sub - 0.5) * lambda_x
    img = np.zeros((N, N), dtype=np.float64)
    for (cx, cy, a, b, phi, rho) in ellipses:
        # bounding box in pixel indices (the ellipse fits in a circle of radius max(a,b))
        R = max(a, b) + lambda_x
        k1 = np.nonzero(np.abs(xc - cx) <= R)[0]
        k2 = np.nonzero(np.abs(xc - cy) <= R)[0]
        if k1.size == 0 or k2.size == 0:
            continue
        X1 = xc[k1][:, None, None, None] + offs[None, None, :, None]
        X2 = xc[k2][None, :, None, None] + offs[None, None, None, :]
        d1, d2 = X1 - cx, X2 - cy
        cp, sp = np.cos(phi), np.sin(phi)
        u = d1 * cp + d2 * sp
        v = -d1 * sp + d2 * cp
        inside = (u / a) ** 2 + (v / b) ** 2 <= 1.0
        frac = inside.mean(axis=(2, 3))
        img[np.ix_(k1, k2)] += rho * frac
    return img


def gaussian_random_field(seed: int, N: int, corr: float, amp: float) -> np.ndarray:
    """White noise on a periodic 2N x 2N grid filtered by exp(-|k|^2 corr^2 / 4)
    (k in rad/px), cropped to N x N, rescaled to zero mean and std = amp
    (covariance exp(-r^2 / (2 corr^2)))."""
    rng = np.random.default_rng(seed)
    n2 = 2 * N
    w = rng.standard_normal((n2, n2))
    k = 2.0 * np.pi * np.fft.fftfreq(n2)
    K2 = k[:, None] ** 2 + k[None, :] ** 2
    f = np.fft.ifft2(np.fft.fft2(w) * np.exp(-K2 * corr * corr / 4.0)).real[:N, :N]
    f = f - f.mean()
    sd = f.std()
    return f * (amp / sd) if sd > 0 else f


def config_image(cfg, slice_index: int = 0) -> np.ndarray:
    """Pixel-coefficient image of a BASELINE.json config (used where the sinogram is a
    pixel-basis forward projection: configs 3-5, and as a test image elsewhere)."""
    seed = cfg.seed + slice_index
    N = cfg.N
    if cfg.index == 5:
        rng = np.random.default_rng(seed)
        corr = rng.uniform(4.0, 16.0)
        img = gaussian_random_field(seed + 7, N, corr, 1.0)
        img = img + rasterize_ellipses(random_ellipses(seed, cfg.n_ellipses, cfg.ellipse_scale,
                                                       rho_range=(0.0, 1.0)), N, cfg.lambda_x)
        lo, hi = img.min(), img.max()
        return 0.05 * (img - lo) / (hi - lo if hi > lo else 1.0)
    img = rasterize_ellipses(random_ellipses(seed, cfg.n_ellipses, cfg.ellipse_scale), N, cfg.lambda_x)
    if cfg.grf_corr > 0:
        img = img + gaussian_random_field(seed + 7, N, cfg.grf_corr, cfg.grf_amp)
    return img


def random_image(seed: int, B: int, N: int) -> np.ndarray:
    """Plain i.i.d. U(-1,1) coefficients, shape [B,N,N] (operator parity inputs)."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, size=(B, N, N))
