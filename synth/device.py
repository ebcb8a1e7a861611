"""Device-side synthesis of the 2048-slice stack of BASELINE.json config 5 (bench only).

Same recipe as synth.phantom.config_image (GRF with corr ~ U(4,16) per slice + 20
ellipses, scaled to [0, 0.05]/px) evaluated with torch on the GPU so that 2048 slices
take seconds; ellipses are point-sampled at pixel centres (no 4x4 supersampling) and
the GRF noise comes from torch's CUDA generator, so values differ from the CPU
generator -- the bench only times, it never compares these values to the oracle.
The sinogram is the pixel-basis forward projection computed by the library itself
 plus Poisson noise at I0 photons/ray (R15, kappa = 1).
"""
from __future__ import annotations

import numpy as np
import torch

from .phantom import random_ellipses


def stack_images(cfg, slice_ids, device="cuda", chunk: int = 64) -> torch.Tensor:
    N = cfg.N
    out = torch.empty((len(slice_ids), N, N), dtype=torch.float32, device=device)
    xc = cfg.lambda_x * (torch.arange(N, device=device, dtype=torch.float32) - (N // 2))
    X1 = xc[:, None].expand(N, N)
    X2 = xc[None, :].expand(N, N)
    k = 2.0 * np.pi * torch.fft.fftfreq(2 * N, device=device)
    K2 = k[:, None] ** 2 + k[None, :] ** 2
    for c0 in range(0, len(slice_ids), chunk):
        ids = slice_ids[c0:c0 + chunk]
        C = len(ids)
        corr = torch.tensor([np.random.default_rng(cfg.seed + s).uniform(4.0, 16.0) for s in ids],
                            device=device, dtype=torch.float32)
        gen = torch.Generator(device=device)
        gen.manual_seed(cfg.seed + int(ids[0]))
        w = torch.randn((C, 2 * N, 2 * N), device=device, generator=gen)
        filt = torch.exp(-K2[None] * (corr[:, None, None] ** 2) / 4.0)
        f = torch.fft.ifft2(torch.fft.fft2(w) * filt).real[:, :N, :N]
        f = f - f.mean(dim=(1, 2), keepdim=True)
        f = f / f.std(dim=(1, 2), keepdim=True)
        ell = np.stack([random_ellipses(cfg.seed + s, cfg.n_ellipses, cfg.ellipse_scale, rho_range=(0.0, 1.0))
                        for s in ids])                                     # [C, E, 6]
        e = torch.tensor(ell, device=device, dtype=torch.float32)
        for j in range(e.shape[1]):
            cx, cy, a, b, phi, rho = (e[:, j, i][:, None, None] for i in range(6))
            d1, d2 = X1[None] - cx, X2[None] - cy
            u = d1 * torch.cos(phi) + d2 * torch.sin(phi)
            v = -d1 * torch.sin(phi) + d2 * torch.cos(phi)
            f = f + rho * (((u / a) ** 2 + (v / b) ** 2) <= 1.0).float()
        lo = f.amin(dim=(1, 2), keepdim=True)
        hi = f.amax(dim=(1, 2), keepdim=True)
        out[c0:c0 + C] = 0.05 * (f - lo) / (hi - lo).clamp_min(1e-30)
    return out


def poisson_log(sino: torch.Tensor, photons: float, seed: int, kappa: float = 1.0) -> torch.Tensor:
    """R15: counts ~ Poisson(I0 exp(-kappa p)), floored at 1; p~ = -ln(counts/I0)/kappa."""
    gen = torch.Generator(device=sino.device)
    gen.manual_seed(seed)
    lam = photons * torch.exp(-kappa * sino)
    counts = torch.poisson(lam, generator=gen).clamp_min(1.0)
    return -torch.log(counts / photons) / kappa
