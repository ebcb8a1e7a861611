"""Normal-operator apply y = G x.

P:131: "the N^2 x N^2 Gram matrix G is a Toeplitz-block-Toeplitz matrix, which implies
that we can compute Gx exactly by applying a (2N-1) x (2N-1) filter on x":
    y[i1, i2] = sum_{j1, j2} G[i1 - j1, i2 - j2] x[j1, j2].

apply_direct is that sum written out.  apply_fft evaluates the same sum by zero
padding to an L x L circular convolution (exact for L >= 2N-1; SciPy FP64 FFT as a
library step) and is pinned against apply_direct in tests.
embed_spectrum is the DFT of the L x L circulant embedding, used only to define the
Landweber step tau = 1/max(spectrum) (reading R-LW) and for information.
"""
from __future__ import annotations

import numpy as np
import scipy.fft as sfft


def embed_size(N: int) -> int:
    """Smallest power of two >= max(2, 2N-1) (the product's FFT size)."""
    L = 2
    while L < 2 * N - 1:
        L *= 2
    return L


def apply_direct(taps: np.ndarray, x: np.ndarray) -> np.ndarray:
    """y = G x by the Toeplitz sum.  x: [..., N, N]."""
    N = x.shape[-1]
    y = np.zeros(x.shape, dtype=np.float64)
    for j1 in range(N):
        for j2 in range(N):
            blk = taps[N - 1 - j1: 2 * N - 1 - j1, N - 1 - j2: 2 * N - 1 - j2]
            y += x[..., j1, j2][..., None, None] * blk
    return y


def embed(taps: np.ndarray, L: int) -> np.ndarray:
    N = (taps.shape[0] + 1) // 2
    E = np.zeros((L, L), dtype=np.float64)
    d = np.arange(-(N - 1), N)
    E[np.ix_(d % L, d % L)] = taps
    return E


def embed_spectrum(taps: np.ndarray, L: int | None = None) -> np.ndarray:
    N = (taps.shape[0] + 1) // 2
    L = embed_size(N) if L is None else L
    return sfft.fft2(embed(taps, L)).real


def apply_fft(taps: np.ndarray, x: np.ndarray, L: int | None = None, workers: int = -1) -> np.ndarray:
    """y = crop(IFFT2(FFT2(E) * FFT2(pad x))) -- the same Toeplitz sum, FP64."""
    N = x.shape[-1]
    L = embed_size(N) if L is None else L
    Gh = sfft.rfft2(embed(taps, L), workers=workers)
    X = sfft.rfft2(x, s=(L, L), axes=(-2, -1), workers=workers)
    y = sfft.irfft2(X * Gh, s=(L, L), axes=(-2, -1), workers=workers)
    return y[..., :N, :N]
