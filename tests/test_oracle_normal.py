"""Pins for oracle/normal.py and the PSD property of G = H^T H."""
import numpy as np
import pytest

from oracle.gram import gram_taps, toeplitz_matrix
from oracle.normal import apply_direct, apply_fft, embed_size, embed_spectrum


def taps_for(N, n=20, zeta=1.0):
    return gram_taps(dict(N=N, lambda_x=1.0, angles=np.arange(n) * np.pi / n, lambda_y=1.0, n_det=3, zeta=zeta))


def test_direct_equals_dense_matrix():
    N = 6
    T = taps_for(N)
    x = np.random.default_rng(0).standard_normal((N, N))
    y = apply_direct(T, x)
    assert np.abs(y.ravel() - toeplitz_matrix(T) @ x.ravel()).max() < 1e-13


@pytest.mark.parametrize("N", [1, 2, 5, 8, 13])
def test_fft_equals_direct(N):
    T = taps_for(N)
    x = np.random.default_rng(N).standard_normal((3, N, N))
    assert np.abs(apply_fft(T, x) - apply_direct(T, x)).max() < 1e-12 * max(1.0, np.abs(apply_direct(T, x)).max())


def test_delta_gives_central_crop():
    N = 7
    T = taps_for(N)
    x = np.zeros((N, N))
    x[0, 0] = 1.0
    # y[i] = G[i - 0]: the lower-right quadrant of the filter
    assert np.abs(apply_fft(T, x) - T[N - 1:, N - 1:]).max() < 1e-13
    x = np.zeros((N, N))
    x[N // 2, N // 2] = 1.0
    c = N - 1 - N // 2
    assert np.abs(apply_direct(T, x) - T[c:c + N, c:c + N]).max() < 1e-15


def test_linearity():
    N = 9
    T = taps_for(N)
    rng = np.random.default_rng(4)
    a, b = rng.standard_normal((2, N, N))
    lhs = apply_fft(T, 2.5 * a - 0.75 * b)
    rhs = 2.5 * apply_fft(T, a) - 0.75 * apply_fft(T, b)
    assert np.abs(lhs - rhs).max() < 1e-12 * np.abs(lhs).max()


def test_psd():
    for N, z in ((8, 0.0), (16, 1.0)):
        T = taps_for(N, 24, z)
        rng = np.random.default_rng(N)
        for _ in range(10):
            c = rng.standard_normal((N, N))
            assert np.vdot(c, apply_fft(T, c)) >= -1e-10 * np.vdot(c, c)
        ev = np.linalg.eigvalsh(toeplitz_matrix(T))
        assert ev.min() > 0


def test_embedding_size_and_spectrum_real():
    assert [embed_size(n) for n in (1, 2, 5, 8, 64, 512)] == [2, 4, 16, 16, 128, 1024]
    import scipy.fft as sfft
    from oracle.normal import embed
    T = taps_for(8)
    E = embed(T, 16)
    assert np.abs(sfft.fft2(E).imag).max() < 1e-12        # G even => real spectrum
    assert embed_spectrum(T).shape == (16, 16)
