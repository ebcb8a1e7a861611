"""Pins for the NEXT-3 harness metrics (tools/experiments.py; "SNR and SSIM").

SSIM is checked against a brute-force per-window evaluation of the definition (explicit loops
over every 11 x 11 window, weights from the 2-D Gaussian exp(-(i^2 + j^2) / 2 sigma^2)
normalised), plus SPEC's examples: identity -> 1, symmetry, inverted binary image < 0.1."""
import math
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import experiments  # noqa: E402


def ssim_brute(a, b, size=11, sigma=1.5, k1=0.01, k2=0.03):
    h = (size - 1) // 2
    i, j = np.meshgrid(np.arange(-h, h + 1), np.arange(-h, h + 1), indexing="ij")
    w2 = np.exp(-(i * i + j * j) / (2 * sigma * sigma))
    w2 /= w2.sum()
    L = a.max() - a.min()
    c1, c2 = (k1 * L) ** 2, (k2 * L) ** 2
    vals = []
    for r in range(a.shape[0] - size + 1):
        for c in range(a.shape[1] - size + 1):
            pa, pb = a[r:r + size, c:c + size], b[r:r + size, c:c + size]
            ma, mb = (w2 * pa).sum(), (w2 * pb).sum()
            va, vb = (w2 * (pa - ma) ** 2).sum(), (w2 * (pb - mb) ** 2).sum()
            cab = (w2 * (pa - ma) * (pb - mb)).sum()
            vals.append(((2 * ma * mb + c1) * (2 * cab + c2)) / ((ma * ma + mb * mb + c1) * (va + vb + c2)))
    return float(np.mean(vals))


@pytest.mark.parametrize("shape", [(11, 11), (16, 23), (20, 14)])
def test_ssim_brute_force(shape):
    rng = np.random.default_rng(sum(shape))
    a = rng.uniform(0, 1, shape)
    b = a + rng.normal(0, 0.2, shape)
    assert experiments.ssim(a, b) == pytest.approx(ssim_brute(a, b), abs=1e-12)
    c = np.roll(a, 1, axis=0) * 0.7 + 0.1
    assert experiments.ssim(a, c) == pytest.approx(ssim_brute(a, c), abs=1e-12)


def test_ssim_spec_examples():
    rng = np.random.default_rng(7)
    a = (rng.uniform(0, 1, (32, 32)) > 0.5).astype(float)
    assert experiments.ssim(a, a) == pytest.approx(1.0, abs=1e-15)
    assert experiments.ssim(a, 1 - a) < 0.1
    b = rng.uniform(0, 1, (32, 32))
    c = rng.permutation(b.ravel()).reshape(b.shape)  # same range, so the same L either way
    assert abs(experiments.ssim(b, c) - experiments.ssim(c, b)) < 1e-12
    with pytest.raises(ValueError):
        experiments.ssim(np.ones((16, 16)), b[:16, :16])


def test_snr_definition():
    rng = np.random.default_rng(9)
    ref = rng.uniform(-1, 1, (20, 20))
    e = rng.normal(0, 1, (20, 20))
    e *= math.sqrt((ref ** 2).sum() / 100 / (e ** 2).sum())
    assert experiments.snr_db(ref, ref + e) == pytest.approx(20.0, abs=1e-9)
    assert experiments.snr_db(ref, np.zeros_like(ref)) == pytest.approx(0.0, abs=1e-12)
