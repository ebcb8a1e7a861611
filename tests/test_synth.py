"""Checks of the seeded input generators (synth/): determinism, closed-form ellipse
projections against brute-force ray sampling and exact mass."""
import numpy as np
import pytest

from synth import CONFIGS
from synth.phantom import random_ellipses, rasterize_ellipses, config_image
from synth.sinogram import config_sinogram, ellipse_sinogram


def test_determinism():
    a = config_sinogram(CONFIGS[1])
    b = config_sinogram(CONFIGS[1])
    assert np.array_equal(a, b)
    assert np.array_equal(random_ellipses(5, 4, 1.0), random_ellipses(5, 4, 1.0))


def test_ellipse_mass_and_ray_sampling():
    e = np.array([[3.0, -5.0, 12.0, 5.0, 0.7, 0.8]])
    th = np.array([0.45])
    M, ly = 81, 0.5
    for zeta in (1.0, 1.5):     # zeta a multiple of lambda_y: the cell averages tile the line exactly
        g = ellipse_sinogram(e, th, M, ly, zeta)
        assert g.sum() * ly == pytest.approx(0.8 * np.pi * 12 * 5, rel=1e-6)
    # brute-force: integrate the indicator along rays (fine sampling)
    g = ellipse_sinogram(e, th, M, ly, 0.0)[0]
    t = th[0]
    n, d = np.array([-np.sin(t), np.cos(t)]), np.array([np.cos(t), np.sin(t)])
    s = np.linspace(-40, 40, 400001)
    for m in (20, 35, 40, 47):
        y = ly * (m - M // 2)
        p = y * n[:, None] + s[None, :] * d[:, None]
        dx, dy = p[0] - 3.0, p[1] + 5.0
        u = dx * np.cos(0.7) + dy * np.sin(0.7)
        v = -dx * np.sin(0.7) + dy * np.cos(0.7)
        brute = 0.8 * ((u / 12) ** 2 + (v / 5) ** 2 <= 1).sum() * (s[1] - s[0])
        assert brute == pytest.approx(g[m], abs=2e-3)


def test_rasterize_full_cover():
    img = rasterize_ellipses(np.array([[0.0, 0.0, 10.0, 10.0, 0.0, 2.0]]), 8)
    assert np.allclose(img[2:6, 2:6], 2.0)


def test_config_images_shapes():
    assert config_image(CONFIGS[1]).shape == (64, 64)
    c5 = config_image(CONFIGS[5].with_(N=64, ellipse_scale=1.0), 3)
    assert c5.min() == pytest.approx(0.0) and c5.max() == pytest.approx(0.05)
