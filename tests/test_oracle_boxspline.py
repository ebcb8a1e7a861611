"""Pins for oracle/boxspline.py (Eq.(1); SPEC S:48 closed form).

Each check is independent of the subset-sum formula it tests: worked values of the
SPEC / textbook B-splines, partition of unity, unit mass, symmetry, and brute-force
numerical convolution of boxes (Eq.(1) itself, evaluated on a grid).
"""
import json
import os

import numpy as np
import pytest

from oracle.boxspline import box_spline, kept_widths

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def test_spec_examples():
    for c in GOLD["box_examples"]["cases"]:
        assert box_spline(c["widths"], c["x"]) == pytest.approx(c["value"], abs=1e-14)


def test_cubic_bspline_textbook():
    v = GOLD["cubic_bspline"]["values"]
    for k in (0, 1, 2):
        assert box_spline([1.0] * 4, float(k)) == pytest.approx(v[str(k)], abs=1e-15)
        assert box_spline([1.0] * 4, -float(k)) == pytest.approx(v[str(k)], abs=1e-15)


def test_scaling_identity():
    # M_[w]^n(x) = (1/w) M_[1]^n(x/w): a change of variables in the density of a sum of uniforms
    x = np.linspace(-2.2, 2.2, 97)
    for w in (0.3, 0.5, 1.7):
        assert np.allclose(box_spline([w] * 4, x * w) * w, box_spline([1.0] * 4, x), atol=1e-12)


def test_partition_of_unity():
    x = np.linspace(-3.0, 3.0, 1000)
    s = sum(box_spline([1.0], x - k) for k in range(-6, 7))
    assert np.abs(s - 1.0).max() < 1e-12
    # unit width within any set of widths -> integer translates sum to 1 (box * anything)
    s = sum(box_spline([1.0, 0.37, 0.81], x - k) for k in range(-6, 7))
    assert np.abs(s - 1.0).max() < 1e-12


def test_unit_integral_and_symmetry():
    rng = np.random.default_rng(1)
    for _ in range(20):
        n = rng.integers(2, 7)
        w = list(rng.uniform(0.05, 2.0, n))
        W = sum(w)
        x = np.linspace(-W / 2, W / 2, 20001)
        v = box_spline(w, x)
        assert np.trapezoid(v, x) == pytest.approx(1.0, abs=1e-6)
        xi = x[1:-1]
        assert np.abs(box_spline(w, xi) - box_spline(w, -xi)).max() < 1e-12 * v.max()


def test_drop_degenerate():
    assert kept_widths([1.0, 0.0]) == [1.0]
    assert kept_widths([np.cos(np.pi / 2), 1.0]) == [1.0]      # cos(pi/2) = 6e-17 (R9)
    with pytest.raises(ValueError):
        box_spline([0.0], 0.0)


def test_convolution_consistency():
    """Eq.(1): M_{A u B} = M_A * M_B, brute-force convolution on a fine grid."""
    rng = np.random.default_rng(2)
    h = 1e-3
    for _ in range(8):
        A = list(rng.uniform(0.2, 1.5, rng.integers(1, 4)))
        B = list(rng.uniform(0.2, 1.5, rng.integers(1, 4)))
        WA, WB = sum(A), sum(B)
        xa = np.arange(-WA / 2 + h / 2, WA / 2, h)        # midpoints
        xb = np.arange(-WB / 2 + h / 2, WB / 2, h)
        conv = np.convolve(box_spline(A, xa), box_spline(B, xb)) * h
        xc = xa[0] + xb[0] + h * np.arange(conv.size)
        ref = box_spline(A + B, xc)
        # midpoint-rule error O(h) at the kinks of a 1- or 2-width factor
        assert np.abs(conv - ref).max() < 5e-3 * ref.max()


def test_gram_rationals_by_quadrature():
    """M_[1,1,z,z](k) = int tri(t) tri_z(k - t) dt (Eq.(1) grouping [1,1] and [z,z]);
    tri_z is the unit-mass triangle of half-width z.  Exact piecewise Gauss-Legendre."""
    xg, wg = np.polynomial.legendre.leggauss(4)
    exact = {0.5: (5 / 6, 1 / 12, 0.0), 1.0: (2 / 3, 1 / 6, 0.0), 1.5: (14 / 27, 25 / 108, 1 / 108)}
    for z, vals in exact.items():
        for k, v in enumerate(vals):
            br = np.unique(np.array([-1.0, 0.0, 1.0, k - z, k, k + z]))
            tot = 0.0
            for a, b in zip(br[:-1], br[1:]):
                t = 0.5 * (a + b) + 0.5 * (b - a) * xg
                f = np.maximum(0, 1 - np.abs(t)) * np.maximum(0, 1 - np.abs(k - t) / z) / z
                tot += 0.5 * (b - a) * np.sum(wg * f)
            assert tot == pytest.approx(v, abs=1e-14)
            assert box_spline([1, 1, z, z], float(k)) == pytest.approx(v, abs=1e-13)
