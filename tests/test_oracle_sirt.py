"""Pins for oracle.forward.adjoint and oracle/sirt.py.

* adjoint: <H c, g> = <c, H^T g> for random c, g (dot-product test; H is pinned against
  geometric footprints in test_oracle_forward.py).
* SIRT: the iterate equals the same recurrence written with dense matrices (H assembled
  column by column from forward on unit images, weights from its row / column sums), the
  weighted residual is non-increasing, and consistent data from a full-column-rank system
  are recovered.
"""
import numpy as np

from oracle.forward import adjoint, forward
from oracle.sirt import sirt, weights


def geom(N, n, M, zeta=0.5, ly=1.0):
    return dict(N=N, lambda_x=1.0, angles=np.arange(n) * np.pi / n + 0.1, lambda_y=ly, n_det=M, zeta=zeta)


def dense_H(g):
    N = g["N"]
    cols = []
    for k in range(N * N):
        e = np.zeros(N * N)
        e[k] = 1.0
        cols.append(forward(g, e.reshape(N, N)).ravel())
    return np.stack(cols, axis=1)


def test_adjoint_dot_product():
    rng = np.random.default_rng(1)
    for zeta, ly in ((0.0, 1.0), (0.7, 0.6), (1.5, 1.3)):
        g = geom(7, 9, 17, zeta, ly)
        c = rng.standard_normal((7, 7))
        s = rng.standard_normal((9, 17))
        lhs = float(np.vdot(forward(g, c), s))
        rhs = float(np.vdot(c, adjoint(g, s)))
        assert abs(lhs - rhs) <= 1e-12 * max(1.0, abs(lhs))
        k1, k2 = np.array([0, 3, 6, 2]), np.array([6, 3, 0, 5])
        full = adjoint(g, s)
        assert np.allclose(adjoint(g, s, pixels=(k1, k2)), full[k1, k2], rtol=1e-13, atol=1e-14)


def test_sirt_equals_dense_recurrence_and_monotone():
    g = geom(4, 10, 9)
    H = dense_H(g)
    rs, cs = H.sum(axis=1), H.sum(axis=0)
    R = np.where(rs > 0, 1 / np.where(rs > 0, rs, 1), 0)
    C = np.where(cs > 0, 1 / np.where(cs > 0, cs, 1), 0)
    Rw, Cw = weights(g)
    assert np.allclose(Rw.ravel(), R, rtol=1e-13) and np.allclose(Cw.ravel(), C, rtol=1e-13)
    sino = np.random.default_rng(2).uniform(0, 1, (10, 9))
    x, hist = sirt(g, sino, 12)
    xd = np.zeros(16)
    for _ in range(12):
        xd = xd + C * (H.T @ (R * (sino.ravel() - H @ xd)))
    assert np.abs(x.ravel() - xd).max() <= 1e-12 * np.abs(xd).max()
    assert np.all(np.diff(hist) <= 1e-12 * hist[0])


def test_sirt_recovers_consistent_data():
    g = geom(3, 12, 9, zeta=1.0)
    H = dense_H(g)
    assert np.linalg.matrix_rank(H) == 9
    c = np.random.default_rng(3).uniform(0, 1, (3, 3))
    x, hist = sirt(g, forward(g, c), 400)
    assert np.abs(x - c).max() < 1e-6
