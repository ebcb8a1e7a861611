"""BASELINE.json configs[1..5] as plain data (no method arithmetic).

Readings:
  * angles theta_i = i*pi/n_theta, i = 0..n_theta-1 (uniform in [0, pi), BASELINE.json)
  * pixel centres x_k = lambda_x*(k - floor(N/2)), detector y_m = lambda_y*(m - floor(M/2))
    (integer lattices as in the paper)
  * seeds: config i uses base seed 1000*i; slice s of config 5 uses 5000 + s.
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace

import numpy as np


def uniform_angles(n_angles: int) -> np.ndarray:
    """theta_i = i*pi/n, FP64 (BASELINE.json: 'angles uniform in [0,pi)')."""
    return np.arange(n_angles, dtype=np.float64) * (np.pi / n_angles)


@dataclass(frozen=True)
class Config:
    index: int
    N: int
    dtype: str            # "f32" | "f64"
    n_angles: int
    n_det: int
    lambda_y: float
    zeta: float
    iters: int
    lambda_x: float = 1.0
    n_ellipses: int = 10
    ellipse_scale: float = 1.0      # spatial scale of ellipse draws (R13: N/64)
    grf_corr: float = 0.0           # correlation length in px (0: no GRF)
    grf_amp: float = 0.0
    noise: str = "gauss"            # "gauss" | "poisson"
    noise_level: float = 0.0        # gauss: sigma as a fraction of max; poisson: photons/ray
    n_slices: int = 1
    sinogram: str = "analytic"      # how BASELINE.json builds the sinogram
    notes: str = ""
    angles: np.ndarray = field(default=None, compare=False, repr=False)

    def __post_init__(self):
        if self.angles is None:
            object.__setattr__(self, "angles", uniform_angles(self.n_angles))

    @property
    def seed(self) -> int:
        return 1000 * self.index

    def with_(self, **kw) -> "Config":
        if "n_angles" in kw and "angles" not in kw:
            kw["angles"] = uniform_angles(kw["n_angles"])
        return replace(self, **kw)

    def geometry(self) -> dict:
        """Plain geometry dict: the paper's problem statement."""
        return dict(N=self.N, lambda_x=self.lambda_x, angles=self.angles.copy(),
                    lambda_y=self.lambda_y, n_det=self.n_det, zeta=self.zeta)


CONFIGS = {
    1: Config(1, N=64, dtype="f64", n_angles=90, n_det=91, lambda_y=1.0, zeta=1.0, iters=20,
              n_ellipses=10, ellipse_scale=1.0, noise="gauss", noise_level=0.01,
              notes="BJ:configs[1]"),
    2: Config(2, N=256, dtype="f32", n_angles=180, n_det=363, lambda_y=1.0, zeta=1.0, iters=50,
              n_ellipses=30, ellipse_scale=4.0, noise="gauss", noise_level=0.005,
              notes="BJ:configs[2]"),
    3: Config(3, N=512, dtype="f32", n_angles=360, n_det=725, lambda_y=1.0, zeta=1.5, iters=100,
              n_ellipses=50, ellipse_scale=8.0, grf_corr=8.0, grf_amp=0.2,
              noise="poisson", noise_level=1e5, sinogram="forward4x",
              notes="BJ:configs[3]"),
    4: Config(4, N=1024, dtype="f32", n_angles=720, n_det=2048, lambda_y=0.5, zeta=0.5, iters=100,
              n_ellipses=100, ellipse_scale=16.0, grf_corr=8.0, grf_amp=0.2,
              noise="gauss", noise_level=0.002, sinogram="analytic+forward_grf",
              notes="BJ:configs[4]; Gram build split over angle shards + allreduce"),
    5: Config(5, N=512, dtype="f32", n_angles=360, n_det=725, lambda_y=1.0, zeta=1.0, iters=50,
              n_ellipses=20, ellipse_scale=8.0, grf_corr=-1.0, grf_amp=1.0,
              noise="poisson", noise_level=1e4, n_slices=2048, sinogram="forward",
              notes="BJ:configs[5]; 2048 slices, GRF corr U(4,16) per slice, values in [0,0.05]"),
}


def config(i: int) -> Config:
    return CONFIGS[i]
