"""Parallel-beam geometry of PAPER.md section 2 and section 4.

* image f_psi(x) = sum_k c_k psi(x - Lambda_x k), Lambda_x = lambda_x I
  with pixel centres x_k = lambda_x (k - floor(N/2)) per axis;
  array index [k1, k2] <-> coordinates (x_k1, x_k2).
* ray direction theta = (cos t, sin t); detector axis theta_perp = (-sin t, cos t)
  (SURVEY.md R4); k_theta = <theta_perp, x_k> ("k_theta = P_theta_perp k").
* detector samples y_m = lambda_y (m - floor(M/2)) ("delta(y - lambda_y m)", R5).
* projected pixel = univariate box spline with widths [lambda_x|cos t|, lambda_x|sin t|]
  (Eq.(3)), plus the detector blur width zeta (Eq.(4)).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class Geometry:
    N: int
    lambda_x: float
    angles: np.ndarray
    lambda_y: float
    n_det: int
    zeta: float

    @classmethod
    def from_dict(cls, d: dict) -> "Geometry":
        return cls(int(d["N"]), float(d["lambda_x"]), np.asarray(d["angles"], dtype=np.float64),
                   float(d["lambda_y"]), int(d["n_det"]), float(d["zeta"]))

    def pixel_centres(self) -> np.ndarray:
        return self.lambda_x * (np.arange(self.N, dtype=np.float64) - (self.N // 2))

    def detector_positions(self) -> np.ndarray:
        return self.lambda_y * (np.arange(self.n_det, dtype=np.float64) - (self.n_det // 2))

    def k_theta(self, t: float) -> np.ndarray:
        """k_theta[k1,k2] = -sin t * x_k1 + cos t * x_k2."""
        x = self.pixel_centres()
        return -np.sin(t) * x[:, None] + np.cos(t) * x[None, :]

    def pixel_widths(self, t: float) -> list[float]:
        """P_theta_perp Xi = [cos t, sin t] scaled by lambda_x."""
        return [self.lambda_x * abs(np.cos(t)), self.lambda_x * abs(np.sin(t))]

    def blurred_widths(self, t: float) -> list[float]:
        """P_theta_perp Xi U zeta_blur; zeta = 0 means no blur."""
        w = self.pixel_widths(t)
        return w + ([self.zeta] if self.zeta > 0 else [])


def as_geometry(g) -> Geometry:
    return g if isinstance(g, Geometry) else Geometry.from_dict(g)
