"""Seeded synthetic inputs shared by the oracle tests, the CUDA parity tests and bench.py.

This package holds NO arithmetic of the paper's method (no box splines, no Gram
filter, no back projection, no Toeplitz apply).  It only describes the
BASELINE.json configurations and draws seeded phantoms / sinograms / noise:

* configs.py   -- geometry + run parameters of BASELINE.json configs[1..5]
* phantom.py   -- seeded random ellipses (the paper's "Spots") and a
                  Gaussian random field, rasterised to pixel coefficients
* sinogram.py  -- closed-form line integrals of ellipses averaged over the
                  detector cell (the *continuous* ground truth, not the
                  pixel-basis model), Gaussian / Poisson noise

Everything is plain NumPy (FP64) so that the CPU oracle and the GPU path see
bit-identical inputs.  bench.py may evaluate the same closed forms with torch on
the device for the 2048-slice stack (config 5); see synth/device.py.
"""
from .configs import CONFIGS, Config, config, uniform_angles  # noqa: F401
