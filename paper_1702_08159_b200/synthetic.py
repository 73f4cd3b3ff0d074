"""Seeded synthetic inputs with the shapes and value distributions of the
BASELINE.json configurations.  MNIST / FASHION-MNIST are not available in
this environment, so these MNIST-shaped stand-ins replace them.

All generators use numpy's PCG64 (``np.random.default_rng``), whose stream is
stable across numpy versions, so the GPU box regenerates the same inputs the
golden fixtures were computed on.
"""

from __future__ import annotations

import numpy as np


def image_rows(m: int, d: int = 784, seed: int = 1234) -> np.ndarray:
    """Configs 0/2: ~80% exact zeros, the rest uniform in (0, 1] (float32)."""
    rng = np.random.default_rng(seed)
    vals = (1.0 - rng.random((m, d), dtype=np.float32))          # (0, 1]
    zero = rng.random((m, d), dtype=np.float32) < 0.8
    vals[zero] = 0.0
    return vals


def gaussian_rows(m: int, n: int, seed: int = 7) -> np.ndarray:
    """Configs 1/4: i.i.d. N(0, 1) float32."""
    return np.random.default_rng(seed).standard_normal((m, n), dtype=np.float32)


def class_images(m: int, d: int = 784, num_classes: int = 10, seed: int = 1234,
                 sample_seed: int | None = None, noise: float = 0.1):
    """Config 3: 10-class MNIST-shaped data.

    Class c has a mean image mu_c ~ U(0,1)^d and a fixed support mask keeping
    ~20% of the pixels (the "~80% zeroed" background of a digit); a sample is
    clip(mu_y + N(0, noise^2), 0, 1) on the class support and exactly 0 off it
    (noise = 0.1 in config 3; 0.25 gives a non-saturated accuracy check).
    Labels are uniform.  ``seed`` fixes the class model; ``sample_seed``
    (default seed+1) draws the samples, so train and test sets share classes.
    """
    crng = np.random.default_rng(seed)
    mu = crng.random((num_classes, d))
    support = crng.random((num_classes, d)) >= 0.8
    srng = np.random.default_rng(seed + 1 if sample_seed is None else sample_seed)
    y = srng.integers(0, num_classes, size=m)
    x = mu[y] + noise * srng.standard_normal((m, d))
    np.clip(x, 0.0, 1.0, out=x)
    x *= support[y]
    return x.astype(np.float32), y.astype(np.int64)
