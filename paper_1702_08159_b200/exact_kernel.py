"""Statistical check of the GPU feature map against the exact RBF kernel.

Mirror of ``kernel_check`` (``pkg/src/mckernel/exact_kernel.py:137-163``):
<phi(x), phi(x')> from the GPU features (normalised) against
exp(-|x - x'|^2 / (2 sigma^2)) in float64, over pairs of inputs.  The rest of
the reference module (Gram matrices, ridge and V-matrix solvers) is an exact
desk-scale oracle and out of scope here.
"""

from __future__ import annotations

from dataclasses import asdict, dataclass

import numpy as np

from . import _native as nat
from . import fastfood


@dataclass
class KernelCheckStats:
    dims: int
    D: int
    pairs: int
    mean_err: float
    max_err: float
    ref_scale: float       # Monte-Carlo scale 1/sqrt(D)

    def to_dict(self) -> dict:
        return asdict(self)


def rbf_kernel(x, y, sigma: float) -> float:
    """exact_kernel.py:22-31."""
    if sigma <= 0.0:
        raise ValueError("sigma must be positive")
    d = np.asarray(x, dtype=np.float64) - np.asarray(y, dtype=np.float64)
    return float(np.exp(-(d @ d) / (2.0 * sigma * sigma)))


def kernel_check(spec, pairs, blocks=None) -> KernelCheckStats:
    """exact_kernel.py:137-163, with the features computed on the GPU."""
    if not isinstance(spec.kernel, fastfood.RBF):
        raise ValueError("kernel_check requires an RBF spec")
    if not pairs:
        raise ValueError("need at least one pair")
    torch = nat.require_cuda()
    if blocks is None:
        blocks = fastfood.build_blocks(spec)
    xs = np.stack([np.asarray(p[0], dtype=np.float32) for p in pairs])
    ys = np.stack([np.asarray(p[1], dtype=np.float32) for p in pairs])
    fx = fastfood.feature_map_batch(spec, blocks, torch.from_numpy(xs).cuda()).double()
    fy = fastfood.feature_map_batch(spec, blocks, torch.from_numpy(ys).cuda()).double()
    approx = (fx * fy).sum(dim=1).cpu().numpy()
    s = spec.kernel.sigma
    diff = xs.astype(np.float64) - ys.astype(np.float64)
    exact = np.exp(-(diff * diff).sum(axis=1) / (2.0 * s * s))
    err = np.abs(approx - exact)
    d = spec.padded_dim * spec.expansions
    return KernelCheckStats(dims=spec.input_dim, D=d, pairs=len(pairs), mean_err=float(err.mean()),
                            max_err=float(err.max()), ref_scale=float(1.0 / np.sqrt(d)))
