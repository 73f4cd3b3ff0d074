"""Oracle restatement of the reference Fastfood feature map.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Follows ``pkg/src/mckernel/fastfood.py``:

* ``OSpec``            -- FeatureMapSpec / RBF / RBFMatern, fastfood.py:32-79
* ``calibration_rbf``  -- fastfood.py:96-107
* ``calibration_matern`` -- fastfood.py:110-130
* ``build_block``      -- fastfood.py:133-162 (streams "B", "Pi", "G", "C")
* ``apply_zhat_batch`` -- fastfood.py:179-198
* ``feature_map_batch``-- fastfood.py:209-226
* ``dense_zhat``       -- fastfood.py:248-259

``wht`` selects the transform: ``"reference"`` (sgemm base, bit-equal to the
reference on the same BLAS) or ``"sequential"`` (BLAS-independent restatement).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import detrand
from . import wht as owht

F32 = np.float32


@dataclass(frozen=True)
class OSpec:
    input_dim: int
    expansions: int
    kind: str            # "rbf" | "matern"
    sigma: float
    t: int
    seed: int

    @property
    def n(self) -> int:
        # next_pow2, fastfood.py:59-62
        return 1 << (self.input_dim - 1).bit_length()

    @classmethod
    def of(cls, spec) -> "OSpec":
        """Accept the product's or the reference's FeatureMapSpec (duck-typed)."""
        k = spec.kernel
        t = getattr(k, "t", 0)
        kind = "matern" if t else "rbf"
        return cls(spec.input_dim, spec.expansions, kind, float(k.sigma), int(t), int(spec.seed))


@dataclass(frozen=True)
class OBlock:
    b_signs: np.ndarray      # float32 +-1
    permutation: np.ndarray  # int64
    g_diag: np.ndarray       # float32
    c_diag: np.ndarray       # float32
    block_index: int


def calibration_rbf(stream: detrand.Stream, n: int, g: np.ndarray) -> np.ndarray:
    """fastfood.py:96-107: c_i = |n fresh gaussians| / |g| (float64)."""
    g_norm = float(np.sqrt((g.astype(np.float64) ** 2).sum()))
    if g_norm == 0.0:
        raise ValueError("degenerate gaussian diagonal")
    out = np.empty(n, dtype=np.float64)
    rows = max(1, (1 << 22) // n)       # bounded memory; same draws, same order
    for r0 in range(0, n, rows):
        k = min(rows, n - r0)
        d = stream.gaussians(k * n).reshape(k, n)
        out[r0:r0 + k] = np.sqrt((d * d).sum(axis=1))
    return out / g_norm


def calibration_matern(stream: detrand.Stream, n: int, t: int) -> np.ndarray:
    """fastfood.py:110-130: c_e = |sum of t unit-ball points| (float64)."""
    if t < 1:
        raise ValueError("t must be a positive integer")
    out = np.empty(n, dtype=np.float64)
    per = t * (n + 1)
    chunk = max(1, (1 << 22) // max(per, 1))
    done = 0
    while done < n:
        k = min(chunk, n - done)
        balls = detrand.unit_ball(stream, k * t, n, 1.0)
        sums = balls.reshape(k, t, n).sum(axis=1)
        out[done:done + k] = np.sqrt((sums * sums).sum(axis=1))
        done += k
    return out


def build_block(spec: OSpec, e: int) -> OBlock:
    """fastfood.py:133-162."""
    if not 0 <= e < spec.expansions:
        raise ValueError(f"block index {e} outside 0..{spec.expansions - 1}")
    n, seed = spec.n, spec.seed
    b = detrand.Stream(seed, "B", e).signs(n)
    perm = detrand.fisher_yates(detrand.Stream(seed, "Pi", e), n)
    g = detrand.Stream(seed, "G", e).gaussians(n)
    cs = detrand.Stream(seed, "C", e)
    if spec.kind == "rbf":
        c = calibration_rbf(cs, n, g)
    else:
        g_norm = float(np.sqrt((g * g).sum()))
        if g_norm == 0.0:
            raise ValueError("degenerate gaussian diagonal")
        c = calibration_matern(cs, n, spec.t) / g_norm
    return OBlock(b.astype(F32), perm, g.astype(F32), c.astype(F32), e)


def build_blocks(spec: OSpec) -> list[OBlock]:
    return [build_block(spec, e) for e in range(spec.expansions)]


def rbf_c_entries(spec: OSpec, e: int, entries: np.ndarray) -> np.ndarray:
    """C-RBF values for selected entries only (counter = i*n, fastfood.py:106-107).

    Used to check the n=16384 configuration without drawing all n^2 gaussians.
    """
    n = spec.n
    g = detrand.Stream(spec.seed, "G", e).gaussians(n)
    g_norm = float(np.sqrt((g.astype(np.float64) ** 2).sum()))
    out = np.empty(len(entries), dtype=np.float64)
    for k, i in enumerate(entries):
        s = detrand.Stream(spec.seed, "C", e)
        s.counter = int(i) * n          # n even: rows start on a pair boundary
        d = s.gaussians(n)
        out[k] = np.sqrt((d * d).sum())
    return (out / g_norm).astype(F32)


def apply_zhat_batch(spec: OSpec, blocks, x: np.ndarray, wht: str = "reference") -> np.ndarray:
    """fastfood.py:179-198: per block pad -> *B -> H -> gather -> *G -> H -> *C -> *scale."""
    if len(blocks) != spec.expansions:
        raise ValueError(f"expected {spec.expansions} blocks, got {len(blocks)}")
    x = np.atleast_2d(np.asarray(x, dtype=F32))
    if x.shape[-1] != spec.input_dim:
        raise ValueError(f"input has {x.shape[-1]} features, spec expects {spec.input_dim}")
    n = spec.n
    scale = F32(1.0 / (spec.sigma * np.sqrt(n)))
    out = np.empty((x.shape[0], n * spec.expansions), dtype=F32)
    for blk in blocks:
        v = np.zeros((x.shape[0], n), dtype=F32)
        v[:, :spec.input_dim] = x
        v *= blk.b_signs
        v = _wht(v, wht)
        v = np.ascontiguousarray(v[:, blk.permutation])
        v *= blk.g_diag
        v = _wht(v, wht)
        v *= blk.c_diag
        v *= scale
        e = blk.block_index
        out[:, e * n:(e + 1) * n] = v
    return out


def _wht(v: np.ndarray, which: str) -> np.ndarray:
    if which == "reference":
        return owht.wht_fast_batch(v)
    if which == "sequential":
        return owht.wht_sequential(v)
    if which == "f64":
        return owht.wht_butterfly_f64(v).astype(F32)
    raise ValueError(which)


def feature_map_batch(spec: OSpec, blocks, x: np.ndarray, normalize: bool = True,
                      wht: str = "reference") -> np.ndarray:
    """fastfood.py:209-226: [cos z | sin z], times float32(1/sqrt(D)) if normalize."""
    z = apply_zhat_batch(spec, blocks, x, wht)
    d = z.shape[1]
    out = np.empty((z.shape[0], 2 * d), dtype=F32)
    np.cos(z, out=out[:, :d])
    np.sin(z, out=out[:, d:])
    if normalize:
        out *= F32(1.0 / np.sqrt(d))
    return out


def dense_zhat(spec: OSpec, blk: OBlock) -> np.ndarray:
    """fastfood.py:248-259: explicit (C H G P H B)/(sigma sqrt n) in float64."""
    n = spec.n
    h = owht.hadamard(n)
    p = np.zeros((n, n))
    p[np.arange(n), blk.permutation] = 1.0
    z = (np.diag(blk.c_diag.astype(np.float64)) @ h @ np.diag(blk.g_diag.astype(np.float64))
         @ p @ h @ np.diag(blk.b_signs.astype(np.float64)))
    return z / (spec.sigma * np.sqrt(n))
