"""Oracle restatement of the reference Walsh-Hadamard transforms.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Follows ``pkg/src/mckernel/wht.py``:

* ``hadamard``       -- dense H with (-1)^popcount(i&j), wht.py:54-64
* ``wht_naive``      -- float64 matrix product oracle, wht.py:67-87
* ``wht_fast_batch`` -- the reference's own pipeline transform, wht.py:103-162:
  every aligned base chunk (256) is multiplied by dense H_256 through
  ``np.matmul`` (OpenBLAS sgemm, 64-row chunks), then combine stages
  h = 256..n/2 compute ``a <- a+b ; b <- (a+b) - 2b``.
* ``wht_sequential`` -- the same arithmetic with the base written out as the
  sequential k = 0..base-1 fp32 sum that OpenBLAS' SkylakeX sgemm performs
  (SURVEY.md section 0.3); it does not depend on the BLAS build and is what
  the CUDA ``parity`` variant reproduces bit for bit.
"""

from __future__ import annotations

import numpy as np

BASE = 256          # wht.py:26
CHUNK_ROWS = 64     # wht.py:27


def is_pow2(n: int) -> bool:
    return n > 0 and (n & (n - 1)) == 0


def _check(n: int) -> None:
    if not is_pow2(n):
        raise ValueError(f"length {n} is not a power of two")


def hadamard(n: int, dtype=np.float64) -> np.ndarray:
    """wht.py:54-64: entry (i, j) = (-1)^popcount(i & j)."""
    _check(n)
    i = np.arange(n, dtype=np.uint32)
    par = np.bitwise_count(i[:, None] & i[None, :]) & 1
    return np.where(par == 1, -1.0, 1.0).astype(dtype)


def wht_naive(v: np.ndarray) -> np.ndarray:
    """wht.py:67-87: float64 H @ v for a vector or the columns of a matrix."""
    x = np.asarray(v, dtype=np.float64)
    single = x.ndim == 1
    if single:
        x = x[:, None]
    n = x.shape[0]
    _check(n)
    out = np.empty_like(x)
    j = np.arange(n, dtype=np.uint32)
    rows = max(1, min(n, (1 << 22) // n))
    for r0 in range(0, n, rows):
        i = np.arange(r0, min(r0 + rows, n), dtype=np.uint32)
        s = np.where(np.bitwise_count(i[:, None] & j[None, :]) & 1, -1.0, 1.0)
        out[r0:r0 + len(i)] = s @ x
    return out[:, 0] if single else out


def _combine(v: np.ndarray, start: int, n: int) -> None:
    """wht.py:115-126: spans start..n/2, (a, b) <- (a+b, (a+b) - 2b)."""
    h = start
    while h < n:
        view = v.reshape(v.shape[:-1] + (-1, 2, h))
        a = view[..., 0, :]
        b = view[..., 1, :]
        a += b
        b *= 2.0
        np.subtract(a, b, out=b)
        h <<= 1


def _validate(v: np.ndarray) -> int:
    # wht.py:150-158 (same messages)
    n = v.shape[-1]
    _check(n)
    if not v.flags.c_contiguous:
        raise ValueError("transform buffer must be C-contiguous")
    if not np.issubdtype(v.dtype, np.floating):
        raise ValueError("transform buffer must be a float array")
    return n


def wht_fast_batch(mat: np.ndarray, base_size: int = BASE) -> np.ndarray:
    """wht.py:142-162: in place on each row; returns its argument."""
    if mat.ndim != 2:
        raise ValueError("wht_fast_batch expects an (m, n) array")
    n = _validate(mat)
    base = min(n, base_size)
    flat = mat.reshape(-1, base)
    h = hadamard(base, flat.dtype)
    scratch = np.empty((min(CHUNK_ROWS, flat.shape[0]), base), dtype=flat.dtype)
    for i in range(0, flat.shape[0], CHUNK_ROWS):      # wht.py:108-112
        chunk = flat[i:i + CHUNK_ROWS]
        out = scratch[:chunk.shape[0]]
        np.matmul(chunk, h, out=out)
        chunk[:] = out
    if base < n:
        _combine(mat, base, n)
    return mat


def wht_sequential(mat: np.ndarray, base_size: int = BASE) -> np.ndarray:
    """BLAS-independent restatement of ``wht_fast_batch`` (returns a new array).

    Each base output y_j = sum_k H[k, j] x_k accumulated in fp32 in the order
    k = 0, 1, ..., base-1 (products by +-1 are exact), then the same combine
    stages.  Equal bit for bit to the reference on OpenBLAS SkylakeX for
    every chunk of >= 2 rows.
    """
    m = np.array(mat, dtype=np.float32, copy=True)
    n = _validate(m)
    base = min(n, base_size)
    flat = m.reshape(-1, base)
    h = hadamard(base, np.float32)
    acc = np.zeros_like(flat)
    for k in range(base):
        acc += flat[:, k:k + 1] * h[k][None, :]
    flat[:] = acc
    if base < n:
        _combine(m, base, n)
    return m


def wht_butterfly_f64(mat: np.ndarray) -> np.ndarray:
    """Radix-2 butterflies in float64 on the last axis (wht.py:90-100 order)."""
    v = np.array(mat, dtype=np.float64, copy=True)
    n = v.shape[-1]
    _check(n)
    h = 1
    while h < n:
        view = v.reshape(v.shape[:-1] + (-1, 2, h))
        a = view[..., 0, :].copy()
        b = view[..., 1, :]
        view[..., 0, :] = a + b
        view[..., 1, :] = a - b
        h <<= 1
    return v
