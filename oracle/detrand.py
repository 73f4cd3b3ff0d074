"""Oracle restatement of the reference's hash-derived randomness.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Follows ``pkg/src/mckernel/detrand.py`` of the reference:

* ``fmix64``      -- MurmurHash3 finalizer, detrand.py:60-68 / :86-93
* ``fnv1a64``     -- label folding, detrand.py:71-75
* ``stream_key``  -- (seed, label, block) packing, detrand.py:78-83
* ``Stream``      -- counter-addressed draws, detrand.py:96-183
* ``fisher_yates``-- downward Fisher-Yates, detrand.py:186-203
* ``unit_ball``   -- n-ball points, detrand.py:216-254
"""

from __future__ import annotations

import numpy as np

M64 = (1 << 64) - 1
GAMMA = 0x9E3779B97F4A7C15
C1 = 0xFF51AFD7ED558CCD
C2 = 0xC4CEB9FE1A85EC53
FNV_OFFSET = 0xCBF29CE484222325
FNV_PRIME = 0x100000001B3
TWO_M53 = 2.0 ** -53

_G = np.uint64(GAMMA)
_C1 = np.uint64(C1)
_C2 = np.uint64(C2)
_S33 = np.uint64(33)


def fmix64(z: int) -> int:
    """detrand.py:60-68 -- three xor-shift-33 steps around two multiplies."""
    z &= M64
    z = ((z ^ (z >> 33)) * C1) & M64
    z = ((z ^ (z >> 33)) * C2) & M64
    return z ^ (z >> 33)


def fmix64_np(z: np.ndarray) -> np.ndarray:
    """Vector form of :func:`fmix64` on uint64 (wraps mod 2^64)."""
    z = z ^ (z >> _S33)
    z = z * _C1
    z = z ^ (z >> _S33)
    z = z * _C2
    return z ^ (z >> _S33)


def fnv1a64(data: bytes) -> int:
    """detrand.py:71-75."""
    h = FNV_OFFSET
    for byte in data:
        h = ((h ^ byte) * FNV_PRIME) & M64
    return h


def stream_key(seed: int, label: str, block: int) -> int:
    """detrand.py:78-83: key = f(f(f(seed) ^ fnv(label)) ^ block*GAMMA)."""
    k = fmix64(seed & M64)
    k = fmix64(k ^ fnv1a64(label.encode("utf-8")))
    return fmix64(k ^ ((block * GAMMA) & M64))


class Stream:
    """Counter-addressed draw stream (detrand.py:96-183).

    ``hashes(count)`` returns fmix64(key + c*GAMMA) for the next ``count``
    counters; distributions are layered on top exactly as the reference
    does, including the cached second Box-Muller variate.
    """

    def __init__(self, seed: int, label: str, block: int = 0):
        if block < 0:
            raise ValueError("block index must be non-negative")
        self.key = stream_key(seed, label, block)
        self.counter = 0
        self.pending: float | None = None

    def hash_at(self, counter: int) -> int:
        return fmix64((self.key + counter * GAMMA) & M64)

    def hashes(self, count: int) -> np.ndarray:
        # detrand.py:128-132
        c = np.arange(self.counter, self.counter + count, dtype=np.uint64)
        self.counter += count
        with np.errstate(over="ignore"):
            return fmix64_np(np.uint64(self.key) + c * _G)

    def uniforms(self, count: int) -> np.ndarray:
        # detrand.py:139-142: top 53 bits * 2^-53
        return (self.hashes(count) >> np.uint64(11)).astype(np.float64) * TWO_M53

    def signs(self, count: int) -> np.ndarray:
        # detrand.py:147-150: top bit set -> +1.0 else -1.0
        top = (self.hashes(count) >> np.uint64(63)).astype(bool)
        return np.where(top, 1.0, -1.0)

    def gaussians(self, count: int) -> np.ndarray:
        # detrand.py:155-171 (pair caching)
        out = np.empty(count, dtype=np.float64)
        pos = 0
        if self.pending is not None and count > 0:
            out[0] = self.pending
            self.pending = None
            pos = 1
        m = count - pos
        if m <= 0:
            return out
        pairs = (m + 1) // 2
        z = box_muller(self.uniforms(2 * pairs))
        out[pos:] = z[:m]
        if m & 1:
            self.pending = float(z[m])
        return out


def box_muller(u: np.ndarray) -> np.ndarray:
    """detrand.py:174-183: (u1,u2) -> (r cos 2pi u2, r sin 2pi u2).

    u1 == 0 maps to 2^-53; 2*pi is formed in double first (``2.0 * np.pi``)
    and then multiplied by u2, which fixes the rounding of the argument.
    """
    u1 = u[0::2].copy()
    u2 = u[1::2]
    u1[u1 == 0.0] = TWO_M53
    r = np.sqrt(-2.0 * np.log(u1))
    ang = 2.0 * np.pi * u2
    z = np.empty_like(u)
    z[0::2] = r * np.cos(ang)
    z[1::2] = r * np.sin(ang)
    return z


def fisher_yates(stream: Stream, n: int) -> np.ndarray:
    """detrand.py:186-203: downward swaps, j = int(u_k * (i+1)) clamped to i.

    The n-1 uniforms are drawn up front; step k uses i = n-1-k.
    """
    if n < 1:
        raise ValueError("empty permutation")
    perm = np.arange(n, dtype=np.int64)
    if n == 1:
        return perm
    u = stream.uniforms(n - 1)
    i = np.arange(n - 1, 0, -1, dtype=np.int64)
    j = np.minimum((u * (i + 1).astype(np.float64)).astype(np.int64), i)
    p = perm.tolist()
    for ii, jj in zip(i.tolist(), j.tolist()):
        p[ii], p[jj] = p[jj], p[ii]
    return np.asarray(p, dtype=np.int64)


def unit_ball(stream: Stream, count: int, n: int, r: float = 1.0) -> np.ndarray:
    """detrand.py:216-254: ``count`` points r*U^(1/n)*X/|X| in the n-ball.

    Per point the stream yields n gaussians then one uniform; the even-n
    fast path reads them as one (count, n+1) block of uniforms.
    """
    if n < 1 or r <= 0.0 or count < 1:
        raise ValueError("bad unit-ball arguments")
    if n % 2 == 0 and stream.pending is None:
        u = stream.uniforms(count * (n + 1)).reshape(count, n + 1)
        x = box_muller_rows(u[:, :n])
        ub = u[:, n]
    else:
        x = np.empty((count, n), dtype=np.float64)
        ub = np.empty(count, dtype=np.float64)
        for k in range(count):
            x[k] = stream.gaussians(n)
            ub[k] = stream.uniforms(1)[0]
    norms = np.sqrt((x * x).sum(axis=-1))
    while (norms == 0.0).any():          # probability zero; kept for parity
        for k in np.flatnonzero(norms == 0.0):
            x[k] = stream.gaussians(n)
        norms = np.sqrt((x * x).sum(axis=-1))
    scale = r * ub ** (1.0 / n) / norms
    return x * scale[:, None]


def box_muller_rows(u: np.ndarray) -> np.ndarray:
    """Row-wise Box-Muller on an (m, even n) uniform block (detrand.py:233-239)."""
    u1 = u[:, 0::2].copy()
    u2 = u[:, 1::2]
    u1[u1 == 0.0] = TWO_M53
    rad = np.sqrt(-2.0 * np.log(u1))
    ang = 2.0 * np.pi * u2
    x = np.empty(u.shape, dtype=np.float64)
    x[:, 0::2] = rad * np.cos(ang)
    x[:, 1::2] = rad * np.sin(ang)
    return x
