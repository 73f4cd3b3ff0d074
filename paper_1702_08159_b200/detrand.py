"""Device-side deterministic streams -- mirror of ``mckernel.detrand``.

The pinned mixer (MurmurHash3 fmix64 over key + counter*GAMMA, FNV-1a label
folding, detrand.py:60-93) is evaluated by the CUDA library; these wrappers
keep the reference's counter semantics (detrand.py:96-183), including the
cached second Box-Muller variate, and return torch CUDA tensors.
"""

from __future__ import annotations

from . import _native as nat

MASK64 = (1 << 64) - 1


def stream_key(seed: int, label: str, block: int) -> int:
    """detrand.py:78-83 (computed by the library)."""
    return int(nat.lib().mck_stream_key(seed & MASK64, label.encode("utf-8"), block & MASK64))


class RandomStream:
    """Counter-addressed stream whose draws are computed on the GPU."""

    def __init__(self, seed: int, label: str, block: int = 0, device=None):
        if block < 0:
            raise ValueError("block index must be non-negative")
        self.seed = seed & MASK64
        self.label = label
        self.block = block
        self.counter = 0
        self.key = stream_key(seed, label, block)
        self.device = device
        self._pending = None

    def _torch(self):
        return nat.require_cuda()

    def _dev(self):
        torch = self._torch()
        return torch.device(self.device) if self.device is not None else torch.device("cuda")

    def hashes(self, count: int):
        """uint64 draws (returned as int64 bit patterns)."""
        torch = self._torch()
        out = torch.empty(count, dtype=torch.int64, device=self._dev())
        nat.call("mck_stream_hashes", self.key, self.counter, count, nat.ptr(out),
                 nat.stream_handle(out.device))
        self.counter += count
        return out

    def hash64(self) -> int:
        """Mixer output at the current counter; does not advance (detrand.py:124-126)."""
        c = self.counter
        v = int(self.hashes(1)[0].item()) & MASK64
        self.counter = c
        return v

    def uniform01_array(self, count: int):
        torch = self._torch()
        out = torch.empty(count, dtype=torch.float64, device=self._dev())
        nat.call("mck_stream_uniforms", self.key, self.counter, count, nat.ptr(out),
                 nat.stream_handle(out.device))
        self.counter += count
        return out

    def sign_array(self, count: int):
        torch = self._torch()
        out = torch.empty(count, dtype=torch.float64, device=self._dev())
        nat.call("mck_stream_signs", self.key, self.counter, count, nat.ptr(out),
                 nat.stream_handle(out.device))
        self.counter += count
        return out

    def uniform01(self) -> float:
        """One uniform in [0, 1) (detrand.py:136-137)."""
        return float(self.uniform01_array(1)[0].item())

    def sign_pm1(self) -> float:
        """One +-1 draw (detrand.py:144-145)."""
        return float(self.sign_array(1)[0].item())

    def gaussian(self) -> float:
        """One standard normal, sharing the pair cache with gaussian_array
        (detrand.py:152-153)."""
        return float(self.gaussian_array(1)[0].item())

    def gaussian_array(self, count: int):
        """detrand.py:155-171 with the cached second variate."""
        torch = self._torch()
        out = torch.empty(count, dtype=torch.float64, device=self._dev())
        pos = 0
        if self._pending is not None and count > 0:
            out[0] = self._pending
            self._pending = None
            pos = 1
        m = count - pos
        if m <= 0:
            return out
        pairs = (m + 1) // 2
        z = torch.empty(2 * pairs, dtype=torch.float64, device=self._dev())
        nat.call("mck_stream_gaussian_pairs", self.key, self.counter, pairs, nat.ptr(z),
                 nat.stream_handle(z.device))
        self.counter += 2 * pairs
        out[pos:] = z[:m]
        if m & 1:
            self._pending = z[m].clone()
        return out


def fisher_yates_permutations(seed: int, label: str, block0: int, count: int, n: int, device=None):
    """``count`` permutations of {0..n-1} for streams (seed, label, block0+b) (detrand.py:186-203)."""
    torch = nat.require_cuda()
    dev = torch.device(device) if device is not None else torch.device("cuda")
    out = torch.empty((count, n), dtype=torch.int32, device=dev)
    nat.call("mck_fisher_yates", seed & MASK64, label.encode("utf-8"), block0, count, n,
             nat.ptr(out), nat.stream_handle(dev))
    return out


def fisher_yates_permutation(stream: RandomStream, n: int):
    """Permutation for ``stream`` (fresh counter), as an int64 CUDA tensor."""
    if n < 1:
        raise ValueError("empty permutation")
    if stream.counter != 0:
        raise ValueError("device Fisher-Yates needs a fresh stream (counter 0)")
    p = fisher_yates_permutations(stream.seed, stream.label, stream.block, 1, n, stream.device)[0]
    stream.counter += n - 1
    return p.long()
