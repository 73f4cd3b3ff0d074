"""Batched Walsh-Hadamard transform on B200 -- drop-in for ``mckernel.wht``.

``wht_fast_batch`` / ``wht_fast`` keep the reference's in-place contract,
return value and error messages (``pkg/src/mckernel/wht.py:129-162``) and run
``mck_fwht_f32`` / ``mck_fwht_f64`` (K1).  numpy buffers are transformed on
the device and copied back into the same array; torch CUDA tensors are
transformed in place on the current stream.

``base_size`` is validated as in the reference but does not change the
result beyond roundoff (the reference uses it only for cache blocking);
``variant="parity"`` selects the bit-exact restatement of the reference's
base-256 arithmetic (fp32 only).
"""

from __future__ import annotations

import numpy as np

from . import _native as nat

DEFAULT_BASE_SIZE = 256


def is_power_of_two(n: int) -> bool:
    return n > 0 and (n & (n - 1)) == 0


def _check_pow2(n: int) -> None:
    if not is_power_of_two(n):
        raise ValueError(f"length {n} is not a power of two")


def _transform(v, base_size: int, variant: str):
    # wht.py:150-162 validation order and messages
    n = int(v.shape[-1])
    _check_pow2(n)
    if not is_power_of_two(base_size):
        raise ValueError(f"base size {base_size} is not a power of two")
    torch = nat.require_cuda()
    if isinstance(v, torch.Tensor):
        if not v.is_contiguous():
            raise ValueError("transform buffer must be C-contiguous")
        if not v.is_floating_point():
            raise ValueError("transform buffer must be a float array")
        if not v.is_cuda:
            dev = v.to("cuda")
            _device_transform(dev, n, variant)
            v.copy_(dev.cpu())
            return v
        if v.dtype not in (torch.float32, torch.float64):
            raise ValueError("transform buffer must be float32 or float64")
        _device_transform(v, n, variant)
        return v
    if not v.flags.c_contiguous:
        raise ValueError("transform buffer must be C-contiguous")
    if not np.issubdtype(v.dtype, np.floating):
        raise ValueError("transform buffer must be a float array")
    if v.dtype not in (np.float32, np.float64):
        raise ValueError("transform buffer must be float32 or float64")
    dev = torch.from_numpy(v).to("cuda")
    _device_transform(dev, n, variant)
    v[...] = dev.cpu().numpy()
    return v


def _device_transform(t, n: int, variant: str):
    torch = nat.require_cuda()
    rows = t.numel() // n if n else 0
    if t.data_ptr() % 16:
        raise ValueError("transform buffer must be 16-byte aligned")
    st = nat.stream_handle(t.device)
    if t.dtype == torch.float32:
        code = {"fast": nat.MCK_WHT_FAST, "parity": nat.MCK_WHT_PARITY}.get(variant)
        if code is None:
            raise ValueError(f"unknown variant {variant!r}")
        nat.call("mck_fwht_f32", nat.ptr(t), rows, n, code, st)
    else:
        if variant != "fast":
            raise ValueError("the parity variant is float32 only")
        nat.call("mck_fwht_f64", nat.ptr(t), rows, n, st)


def wht_fast(v, base_size: int = DEFAULT_BASE_SIZE, *, variant: str = "fast"):
    """In-place transform of a 1-D float buffer; returns its argument (wht.py:129-139)."""
    if v.ndim != 1:
        raise ValueError("wht_fast expects a 1-D buffer; see wht_fast_batch")
    return _transform(v, base_size, variant)


def wht_fast_batch(mat, base_size: int = DEFAULT_BASE_SIZE, *, variant: str = "fast"):
    """Transform every row of a contiguous (m, n) array in place (wht.py:142-147)."""
    if mat.ndim != 2:
        raise ValueError("wht_fast_batch expects an (m, n) array")
    return _transform(mat, base_size, variant)


# -- benchmark (wht.py:165-205; paper Table 1) -------------------------------

from dataclasses import dataclass  # noqa: E402


@dataclass
class BenchRecord:
    size: int
    fast_ms: float
    naive_ms: float | None
    reps: int


def _naive_gpu(torch, v):
    """The reference's naive oracle (wht.py:67-87) on the GPU: float64 product
    with sign rows (-1)^popcount(i & j) generated in bounded chunks (the same
    2^22-entry chunks), O(n^2) work and a fixed memory footprint."""
    n = v.shape[0]
    x = v.to(torch.float64)
    out = torch.empty_like(x)
    j = torch.arange(n, device=v.device, dtype=torch.int64)
    rows = max(1, min(n, (1 << 22) // n))
    for r0 in range(0, n, rows):
        i = torch.arange(r0, min(r0 + rows, n), device=v.device, dtype=torch.int64)
        a = i[:, None] & j[None, :]
        for sh in (16, 8, 4, 2, 1):              # parity of popcount
            a = a ^ (a >> sh)
        signs = 1.0 - 2.0 * (a & 1).to(torch.float64)
        out[r0:r0 + len(i)] = signs @ x
    return out


def wht_naive(v):
    """Transform by explicit +-1 matrix product in float64 (wht.py:67-87), on
    the GPU: a vector of length n or an (n, k) matrix of k column vectors;
    returns a new float64 array (numpy in -> numpy out)."""
    torch = nat.require_cuda()
    host = not isinstance(v, torch.Tensor)
    t = torch.from_numpy(np.asarray(v, dtype=np.float64)) if host else v
    single = t.dim() == 1
    if t.dim() not in (1, 2):
        raise ValueError("wht_naive expects a vector or an (n, k) matrix")
    _check_pow2(int(t.shape[0]))
    t = t.to(device="cuda", dtype=torch.float64)
    out = _naive_gpu(torch, t if not single else t[:, None])
    out = out[:, 0] if single else out
    return out.cpu().numpy() if host else out


def bench_wht(sizes, repetitions: int = 5, naive_cutoff: int = 1 << 16, dtype=np.float32):
    """Median device time per single-vector transform (CUDA events), Table-1 style.

    ``fast_ms`` times ``mck_fwht_f32`` on one resident vector of each size
    (the reference times ``wht_fast`` on the host, wht.py:183-205).
    ``naive_ms`` times the reference's naive oracle (float64 product with
    chunk-generated sign rows, wht.py:67-87) on the GPU up to
    ``naive_cutoff`` (2^16 by default, as the reference).
    """
    if repetitions < 3:
        raise ValueError("repetitions must be at least 3")
    for s in sizes:
        _check_pow2(s)
    torch = nat.require_cuda()
    rng = np.random.default_rng(0)
    recs = []
    for size in sizes:
        proto = torch.from_numpy(rng.standard_normal(size).astype(dtype)).cuda()

        def med(fn):
            times = []
            for _ in range(repetitions):
                buf = proto.clone()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                fn(buf)
                e.record()
                e.synchronize()
                times.append(s.elapsed_time(e))
            return float(np.median(times))

        wht_fast(proto.clone())                     # warm-up
        fast = med(wht_fast)
        naive = None
        if size <= naive_cutoff:
            naive = med(lambda b: _naive_gpu(torch, b))
        recs.append(BenchRecord(size, fast, naive, repetitions))
    return recs


def bench_wht_csv(records) -> str:
    """CSV ``size,impl,median_ms,reps`` exactly as ``mckernel bench-wht`` (cli.py:115-132)."""
    lines = ["size,impl,median_ms,reps"]
    for r in records:
        lines.append(f"{r.size},fast,{r.fast_ms:.6f},{r.reps}")
        if r.naive_ms is not None:
            lines.append(f"{r.size},naive,{r.naive_ms:.6f},{r.reps}")
    return "\n".join(lines) + "\n"
