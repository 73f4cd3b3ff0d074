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
