"""ctypes binding of ``libmckernel_b200.so`` (the C ABI in include/mckernel_b200.h).

The library is the product: every computing entry point of this package
goes through it.  There is no CPU fallback -- if the library is missing or no
CUDA device is present, calls raise.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

LIB_PATH = Path(os.environ.get("MCK_LIB_PATH") or
                Path(__file__).resolve().parent / "libmckernel_b200.so")  # override: A/B experiments

MCK_OK, MCK_ERR_VALUE, MCK_ERR_CUDA = 0, 1, 2
MCK_KERNEL_RBF, MCK_KERNEL_MATERN = 0, 1
MCK_WHT_FAST, MCK_WHT_PARITY = 0, 1

_p = C.c_void_p
_i32, _i64, _u64, _f64 = C.c_int32, C.c_int64, C.c_uint64, C.c_double

# name -> (restype, argtypes); mirrors include/mckernel_b200.h
SIGNATURES: dict[str, tuple] = {
    "mck_abi_version": (C.c_int, []),
    "mck_last_error": (C.c_char_p, []),
    "mck_stream_key": (_u64, [_u64, C.c_char_p, _u64]),
    "mck_stream_hashes": (C.c_int, [_u64, _u64, _i64, _p, _p]),
    "mck_stream_uniforms": (C.c_int, [_u64, _u64, _i64, _p, _p]),
    "mck_stream_signs": (C.c_int, [_u64, _u64, _i64, _p, _p]),
    "mck_stream_gaussian_pairs": (C.c_int, [_u64, _u64, _i64, _p, _p]),
    "mck_fisher_yates": (C.c_int, [_u64, C.c_char_p, _u64, _i32, _i64, _p, _p]),
    "mck_tables_bytes": (_i64, [_i64, _i32]),
    "mck_tables_build": (C.c_int, [_p, _i64, _i32, _i32, _f64, _i32, _u64, _p]),
    "mck_tables_from_factors": (C.c_int, [_p, _i64, _i32, _f64, _p, _p, _p, _p, _p]),
    "mck_tables_factors": (C.c_int, [_p, _i64, _i32, _p, _p, _p, _p]),
    "mck_fwht_f32": (C.c_int, [_p, _i64, _i64, _i32, _p]),
    "mck_fwht_f64": (C.c_int, [_p, _i64, _i64, _p]),
    "mck_zhat_f32": (C.c_int, [_p, _i64, _i32, _f64, _p, _i64, _i64, _p, _p, _i64, _i32, _p]),
    "mck_features_f32": (C.c_int, [_p, _i64, _i32, _f64, _p, _i64, _i64, _p, _i32, _p, _i64,
                                   _i32, _p]),
    "mck_head_scratch_bytes": (_i64, [_i64, _i64, _i32]),
    "mck_head_forward": (C.c_int, [_p, _i64, _i64, _i64, _p, _p, _i32, _p, _p, _i64, _p, _p,
                                   _p, _p, _p, _p]),
    "mck_head_backward": (C.c_int, [_p, _i64, _i64, _i64, _p, _i32, _p, _p, _p, _p]),
    "mck_head_sgd_update": (C.c_int, [_p, _p, _p, _p, _i64, _i32, _f64, _f64, _p]),
    "mck_head_backward_sgd": (C.c_int, [_p, _i64, _i64, _i64, _p, _i32, _p, _p, _f64, _f64, _p,
                                        _p]),
    "mck_fused_scratch_bytes": (_i64, [_i64, _i64, _i32]),
    "mck_fused_scratch_bytes_ex": (_i64, [_i64, _i64, _i32, _i32, _i32]),
    "mck_fused_forward": (C.c_int, [_p, _i64, _i32, _f64, _p, _i64, _i64, _p, _p, _p, _i32, _p,
                                    _p, _i64, _p, _p, _p, _p, _p, _p, _i32, _p]),
    "mck_fused_backward": (C.c_int, [_p, _i64, _i32, _f64, _p, _i64, _i64, _p, _p, _i32, _p, _p,
                                     _p, _p, _f64, _f64, _p, _i32, _p]),
    "mck_fused_backward_bucket": (C.c_int, [_p, _i64, _i32, _f64, _p, _i64, _i64, _p, _p, _i32,
                                            _i32, _i32, _p, _p, _i32, _p]),
    "mck_fused_bias_grad": (C.c_int, [_p, _i64, _i32, _p, _p]),
    "mck_fused_apply_bucket": (C.c_int, [_p, _i64, _i32, _i32, _i32, _i32, _p, _f64, _f64, _p, _p,
                                         _p]),
    "mck_diag_umma_tf32": (C.c_int, [_p, _p, _p, _i32, _p]),
    "mck_diag_edge_color32": (C.c_int, [_i32, _p, _p, _p]),
}

_lib = None
_lock = threading.Lock()


def lib():
    """Load (once) and return the native library; raise if it is not built."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not LIB_PATH.exists():
                    raise RuntimeError(
                        f"{LIB_PATH.name} is not built; run `python -m paper_1702_08159_b200.build` "
                        "(or __graft_entry__.build()). There is no CPU fallback.")
                handle = C.CDLL(str(LIB_PATH))
                for name, (res, args) in SIGNATURES.items():
                    fn = getattr(handle, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = handle
    return _lib


def last_error() -> str:
    msg = lib().mck_last_error()
    return msg.decode() if msg else ""


def check(rc: int) -> None:
    if rc == MCK_OK:
        return
    msg = last_error()
    if rc == MCK_ERR_VALUE:
        raise ValueError(msg)
    raise RuntimeError(msg or f"native call failed with status {rc}")


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))


def ptr(t) -> int | None:
    """Device address of a torch tensor (None for None)."""
    return None if t is None else t.data_ptr()


def stream_handle(device=None) -> int:
    import torch
    return torch.cuda.current_stream(device).cuda_stream


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("a CUDA device is required (B200, sm_100a); there is no CPU fallback")
    lib()
    return torch
