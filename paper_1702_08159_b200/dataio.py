"""On-disk formats shared with the reference (``pkg/src/mckernel/dataio.py``).

* ``MCKMAT4`` / ``MCKMAT8`` / ``MCKMATi4`` matrix records: 8-byte magic, rows
  and cols as little-endian uint32, row-major data (dataio.py:9-16, :208-229)
  -- the format of the reference's ``features`` dump (cli.py:221-247).
* ``features_to_file``: the GPU equivalent of ``mckernel features``: rows are
  expanded batch by batch on the device and streamed into one MCKMAT4 file, so
  a dump of any size never needs the whole feature matrix in memory.
"""

from __future__ import annotations

import struct

import numpy as np

MAGIC_F32 = b"MCKMAT4\n"
MAGIC_F64 = b"MCKMAT8\n"
MAGIC_I32 = b"MCKMATi4"
_DTYPE_MAGIC = {np.dtype(np.float32): MAGIC_F32, np.dtype(np.float64): MAGIC_F64,
                np.dtype(np.int32): MAGIC_I32}
_MAGIC_DTYPE = {v: k for k, v in _DTYPE_MAGIC.items()}


def write_matrix_record(f, arr) -> None:
    """dataio.py:208-217."""
    arr = np.ascontiguousarray(arr)
    magic = _DTYPE_MAGIC.get(arr.dtype)
    if magic is None:
        raise ValueError(f"unsupported record dtype {arr.dtype}")
    if arr.ndim != 2:
        raise ValueError("records hold 2-D matrices")
    f.write(magic)
    f.write(struct.pack("<II", arr.shape[0], arr.shape[1]))
    f.write(arr.tobytes())


def read_matrix_record(f) -> np.ndarray:
    """dataio.py:220-229."""
    magic = f.read(8)
    dtype = _MAGIC_DTYPE.get(magic)
    if dtype is None:
        raise ValueError(f"unknown record magic {magic!r}")
    rows, cols = struct.unpack("<II", f.read(8))
    data = f.read(rows * cols * dtype.itemsize)
    if len(data) != rows * cols * dtype.itemsize:
        raise ValueError("truncated matrix record")
    return np.frombuffer(data, dtype=dtype).reshape(rows, cols).copy()


def write_matrix(path, arr) -> None:
    with open(path, "wb") as f:
        write_matrix_record(f, arr)


def read_matrix(path) -> np.ndarray:
    with open(path, "rb") as f:
        return read_matrix_record(f)


def features_to_file(spec, blocks, x, path, *, normalize: bool = True,
                     batch_rows: int = 4096) -> tuple[int, int]:
    """Expand rows of ``x`` on the GPU and stream them into an MCKMAT4 file.

    Same bytes as the reference's ``write_matrix(out, feature_map_batch(...))``
    up to the feature tolerance (normalised features within 1e-5/1e-6).
    Returns (rows, cols).
    """
    from . import _native as nat
    from . import fastfood
    torch = nat.require_cuda()
    bs = fastfood._as_blockset(spec, blocks)
    xt = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x, np.float32))
    m = int(xt.shape[0])
    width = fastfood.feature_dim(spec)
    out = torch.empty((min(batch_rows, max(m, 1)), width), dtype=torch.float32, device=bs.device)
    host = torch.empty(out.shape, dtype=torch.float32, pin_memory=True)
    with open(path, "wb") as f:
        f.write(MAGIC_F32)
        f.write(struct.pack("<II", m, width))
        for r0 in range(0, m, batch_rows):
            r1 = min(m, r0 + batch_rows)
            xb = xt[r0:r1].to(bs.device, torch.float32)
            fastfood.feature_map_batch(spec, bs, xb, normalize=normalize, out=out)
            host[:r1 - r0].copy_(out[:r1 - r0])
            f.write(host[:r1 - r0].numpy().tobytes())
    return m, width
