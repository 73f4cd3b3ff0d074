"""Fastfood feature map on B200 -- drop-in for ``mckernel.fastfood``.

Same names, arguments, validation and error messages as the reference
(``pkg/src/mckernel/fastfood.py``); the computation runs in
``libmckernel_b200.so``:

* ``build_blocks``      -> ``mck_tables_build``  (fastfood.py:133-166, K2)
* ``apply_zhat_batch``  -> ``mck_zhat_f32``      (fastfood.py:179-198, K3)
* ``feature_map_batch`` -> ``mck_features_f32``  (fastfood.py:209-226, K3)

Array conventions: numpy in -> numpy out (host copies, like the reference);
torch CUDA tensors in -> torch CUDA tensors out, computed on the current
stream without host synchronisation.
"""

from __future__ import annotations

import functools
from collections.abc import Sequence
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat

PIPELINE_DTYPE = np.float32


@dataclass(frozen=True)
class RBF:
    """Gaussian kernel exp(-|x - x'|^2 / (2 sigma^2)) (fastfood.py:32-39)."""
    sigma: float

    def __post_init__(self):
        if self.sigma <= 0.0:
            raise ValueError("sigma must be positive")


@dataclass(frozen=True)
class RBFMatern:
    """Matern-type radial kernel of order t (fastfood.py:42-53)."""
    sigma: float
    t: int

    def __post_init__(self):
        if self.sigma <= 0.0:
            raise ValueError("sigma must be positive")
        if self.t < 1:
            raise ValueError("t must be a positive integer")


Kernel = RBF | RBFMatern


def next_pow2(d: int) -> int:
    if d < 1:
        raise ValueError("dimension must be positive")
    return 1 << (d - 1).bit_length()


@dataclass(frozen=True)
class FeatureMapSpec:
    """Complete description of one feature map (fastfood.py:65-79)."""
    input_dim: int
    expansions: int
    kernel: Kernel
    seed: int
    padded_dim: int = field(init=False)

    def __post_init__(self):
        if self.input_dim < 1:
            raise ValueError("input_dim must be positive")
        if self.expansions < 1:
            raise ValueError("expansions must be positive")
        object.__setattr__(self, "padded_dim", next_pow2(self.input_dim))


@dataclass(frozen=True)
class FastfoodBlock:
    """One block's factors (fastfood.py:82-93), as device tensors (views)."""
    b_signs: object      # torch.float32 [n], entries +-1
    permutation: object  # torch.int32 [n], gather out[i] = in[perm[i]]
    g_diag: object       # torch.float32 [n]
    c_diag: object       # torch.float32 [n]
    block_index: int

    @property
    def n(self) -> int:
        return int(self.b_signs.shape[0])

    def numpy(self):
        """Host copy in the reference's dtypes (float32, int64 permutation)."""
        return (self.b_signs.cpu().numpy(), self.permutation.cpu().numpy().astype(np.int64),
                self.g_diag.cpu().numpy(), self.c_diag.cpu().numpy())


class BlockSet(Sequence):
    """All E blocks of a spec, resident in one device buffer.

    Behaves as the reference's ``list[FastfoodBlock]`` (len, indexing,
    iteration); ``tables`` is the opaque buffer the kernels read.
    """

    def __init__(self, spec: FeatureMapSpec, tables, device):
        self.spec = spec
        self.tables = tables
        self.device = device
        n, e = spec.padded_dim, spec.expansions
        torch = nat.require_cuda()
        ptrs = [nat.C.c_void_p() for _ in range(4)]
        nat.call("mck_tables_factors", nat.ptr(tables), n, e, *[nat.C.byref(p) for p in ptrs])
        base = tables.data_ptr()
        views = []
        for p, dt in zip(ptrs, (torch.float32, torch.int32, torch.float32, torch.float32)):
            off = p.value - base
            views.append(tables[off:off + 4 * n * e].view(dt).view(e, n))
        self.b_signs, self.permutation, self.g_diag, self.c_diag = views

    def __len__(self) -> int:
        return self.spec.expansions

    def __getitem__(self, e):
        if isinstance(e, slice):
            return [self[i] for i in range(*e.indices(len(self)))]
        if e < 0:
            e += len(self)
        if not 0 <= e < len(self):
            raise IndexError(e)
        return FastfoodBlock(self.b_signs[e], self.permutation[e], self.g_diag[e],
                             self.c_diag[e], e)


def _tables_alloc(spec: FeatureMapSpec, device):
    torch = nat.require_cuda()
    nbytes = nat.lib().mck_tables_bytes(spec.padded_dim, spec.expansions)
    return torch.empty(nbytes, dtype=torch.uint8, device=device)


def _kernel_args(spec: FeatureMapSpec):
    k = spec.kernel
    if isinstance(k, RBF):
        return nat.MCK_KERNEL_RBF, float(k.sigma), 0
    return nat.MCK_KERNEL_MATERN, float(k.sigma), int(k.t)


@functools.lru_cache(maxsize=16)
def _cached_blocks(spec: FeatureMapSpec, device_index: int) -> BlockSet:
    torch = nat.require_cuda()
    device = torch.device("cuda", device_index)
    with torch.cuda.device(device):
        tables = _tables_alloc(spec, device)
        kind, sigma, t = _kernel_args(spec)
        nat.call("mck_tables_build", nat.ptr(tables), spec.input_dim, spec.expansions, kind,
                 sigma, t, spec.seed & ((1 << 64) - 1), nat.stream_handle(device))
    return BlockSet(spec, tables, device)


def build_blocks(spec: FeatureMapSpec, device=None) -> BlockSet:
    """All blocks of ``spec`` generated on the GPU from the seed (fastfood.py:165-166)."""
    torch = nat.require_cuda()
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    return _cached_blocks(spec, dev.index if dev.index is not None else torch.cuda.current_device())


def build_block(spec: FeatureMapSpec, block_index: int) -> FastfoodBlock:
    """One block (fastfood.py:133-162); realised with its siblings and cached."""
    if not 0 <= block_index < spec.expansions:
        raise ValueError(f"block index {block_index} outside 0..{spec.expansions - 1}")
    return build_blocks(spec)[block_index]


def blocks_from_reference(spec: FeatureMapSpec, blocks, device=None) -> BlockSet:
    """Upload host blocks (e.g. the reference's numpy FastfoodBlocks) as a BlockSet."""
    torch = nat.require_cuda()
    if len(blocks) != spec.expansions:
        raise ValueError(f"expected {spec.expansions} blocks, got {len(blocks)}")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    n = spec.padded_dim
    order = sorted(blocks, key=lambda b: b.block_index)

    def stack(attr, dt):
        arrs = []
        for b in order:
            a = getattr(b, attr)
            a = a.detach().cpu().numpy() if hasattr(a, "detach") else np.asarray(a)
            if a.shape != (n,):
                raise ValueError(f"block factor {attr} must have length {n}")
            arrs.append(a.astype(dt))
        return torch.from_numpy(np.stack(arrs)).to(dev)

    b = stack("b_signs", np.float32)
    p = stack("permutation", np.int32)
    g = stack("g_diag", np.float32)
    c = stack("c_diag", np.float32)
    tables = _tables_alloc(spec, dev)
    with torch.cuda.device(dev):
        nat.call("mck_tables_from_factors", nat.ptr(tables), spec.input_dim, spec.expansions,
                 float(spec.kernel.sigma), nat.ptr(b), nat.ptr(p), nat.ptr(g), nat.ptr(c),
                 nat.stream_handle(dev))
    return BlockSet(spec, tables, dev)


def _as_blockset(spec: FeatureMapSpec, blocks) -> BlockSet:
    if isinstance(blocks, BlockSet):
        if len(blocks) != spec.expansions:
            raise ValueError(f"expected {spec.expansions} blocks, got {len(blocks)}")
        if blocks.spec.padded_dim != spec.padded_dim or blocks.spec.kernel.sigma != spec.kernel.sigma:
            raise ValueError("blocks were built for a different spec")
        return blocks
    if len(blocks) != spec.expansions:
        raise ValueError(f"expected {spec.expansions} blocks, got {len(blocks)}")
    return blocks_from_reference(spec, blocks)


def _ndim(x) -> int:
    return x.ndim if hasattr(x, "ndim") else np.ndim(x)


_VARIANTS = {"fast": nat.MCK_WHT_FAST, "parity": nat.MCK_WHT_PARITY}


def _input(spec: FeatureMapSpec, x, device):
    """x -> (contiguous float32 device tensor (m, d), was_numpy)."""
    torch = nat.require_cuda()
    if isinstance(x, torch.Tensor):
        t = x
        host = not t.is_cuda
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.atleast_2d(np.asarray(x, dtype=np.float32))))
        host = True
    if t.dim() == 1:
        t = t.unsqueeze(0)
    if t.shape[-1] != spec.input_dim:
        raise ValueError(f"input has {t.shape[-1]} features, spec expects {spec.input_dim}")
    t = t.to(device=device, dtype=torch.float32)
    if t.stride(-1) != 1 or (t.data_ptr() % 16):
        t = t.contiguous()
    return t, host


def _row_index(rows, n_rows: int, device):
    """Gather index -> contiguous int32 tensor on `device`, every entry in [0, n_rows)."""
    torch = nat.require_cuda()
    r = rows if isinstance(rows, torch.Tensor) else torch.from_numpy(np.asarray(rows))
    if r.dim() != 1:
        raise ValueError("rows must be a 1-D index array")
    if r.dtype.is_floating_point or r.dtype == torch.bool:
        raise ValueError("rows must hold integer indices")
    if r.numel() and (int(r.min()) < 0 or int(r.max()) >= n_rows):
        raise ValueError(f"rows must lie in [0, {n_rows})")
    return r.to(device=device, dtype=torch.int32).contiguous()


def _check_out(out, m: int, width: int, device):
    torch = nat.require_cuda()
    if not isinstance(out, torch.Tensor) or out.dtype != torch.float32:
        raise ValueError("output buffer must be a float32 tensor")
    if not out.is_cuda or out.device != device:
        raise ValueError(f"output buffer must live on {device}")
    if (out.dim() != 2 or out.shape[0] < m or out.shape[1] < width or out.stride(1) != 1
            or (m > 1 and out.stride(0) < width)):
        raise ValueError("output buffer has the wrong shape")


def _run(spec, blocks, x, features: bool, normalize: bool, variant: str, out=None, rows=None,
         trusted_rows=False):
    torch = nat.require_cuda()
    bs = _as_blockset(spec, blocks)
    xt, host = _input(spec, x, bs.device)
    if rows is not None and not trusted_rows:
        rows = _row_index(rows, xt.shape[0], bs.device)
    m = xt.shape[0] if rows is None else rows.shape[0]
    width = spec.padded_dim * spec.expansions * (2 if features else 1)
    if out is None:
        out = torch.empty((m, width), dtype=torch.float32, device=bs.device)
    else:
        _check_out(out, m, width, bs.device)
    v = _VARIANTS.get(variant)
    if v is None:
        raise ValueError(f"unknown variant {variant!r}")
    # size-1 leading dims may carry any stride; rows are d floats apart then
    ldx = xt.stride(0) if xt.shape[0] > 1 else spec.input_dim
    ldo = out.stride(0) if out.shape[0] > 1 else width
    with torch.cuda.device(bs.device):
        st = nat.stream_handle(bs.device)
        if features:
            nat.call("mck_features_f32", nat.ptr(bs.tables), spec.input_dim, spec.expansions,
                     float(spec.kernel.sigma), nat.ptr(xt), m, ldx, nat.ptr(rows),
                     1 if normalize else 0, nat.ptr(out), ldo, v, st)
        else:
            nat.call("mck_zhat_f32", nat.ptr(bs.tables), spec.input_dim, spec.expansions,
                     float(spec.kernel.sigma), nat.ptr(xt), m, ldx, nat.ptr(rows),
                     nat.ptr(out), ldo, v, st)
    if host:
        return out.cpu().numpy() if not isinstance(x, torch.Tensor) else out.cpu()
    return out


def apply_zhat_batch(spec: FeatureMapSpec, blocks, x, *, variant: str = "fast", out=None):
    """Stacked block outputs z, shape (m, n*E) (fastfood.py:179-198)."""
    return _run(spec, blocks, x, False, False, variant, out)


def apply_zhat(spec: FeatureMapSpec, blocks, x, *, variant: str = "fast"):
    if _ndim(x) != 1:
        raise ValueError("apply_zhat expects a single vector")
    return apply_zhat_batch(spec, blocks, x, variant=variant)[0]


def feature_map_batch(spec: FeatureMapSpec, blocks, x, normalize: bool = True, *,
                      variant: str = "fast", out=None, rows=None):
    """[cos z | sin z] features, shape (m, 2*n*E) (fastfood.py:209-226).

    ``rows`` (integer indices, any dtype/device; range-checked) selects
    x[rows] as the batch (fused gather); ``out`` lets callers stream into a
    preallocated float32 (m, >= 2nE) buffer on the blocks' device.
    """
    return _run(spec, blocks, x, True, normalize, variant, out, rows)


def _feature_rows_device(spec, blocks, x, rows, out, variant="fast"):
    """Raw pairs of x[rows] for in-package callers whose ``rows`` is already a
    valid contiguous int32 index on the device (no host synchronisation)."""
    return _run(spec, blocks, x, True, False, variant, out, rows, trusted_rows=True)


def feature_map(spec: FeatureMapSpec, blocks, x, normalize: bool = True, *, variant: str = "fast"):
    if _ndim(x) != 1:
        raise ValueError("feature_map expects a single vector")
    return feature_map_batch(spec, blocks, x, normalize=normalize, variant=variant)[0]


def feature_dim(spec: FeatureMapSpec) -> int:
    """2 * padded_dim * expansions (fastfood.py:236-238)."""
    return 2 * spec.padded_dim * spec.expansions


def param_count(spec: FeatureMapSpec, num_classes: int) -> int:
    """fastfood.py:241-245."""
    if num_classes < 2:
        raise ValueError("need at least two classes")
    return num_classes * (feature_dim(spec) + 1)


# -- plain-text spec config (checkpoints) -----------------------------------

def spec_to_config(spec: FeatureMapSpec) -> str:
    """key=value text used inside MCKMODL1 checkpoints (fastfood.py:264-274)."""
    lines = [
        f"d={spec.input_dim}",
        f"E={spec.expansions}",
        f"kernel={'rbf' if isinstance(spec.kernel, RBF) else 'matern'}",
        f"sigma={spec.kernel.sigma!r}",
        f"t={spec.kernel.t if isinstance(spec.kernel, RBFMatern) else 0}",
        f"seed={spec.seed}",
    ]
    return "\n".join(lines) + "\n"


def spec_from_config(text: str) -> FeatureMapSpec:
    """Inverse of :func:`spec_to_config` (fastfood.py:277-300)."""
    fields: dict[str, str] = {}
    for line in text.strip().splitlines():
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        key, _, value = line.partition("=")
        fields[key.strip()] = value.strip()
    try:
        d = int(fields["d"])
        expansions = int(fields["E"])
        kind = fields["kernel"]
        sigma = float(fields["sigma"])
        seed = int(fields["seed"])
    except KeyError as exc:
        raise ValueError(f"config is missing key {exc}") from exc
    if kind == "rbf":
        kernel: Kernel = RBF(sigma)
    elif kind == "matern":
        kernel = RBFMatern(sigma, int(fields.get("t", "0")))
    else:
        raise ValueError(f"unknown kernel kind {kind!r}")
    return FeatureMapSpec(input_dim=d, expansions=expansions, kernel=kernel, seed=seed)
