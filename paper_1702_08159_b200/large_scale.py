"""Config-4 training step: Fastfood features consumed by the softmax head
without ever being written to HBM (K6, ``mck_fused_forward/backward``).

BASELINE config 4: 2^20 rows of d = 16384, E = 32, sigma = 4, RBF -> 2^20
features per row, 10 classes, global batch 8192 sharded over the ranks of one
node.  Per step each rank expands its 1024-row shard twice (forward, and
again in the backward instead of storing 4 GB of features).  The arithmetic
follows linear_model.py:95-142 of the reference (softmax, mean cross-entropy,
delta = (p - y)/m_global, W -= lr*(dW + 2*l2*W), b -= lr*db).

Multi-rank: the gradient is all-reduced in buckets of
16 blocks (one z group of the backward: 21 MB of float32 dW at config 4),
each bucket's all-reduce issued as soon as its backward is enqueued, so it
runs on the communicator's stream while the next group's backward computes;
a small float64 bucket [db | loss_sum | hits] goes first.  Every rank then
applies the identical update (``mck_fused_apply_bucket``).
"""

from __future__ import annotations

import numpy as np

from . import _native as nat
from . import fastfood
from .distributed import world
from .linear_model import FUSED_MAX_CLASSES, _check_classes

BUCKET_BLOCKS = 16  # blocks per all-reduce bucket = the backward's z group (csrc/fused_head.cu)
# Contraction engines: packed-FFMA2 CUDA-core kernels (default: with 10
# classes the contraction is MUFU- and HBM-bound, csrc/fused_cc.cu), tcgen05
# tensor cores (kind::tf32, 3xTF32 split, csrc/fused_tc.cu) and a simple
# CUDA-core cross-check.
ENGINES = {"ffma2": 0, "tcgen05": 4, "reference": 1}


class FusedClassifier:
    """Softmax head (W float32 C x 2nE, b float64) over fused Fastfood features."""

    def __init__(self, spec, num_classes: int, max_rows: int, device=None, *,
                 engine: str = "ffma2", bucket_blocks: int = BUCKET_BLOCKS,
                 keep_z: bool = True):
        torch = nat.require_cuda()
        _check_classes(num_classes, FUSED_MAX_CLASSES)
        self.dev = torch.device(device) if device is not None else torch.device("cuda")
        if self.dev.index is None:
            self.dev = torch.device("cuda", torch.cuda.current_device())
        self.spec = spec
        self.blocks = fastfood.build_blocks(spec, self.dev)
        self.C = num_classes
        self.F = fastfood.feature_dim(spec)
        self.max_rows = max_rows
        self.w = torch.zeros((num_classes, self.F), dtype=torch.float32, device=self.dev)
        self.b = torch.zeros(num_classes, dtype=torch.float64, device=self.dev)
        # keep_z: the forward's z of all blocks (m x nE fp32; 2 GiB at 1,024 c4 rows) stays
        # in scratch for the backward, which then skips the second expansion
        nbytes = nat.lib().mck_fused_scratch_bytes_ex(max_rows, spec.padded_dim, spec.expansions,
                                                      num_classes, 1 if keep_z else 0)
        self.scratch = torch.empty(nbytes, dtype=torch.uint8, device=self.dev)
        self.delta = torch.empty((max_rows, num_classes), dtype=torch.float64, device=self.dev)
        self.loss_sum = torch.zeros(1, dtype=torch.float64, device=self.dev)
        self.hits = torch.zeros(1, dtype=torch.int64, device=self.dev)
        self.rank, self.ws = world()
        # contraction engine (bits 0/2) and keep-z (bit 1) of mck_fused_forward/backward
        if engine not in ENGINES:
            raise ValueError(f"engine must be one of {sorted(ENGINES)}")
        self.engine = engine
        self.variant = ENGINES[engine] | (2 if keep_z else 0)
        self.bucket_blocks = max(1, int(bucket_blocks))
        self._buckets = None
        self._checked = set()   # validated index tensors (see _index)

    # -- inputs ------------------------------------------------------------
    def _x(self, x):
        torch = nat.require_cuda()
        t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.asarray(x))
        t = t.to(device=self.dev, dtype=torch.float32)
        if t.dim() != 2 or t.shape[1] != self.spec.input_dim:
            raise ValueError(f"input has {t.shape[-1]} features, spec expects {self.spec.input_dim}")
        return t.contiguous()

    def _index(self, v, bound: int, what: str):
        """Integer vector -> contiguous int32 on the device, entries in [0, bound).

        The range check reads the tensor back (a host synchronisation); an
        int32 device tensor that already passed is remembered by (address,
        version, length), so a label vector reused every step is checked once."""
        torch = nat.require_cuda()
        if v is None:
            return None
        if (isinstance(v, torch.Tensor) and v.dtype == torch.int32 and v.device == self.dev
                and v.is_contiguous()):
            key = (v.data_ptr(), v._version, v.numel(), bound)
            if key in self._checked:
                return v
        t = v if isinstance(v, torch.Tensor) else torch.from_numpy(np.asarray(v))
        if t.dim() != 1 or t.dtype.is_floating_point or t.dtype == torch.bool:
            raise ValueError(f"{what} must be a 1-D integer array")
        if t.numel() and (int(t.min()) < 0 or int(t.max()) >= bound):
            raise ValueError(f"{what} must lie in [0, {bound})")
        t = t.to(device=self.dev, dtype=torch.int32).contiguous()
        if len(self._checked) > 64:
            self._checked.clear()
        self._checked.add((t.data_ptr(), t._version, t.numel(), bound))
        return t

    def _ld(self, xt, m):
        return xt.stride(0) if xt.shape[0] > 1 else self.spec.input_dim

    # -- forward / backward ------------------------------------------------
    def forward(self, x, labels=None, rows=None, m_total=None, logits=None, probs=None):
        """Logits/probs/loss/hits/delta for x (or x[rows]); delta kept for backward.

        ``labels`` are indexed like x (label of batch row r is labels[rows[r]]
        when ``rows`` is given, else labels[r])."""
        torch = nat.require_cuda()
        xt = self._x(x)
        rows = self._index(rows, xt.shape[0], "rows")
        labels = self._index(labels, self.C, "labels")
        m = int(rows.shape[0]) if rows is not None else int(xt.shape[0])
        if m > self.max_rows:
            raise ValueError(f"batch of {m} rows exceeds max_rows={self.max_rows}")
        if labels is not None and labels.shape[0] < (xt.shape[0] if rows is not None else m):
            raise ValueError("labels are shorter than the batch")
        for buf, shape in ((logits, (m, self.C)), (probs, (m, self.C))):
            if buf is not None and (buf.dtype != torch.float64 or buf.device != self.dev
                                    or not buf.is_contiguous() or buf.numel() < m * self.C):
                raise ValueError(f"output buffer must be a contiguous float64 {shape} tensor on {self.dev}")
        s = self.spec
        self._last = (xt, rows, m)
        if m == 0 and labels is not None:  # an empty shard contributes no loss / hits
            self.loss_sum.zero_()
            self.hits.zero_()
        with torch.cuda.device(self.dev):
            nat.call("mck_fused_forward", nat.ptr(self.blocks.tables), s.input_dim, s.expansions,
                     float(s.kernel.sigma), nat.ptr(xt), m, self._ld(xt, m), nat.ptr(rows),
                     nat.ptr(self.w), nat.ptr(self.b), self.C, nat.ptr(labels),
                     nat.ptr(rows) if labels is not None and rows is not None else None,
                     m_total or m, nat.ptr(logits), nat.ptr(probs), nat.ptr(self.delta),
                     nat.ptr(self.loss_sum) if labels is not None else None,
                     nat.ptr(self.hits) if labels is not None else None, nat.ptr(self.scratch),
                     self.variant, nat.stream_handle(self.dev))
        return m

    def _bwd_args(self):
        xt, rows, m = self._last
        s = self.spec
        return (nat.ptr(self.blocks.tables), s.input_dim, s.expansions, float(s.kernel.sigma),
                nat.ptr(xt), m, self._ld(xt, m), nat.ptr(rows), nat.ptr(self.delta), self.C)

    def backward(self, lr=None, l2=0.0):
        """Gradient of the last forward.  With ``lr`` (one rank) the SGD
        update is fused into the contraction; otherwise returns (dW f32, db f64)."""
        torch = nat.require_cuda()
        st = nat.stream_handle(self.dev)
        with torch.cuda.device(self.dev):
            if lr is not None:
                nat.call("mck_fused_backward", *self._bwd_args(), None, None, nat.ptr(self.w),
                         nat.ptr(self.b), float(lr), float(l2), nat.ptr(self.scratch),
                         self.variant, st)
                return None
            dw = torch.empty_like(self.w)
            db = torch.empty_like(self.b)
            nat.call("mck_fused_backward", *self._bwd_args(), nat.ptr(dw), nat.ptr(db), None, None,
                     0.0, 0.0, nat.ptr(self.scratch), self.variant, st)
            return dw, db

    # -- multi-rank ----------------------------------------------------------
    def bucket_ranges(self):
        E, k = self.spec.expansions, self.bucket_blocks
        return [(e, min(k, E - e)) for e in range(0, E, k)]

    def _alloc_buckets(self):
        torch = nat.require_cuda()
        n = self.spec.padded_dim
        self._buckets = [torch.empty((self.C, 2 * cnt * n), dtype=torch.float32, device=self.dev)
                         for _, cnt in self.bucket_ranges()]
        self._tail = torch.zeros(self.C + 2, dtype=torch.float64, device=self.dev)  # [db | loss | hits]

    def _step_allreduce(self, lr, l2, m_total):
        import torch.distributed as dist
        torch = nat.require_cuda()
        if self._buckets is None:
            self._alloc_buckets()
        st = nat.stream_handle(self.dev)
        xt, rows, m = self._last
        tail = self._tail
        nat.call("mck_fused_bias_grad", nat.ptr(self.delta), m, self.C, nat.ptr(tail), st)
        tail[self.C:self.C + 1].copy_(self.loss_sum)
        tail[self.C + 1:].copy_(self.hits)
        works = [dist.all_reduce(tail, op=dist.ReduceOp.SUM, async_op=True)]
        for (e0, cnt), buf in zip(self.bucket_ranges(), self._buckets):
            nat.call("mck_fused_backward_bucket", *self._bwd_args(), e0, cnt, nat.ptr(buf),
                     nat.ptr(self.scratch), self.variant, st)
            # issued now: the collective waits for this bucket only and overlaps
            # the next bucket's backward on the compute stream
            works.append(dist.all_reduce(buf, op=dist.ReduceOp.SUM, async_op=True))
        for wk in works:
            wk.wait()
        st = nat.stream_handle(self.dev)
        for k, ((e0, cnt), buf) in enumerate(zip(self.bucket_ranges(), self._buckets)):
            last = k == len(self._buckets) - 1
            nat.call("mck_fused_apply_bucket", nat.ptr(self.w), self.spec.input_dim,
                     self.spec.expansions, self.C, e0, cnt, nat.ptr(buf), float(lr), float(l2),
                     nat.ptr(self.b) if last else None, nat.ptr(tail) if last else None, st)
        self.loss_sum.copy_(tail[self.C:self.C + 1])
        self.hits.copy_(tail[self.C + 1:].to(torch.int64))

    def step(self, x, labels, rows=None, m_total=None, lr=0.01, l2=0.0):
        """One SGD step on this rank's shard of a global batch of ``m_total``
        rows; returns the device loss-sum tensor (summed over ranks)."""
        torch = nat.require_cuda()
        self.forward(x, labels, rows=rows, m_total=m_total)
        with torch.cuda.device(self.dev):
            if self.ws == 1:
                self.backward(lr=lr, l2=l2)
            else:
                self._step_allreduce(lr, l2, m_total)
        return self.loss_sum
