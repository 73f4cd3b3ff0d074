"""Config-4 training step: Fastfood features consumed by the softmax head
without ever being written to HBM (K6, ``mck_fused_forward/backward``).

BASELINE config 4: 2^20 rows of d = 16384, E = 32, sigma = 4, RBF -> 2^20
features per row, 10 classes, global batch 8192 sharded over the ranks of one
node.  Per step each rank expands its 1024-row shard twice (forward, and
again in the backward instead of storing 4 GB of features), the float32
gradient [dW | db] (41.9 MB) is summed by one all-reduce, and every rank
applies the same update.  The arithmetic follows linear_model.py:95-142 of
the reference (softmax, mean cross-entropy, delta = (p - y)/m, W -= lr*dW).
"""

from __future__ import annotations

from . import _native as nat
from . import fastfood
from .distributed import world


class FusedClassifier:
    """Softmax head (W float32 C x 2nE, b float64) over fused Fastfood features."""

    def __init__(self, spec, num_classes: int, max_rows: int, device=None, *,
                 tensor_cores: bool = True):
        torch = nat.require_cuda()
        if num_classes < 2:
            raise ValueError("need at least two classes")
        self.dev = torch.device(device) if device is not None else torch.device("cuda")
        self.spec = spec
        self.blocks = fastfood.build_blocks(spec, self.dev)
        self.C = num_classes
        self.F = fastfood.feature_dim(spec)
        self.max_rows = max_rows
        self.w = torch.zeros((num_classes, self.F), dtype=torch.float32, device=self.dev)
        self.b = torch.zeros(num_classes, dtype=torch.float64, device=self.dev)
        nbytes = nat.lib().mck_fused_scratch_bytes(max_rows, spec.padded_dim, num_classes)
        self.scratch = torch.empty(nbytes, dtype=torch.uint8, device=self.dev)
        self.delta = torch.empty((max_rows, num_classes), dtype=torch.float64, device=self.dev)
        self.loss_sum = torch.zeros(1, dtype=torch.float64, device=self.dev)
        self.hits = torch.zeros(1, dtype=torch.int64, device=self.dev)
        self.rank, self.ws = world()
        self.dw = None
        self.variant = 0 if tensor_cores else 1   # tcgen05 contraction / CUDA-core cross-check

    def _x(self, x):
        torch = nat.require_cuda()
        t = x if isinstance(x, torch.Tensor) else torch.from_numpy(x)
        t = t.to(device=self.dev, dtype=torch.float32)
        if t.dim() != 2 or t.shape[1] != self.spec.input_dim:
            raise ValueError(f"input has {t.shape[-1]} features, spec expects {self.spec.input_dim}")
        return t.contiguous()

    def forward(self, x, labels=None, rows=None, m_total=None, logits=None, probs=None):
        """Logits/probs/loss/hits/delta for x (or x[rows]); delta kept for backward."""
        xt = self._x(x)
        m = int(rows.shape[0]) if rows is not None else int(xt.shape[0])
        if m > self.max_rows:
            raise ValueError(f"batch of {m} rows exceeds max_rows={self.max_rows}")
        s = self.spec
        nat.call("mck_fused_forward", nat.ptr(self.blocks.tables), s.input_dim, s.expansions,
                 float(s.kernel.sigma), nat.ptr(xt), m, xt.stride(0) if m > 1 else s.input_dim,
                 nat.ptr(rows), nat.ptr(self.w), nat.ptr(self.b), self.C, nat.ptr(labels),
                 nat.ptr(rows) if labels is not None and rows is not None else None,
                 m_total or m, nat.ptr(logits), nat.ptr(probs), nat.ptr(self.delta),
                 nat.ptr(self.loss_sum) if labels is not None else None,
                 nat.ptr(self.hits) if labels is not None else None, nat.ptr(self.scratch),
                 self.variant, nat.stream_handle(self.dev))
        return m

    def backward(self, x, m, rows=None, lr=None, l2=0.0):
        """Gradient of the last forward; fused update if lr is given and one rank."""
        torch = nat.require_cuda()
        xt = self._x(x)
        s = self.spec
        st = nat.stream_handle(self.dev)
        args = (nat.ptr(self.blocks.tables), s.input_dim, s.expansions, float(s.kernel.sigma),
                nat.ptr(xt), m, xt.stride(0) if m > 1 else s.input_dim, nat.ptr(rows),
                nat.ptr(self.delta), self.C)
        if lr is not None and self.ws == 1:
            nat.call("mck_fused_backward", *args, None, None, nat.ptr(self.w), nat.ptr(self.b),
                     float(lr), float(l2), nat.ptr(self.scratch), self.variant, st)
            return None
        if self.dw is None:
            # flat [dW (f32, C*F) | db (f32 copy, C) | loss_sum | hits] for one all-reduce
            self.flat = torch.zeros(self.C * self.F + self.C + 2, dtype=torch.float32, device=self.dev)
            self.dw = self.flat[:self.C * self.F].view(self.C, self.F)
            self.db64 = torch.zeros(self.C, dtype=torch.float64, device=self.dev)
        nat.call("mck_fused_backward", *args, nat.ptr(self.dw), nat.ptr(self.db64), None, None,
                 0.0, 0.0, nat.ptr(self.scratch), self.variant, st)
        return self.dw

    def step(self, x, labels, rows=None, m_total=None, lr=0.01, l2=0.0):
        """One SGD step on this rank's shard; returns the device loss-sum tensor."""
        m = self.forward(x, labels, rows=rows, m_total=m_total)
        if self.ws == 1:
            self.backward(x, m, rows=rows, lr=lr, l2=l2)
            return self.loss_sum
        import torch.distributed as dist
        self.backward(x, m, rows=rows)
        cf = self.C * self.F
        self.flat[cf:cf + self.C].copy_(self.db64)
        self.flat[-2:-1].copy_(self.loss_sum)
        dist.all_reduce(self.flat, op=dist.ReduceOp.SUM)
        if l2:
            self.dw.add_(self.w, alpha=2.0 * l2)
        self.w.add_(self.dw, alpha=-lr)
        self.b.sub_(lr * self.flat[cf:cf + self.C].double())
        self.loss_sum.copy_(self.flat[-2:-1])
        return self.loss_sum
