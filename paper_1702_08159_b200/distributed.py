"""Data-parallel plumbing for mini-batch SGD over 1..8 GPUs of one node.

The reference trains on one process (linear_model.py:191-223; distributed
training is a non-goal).  Here every global mini-batch -- taken
in the reference's shuffle order -- is split into contiguous row shards, one
per rank.  Each rank expands its shard, forms delta = (p - y) / m_global and
its partial [dW | db | loss_sum | hits]; one float64 all-reduce (NCCL over
NVLink on GPUs, gloo in the CPU tests) sums the partials, and every rank
applies the identical SGD update.  Factor tables are regenerated per rank
from the seed, so they never cross the wire.
"""

from __future__ import annotations

from dataclasses import dataclass


def world():
    """(rank, world_size) of the default process group, or (0, 1)."""
    try:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            return dist.get_rank(), dist.get_world_size()
    except ImportError:
        pass
    return 0, 1


def shard_range(m: int, rank: int, world_size: int) -> tuple[int, int]:
    """Contiguous shard [lo, hi) of m rows for `rank`; sizes differ by at most 1."""
    if world_size < 1 or not 0 <= rank < world_size:
        raise ValueError("bad rank/world size")
    base, extra = divmod(m, world_size)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


@dataclass
class GradBucket:
    """Flat float64 buffer [dW (C*F) | db (C) | loss_sum | hits] reduced in one call."""
    flat: object          # torch.float64 tensor
    num_classes: int
    num_features: int

    @classmethod
    def empty(cls, num_classes: int, num_features: int, device):
        import torch
        flat = torch.zeros(num_classes * num_features + num_classes + 2, dtype=torch.float64,
                           device=device)
        return cls(flat, num_classes, num_features)

    @property
    def dw(self):
        c, f = self.num_classes, self.num_features
        return self.flat[:c * f].view(c, f)

    @property
    def db(self):
        c, f = self.num_classes, self.num_features
        return self.flat[c * f:c * f + c]

    @property
    def loss_sum(self):
        return self.flat[-2:-1]

    @property
    def hits(self):
        return self.flat[-1:]

    def allreduce(self, group=None, async_op: bool = False):
        """Sum the bucket over ranks.  With ``async_op`` the collective is
        enqueued behind the work already on the current stream and a handle
        is returned; ``handle.wait()`` orders later work after it."""
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
            return dist.all_reduce(self.flat, op=dist.ReduceOp.SUM, group=group, async_op=async_op)
        return _Done() if async_op else None


class _Done:
    def wait(self):
        return True
