"""Host-to-host streaming of the feature map (the drop-in call with host buffers).

``feature_map_to_host`` is what a caller of the reference's
``feature_map_batch(spec, blocks, x)`` gets when x and the result live in host
memory: batches of rows are copied in, expanded by ``mck_features_f32`` and
copied out, with copy-in, compute and copy-out of consecutive batches
overlapped on three CUDA streams.  Host buffers should be pinned
(``torch.empty(..., pin_memory=True)``) for full PCIe bandwidth.
"""

from __future__ import annotations

from . import _native as nat
from . import fastfood


class HostStreamer:
    """Reusable device staging for ``feature_map_to_host``."""

    def __init__(self, spec, blocks, batch_rows: int = 4096, normalize: bool = True,
                 device=None):
        torch = nat.require_cuda()
        self.spec = spec
        self.blocks = fastfood._as_blockset(spec, blocks)
        self.dev = self.blocks.device if device is None else torch.device(device)
        self.batch = batch_rows
        self.normalize = normalize
        width = fastfood.feature_dim(spec)
        self.xin = [torch.empty((batch_rows, spec.input_dim), dtype=torch.float32, device=self.dev)
                    for _ in range(2)]
        self.out = [torch.empty((batch_rows, width), dtype=torch.float32, device=self.dev)
                    for _ in range(2)]
        self.s_in = torch.cuda.Stream(self.dev)
        self.s_cmp = torch.cuda.Stream(self.dev)
        self.s_out = torch.cuda.Stream(self.dev)
        self.launches = 0

    def run(self, x_host, out_host):
        """Expand all rows of pinned host ``x_host`` into pinned host ``out_host``."""
        torch = nat.require_cuda()
        m = x_host.shape[0]
        ev_in = [torch.cuda.Event() for _ in range(2)]
        ev_cmp = [torch.cuda.Event() for _ in range(2)]
        ev_out = [None, None]
        for k, r0 in enumerate(range(0, m, self.batch)):
            b = k & 1
            r1 = min(m, r0 + self.batch)
            with torch.cuda.stream(self.s_in):
                if k >= 2:
                    self.s_in.wait_event(ev_cmp[b])      # xin[b] free again
                self.xin[b][:r1 - r0].copy_(x_host[r0:r1], non_blocking=True)
                ev_in[b].record(self.s_in)
            with torch.cuda.stream(self.s_cmp):
                self.s_cmp.wait_event(ev_in[b])
                if ev_out[b] is not None:
                    self.s_cmp.wait_event(ev_out[b])     # out[b] drained
                fastfood.feature_map_batch(self.spec, self.blocks, self.xin[b][:r1 - r0],
                                           normalize=self.normalize, out=self.out[b])
                self.launches += 1
                ev_cmp[b].record(self.s_cmp)
            with torch.cuda.stream(self.s_out):
                self.s_out.wait_event(ev_cmp[b])
                out_host[r0:r1].copy_(self.out[b][:r1 - r0], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(self.s_out)
                ev_out[b] = ev
        self.s_out.synchronize()
        return out_host


def feature_map_to_host(spec, blocks, x_host, out_host=None, *, batch_rows: int = 4096,
                        normalize: bool = True):
    """[cos z | sin z] of host rows into a host array, pipelined over the PCIe link."""
    torch = nat.require_cuda()
    if out_host is None:
        out_host = torch.empty((x_host.shape[0], fastfood.feature_dim(spec)), dtype=torch.float32,
                               pin_memory=True)
    return HostStreamer(spec, blocks, batch_rows, normalize).run(x_host, out_host)
