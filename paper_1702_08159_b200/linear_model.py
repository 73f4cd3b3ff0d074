"""Softmax head and mini-batch SGD on B200 -- drop-in for ``mckernel.linear_model``.

Same objects and semantics as the reference (``pkg/src/mckernel/linear_model.py``):
float64 W and b starting at zero, stable softmax, mean cross-entropy plus
l2*|W|^2, analytic gradients, W -= lr*dW, epoch shuffles from the stream
("shuffle", epoch) keyed by ``shuffle_seed``, batches in shuffle order (last
one partial), per-epoch mean train loss and test accuracy.

Differences are in where the work runs: one training step is
  mck_features_f32 (fused gather of the batch rows + expansion, raw pairs)
  -> mck_head_forward (logits, softmax, loss, delta in one pass)
  -> mck_head_backward_sgd (dW = delta^T phi fused with the update)
on the current CUDA stream, with no host synchronisation inside an epoch.
The reference evaluates the forward twice per step (loss, then gradients,
linear_model.py:218-219); both see the same W, so one pass suffices.
With torch.distributed initialised, batches are sharded over ranks and the
gradient is summed by one all-reduce (see distributed.py).
"""

from __future__ import annotations

import io
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from . import fastfood
from .detrand import fisher_yates_permutations
from .distributed import GradBucket, shard_range, world


@dataclass
class TrainConfig:
    learning_rate: float
    batch_size: int
    epochs: int
    l2_lambda: float = 0.0
    shuffle_seed: int = 0

    def __post_init__(self):
        if self.learning_rate <= 0.0:
            raise ValueError("learning rate must be positive")
        if self.batch_size < 1:
            raise ValueError("batch size must be positive")
        if self.epochs < 0:
            raise ValueError("epochs must be non-negative")
        if self.l2_lambda < 0.0:
            raise ValueError("l2_lambda must be non-negative")


@dataclass
class Dataset:
    """Dense samples + integer labels (mirror of mckernel.dataio.Dataset)."""
    features: object
    labels: object
    num_classes: int

    @property
    def dim(self) -> int:
        return int(self.features.shape[1])

    def __len__(self) -> int:
        return int(self.labels.shape[0])


class SoftmaxModel:
    """W (C x F) and b (C), float64, resident on the GPU (linear_model.py:53-76)."""

    def __init__(self, w, b, device=None):
        torch = nat.require_cuda()
        dev = torch.device(device) if device is not None else torch.device("cuda")
        w = torch.as_tensor(np.asarray(w) if not isinstance(w, torch.Tensor) else w)
        b = torch.as_tensor(np.asarray(b) if not isinstance(b, torch.Tensor) else b)
        if w.dim() != 2 or tuple(b.shape) != (w.shape[0],):
            raise ValueError("W must be (C, F) and b length C")
        _check_classes(int(w.shape[0]))
        self.w = w.to(device=dev, dtype=torch.float64).contiguous()
        self.b = b.to(device=dev, dtype=torch.float64).contiguous()

    @classmethod
    def zeros(cls, num_classes: int, num_features: int, device=None) -> "SoftmaxModel":
        _check_classes(num_classes)
        return cls(np.zeros((num_classes, num_features)), np.zeros(num_classes), device)

    @property
    def num_classes(self) -> int:
        return int(self.w.shape[0])

    @property
    def num_features(self) -> int:
        return int(self.w.shape[1])

    def numpy(self):
        return self.w.cpu().numpy(), self.b.cpu().numpy()


@dataclass
class EpochRecord:
    epoch: int
    train_loss: float
    test_acc: float


@dataclass
class RunMetrics:
    records: list[EpochRecord] = field(default_factory=list)

    def to_csv(self) -> str:
        buf = io.StringIO()
        buf.write("epoch,train_loss,test_acc\n")
        for r in self.records:
            buf.write(f"{r.epoch},{r.train_loss!r},{r.test_acc!r}\n")
        return buf.getvalue()

    def save_csv(self, path) -> None:
        with open(path, "w", encoding="utf-8") as f:
            f.write(self.to_csv())


# The softmax head takes any number of classes (groups of 16 classes per
# kernel launch above 16, csrc/classifier.cu); the fused config-4 classifier
# (large_scale.py) takes at most FUSED_MAX_CLASSES.
FUSED_MAX_CLASSES = 16


def _check_classes(num_classes: int, limit: int | None = None) -> None:
    if num_classes < 2:
        raise ValueError("need at least two classes")
    if limit is not None and num_classes > limit:
        raise ValueError(f"num_classes must be in 2..{limit} (fused config-4 kernels); "
                         f"got {num_classes}")


def _check_labels(labels, num_classes: int) -> None:
    if len(labels) and (int(labels.min()) < 0 or int(labels.max()) >= num_classes):
        raise ValueError(f"labels must lie in [0, {num_classes})")


def _feat_tensor(x, device):
    torch = nat.require_cuda()
    t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x))
    return t.to(device=device, dtype=torch.float32).contiguous()


def _labels_tensor(y, device):
    torch = nat.require_cuda()
    t = y if isinstance(y, torch.Tensor) else torch.from_numpy(np.asarray(y))
    return t.to(device=device, dtype=torch.int32).contiguous()


class _Head:
    """Device buffers for the head kernels at a maximum batch size."""

    def __init__(self, m_max: int, num_features: int, num_classes: int, device):
        torch = nat.require_cuda()
        self.m_max, self.F, self.C = m_max, num_features, num_classes
        nbytes = nat.lib().mck_head_scratch_bytes(m_max, num_features, num_classes)
        self.scratch = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
        self.delta = torch.empty((m_max, num_classes), dtype=torch.float64, device=device)
        self.device = device

    def forward(self, phi, m, model, labels=None, label_index=None, m_total=None, probs=None,
                delta=True, loss_sum=None, hits=None):
        nat.call("mck_head_forward", nat.ptr(phi), m, self.F, phi.stride(0), nat.ptr(model.w),
                 nat.ptr(model.b), self.C, nat.ptr(labels), nat.ptr(label_index),
                 m_total or m, nat.ptr(probs), nat.ptr(self.delta) if delta else None,
                 loss_sum, hits, nat.ptr(self.scratch), nat.stream_handle(self.device))


def forward_batch(model: SoftmaxModel, x):
    """Class probabilities (float64) for a batch of features (linear_model.py:95-97)."""
    torch = nat.require_cuda()
    phi = _feat_tensor(x, model.w.device)
    if phi.shape[1] != model.num_features:
        raise ValueError(f"feature length {phi.shape[1]} does not match model F={model.num_features}")
    m = phi.shape[0]
    probs = torch.empty((m, model.num_classes), dtype=torch.float64, device=model.w.device)
    _Head(m, model.num_features, model.num_classes, model.w.device).forward(
        phi, m, model, probs=probs, delta=False)
    return probs


def forward(model: SoftmaxModel, x):
    if x.ndim != 1:
        raise ValueError("forward expects a single feature vector")
    return forward_batch(model, x[None, :])[0]


def loss(model: SoftmaxModel, x, labels, l2_lambda: float = 0.0) -> float:
    """Mean cross-entropy plus l2*|W|_F^2 (linear_model.py:105-115)."""
    torch = nat.require_cuda()
    _check_labels(np.asarray(labels) if not isinstance(labels, torch.Tensor) else labels,
                  model.num_classes)
    phi = _feat_tensor(x, model.w.device)
    m = phi.shape[0]
    y = _labels_tensor(labels, model.w.device)
    acc = torch.zeros(1, dtype=torch.float64, device=model.w.device)
    _Head(m, model.num_features, model.num_classes, model.w.device).forward(
        phi, m, model, labels=y, delta=False, loss_sum=acc.data_ptr())
    ce = float(acc.item()) / m
    if l2_lambda:
        ce += l2_lambda * float((model.w * model.w).sum().item())
    return ce


def gradients(model: SoftmaxModel, x, labels, l2_lambda: float = 0.0):
    """(dW, db) of the regularised batch objective (linear_model.py:118-131)."""
    torch = nat.require_cuda()
    _check_labels(np.asarray(labels) if not isinstance(labels, torch.Tensor) else labels,
                  model.num_classes)
    phi = _feat_tensor(x, model.w.device)
    m = phi.shape[0]
    y = _labels_tensor(labels, model.w.device)
    head = _Head(m, model.num_features, model.num_classes, model.w.device)
    head.forward(phi, m, model, labels=y)
    dw = torch.empty_like(model.w)
    db = torch.empty_like(model.b)
    nat.call("mck_head_backward", nat.ptr(phi), m, model.num_features, phi.stride(0),
             nat.ptr(head.delta), model.num_classes, nat.ptr(dw), nat.ptr(db),
             nat.ptr(head.scratch), nat.stream_handle(model.w.device))
    if l2_lambda:
        dw += 2.0 * l2_lambda * model.w
    return dw, db


def sgd_step(model: SoftmaxModel, x, labels, config: TrainConfig) -> SoftmaxModel:
    """W <- W - lr dW, b <- b - lr db (linear_model.py:134-142)."""
    if len(labels) == 0:
        raise ValueError("batch must be non-empty")
    dw, db = gradients(model, x, labels, config.l2_lambda)
    model.w -= config.learning_rate * dw
    model.b -= config.learning_rate * db
    return model


class Trainer:
    """Device-resident training state for one (spec, dataset, config)."""

    def __init__(self, spec, train_ds, test_ds, config: TrainConfig, *, variant="fast",
                 eval_chunk: int = 4096):
        torch = nat.require_cuda()
        if spec is not None and spec.input_dim != train_ds.dim:
            raise ValueError(f"spec input_dim {spec.input_dim} != dataset dim {train_ds.dim}")
        if train_ds.dim != test_ds.dim:
            raise ValueError("train and test dimensions differ")
        _check_classes(int(train_ds.num_classes))
        self.rank, self.ws = world()
        self.dev = torch.device("cuda", torch.cuda.current_device())
        self.spec, self.config, self.variant = spec, config, variant
        self.C = int(train_ds.num_classes)
        self.X = _feat_tensor(train_ds.features, self.dev)
        self.y = _labels_tensor(train_ds.labels, self.dev)
        self.Xt = _feat_tensor(test_ds.features, self.dev)
        self.yt = _labels_tensor(test_ds.labels, self.dev)
        _check_labels(self.y, self.C)
        _check_labels(self.yt, self.C)
        self.n = int(self.y.shape[0])
        self.blocks = fastfood.build_blocks(spec, self.dev) if spec is not None else None
        self.F = fastfood.feature_dim(spec) if spec is not None else train_ds.dim
        self.model = SoftmaxModel.zeros(self.C, self.F, self.dev)
        self.local_max = shard_range(config.batch_size, 0, self.ws)[1]
        self.eval_chunk = eval_chunk
        m_buf = max(self.local_max, min(eval_chunk, max(len(self.yt), 1)))
        self.phi = torch.empty((m_buf, self.F), dtype=torch.float32, device=self.dev)
        self.head = _Head(m_buf, self.F, self.C, self.dev)
        self.steps = (self.n + config.batch_size - 1) // config.batch_size
        self.step_loss = torch.zeros(max(self.steps, 1), dtype=torch.float64, device=self.dev)
        self.bucket = GradBucket.empty(self.C, self.F, self.dev) if self.ws > 1 else None
        self.orders = (fisher_yates_permutations(config.shuffle_seed, "shuffle", 0, config.epochs,
                                                 self.n, self.dev)
                       if config.epochs > 0 else None)

    def featurize(self, x, rows, m):
        """Raw cos/sin pairs of x[rows] (or the first m rows of x) into self.phi."""
        if self.spec is None:
            sel = x.index_select(0, rows.long()) if rows is not None else x[:m]
            self.phi[:m].copy_(sel)
            return self.phi
        if rows is None:
            fastfood.feature_map_batch(self.spec, self.blocks, x, normalize=False,
                                       variant=self.variant, out=self.phi)
        else:  # slices of the device epoch shuffles: int32, in range by construction
            fastfood._feature_rows_device(self.spec, self.blocks, x, rows, self.phi, self.variant)
        return self.phi

    def _rows(self, epoch: int, s: int):
        cfg = self.config
        start = s * cfg.batch_size
        mg = min(cfg.batch_size, self.n - start)
        lo, hi = shard_range(mg, self.rank, self.ws)
        return self.orders[epoch, start + lo:start + hi], hi - lo, mg

    def _expand(self, epoch: int, s: int) -> None:
        """Features of this rank's shard of batch s (fused row gather) into phi."""
        rows, ml, _ = self._rows(epoch, s)
        if ml > 0:
            self.featurize(self.X, rows, ml)

    def _grad(self, epoch: int, s: int):
        """Forward + gradient of batch s from phi.  One rank: the SGD update is
        fused into the backward and None is returned.  Several ranks: the
        partial [dW | db | loss] is written to the bucket and its all-reduce
        is issued asynchronously; the work handle is returned."""
        cfg = self.config
        rows, ml, mg = self._rows(epoch, s)
        st = nat.stream_handle(self.dev)
        loss_ptr = self.step_loss.data_ptr() + 8 * s
        phi = self.phi
        if ml > 0:
            self.head.forward(phi, ml, self.model, labels=self.y, label_index=rows, m_total=mg,
                              loss_sum=loss_ptr if self.ws == 1 else self.bucket.loss_sum.data_ptr())
        if self.ws == 1:
            if cfg.l2_lambda:
                self.step_loss[s] += mg * cfg.l2_lambda * (self.model.w * self.model.w).sum()
            nat.call("mck_head_backward_sgd", nat.ptr(phi), ml, self.F, phi.stride(0),
                     nat.ptr(self.head.delta), self.C, nat.ptr(self.model.w),
                     nat.ptr(self.model.b), float(cfg.learning_rate), float(cfg.l2_lambda),
                     nat.ptr(self.head.scratch), st)
            return None
        b = self.bucket
        if ml > 0:
            nat.call("mck_head_backward", nat.ptr(phi), ml, self.F, phi.stride(0),
                     nat.ptr(self.head.delta), self.C, nat.ptr(b.dw), nat.ptr(b.db),
                     nat.ptr(self.head.scratch), st)
        else:
            b.flat.zero_()
        return b.allreduce(async_op=True)

    def _update(self, s: int, work) -> None:
        """Wait for batch s's all-reduce and apply the identical update on every rank."""
        if self.ws == 1:
            return
        cfg = self.config
        _, _, mg = self._rows(0, s)
        b = self.bucket
        work.wait()
        if cfg.l2_lambda:
            b.loss_sum.add_(mg * cfg.l2_lambda * (self.model.w * self.model.w).sum())
        self.step_loss[s:s + 1].copy_(b.loss_sum)
        nat.call("mck_head_sgd_update", nat.ptr(self.model.w), nat.ptr(self.model.b),
                 nat.ptr(b.dw), nat.ptr(b.db), self.F, self.C, float(cfg.learning_rate),
                 float(cfg.l2_lambda), nat.stream_handle(self.dev))

    def step(self, epoch: int, s: int) -> None:
        """One SGD step on global batch s of `epoch` (linear_model.py:213-220)."""
        self._expand(epoch, s)
        self._update(s, self._grad(epoch, s))

    def run_epoch(self, epoch: int) -> None:
        """All steps of an epoch.  With several ranks the expansion of batch
        s+1 is enqueued while batch s's gradient all-reduce is in flight (it
        does not depend on W), so the collective overlaps the expansion."""
        if self.ws == 1:
            for s in range(self.steps):
                self.step(epoch, s)
            return
        if self.steps:
            self._expand(epoch, 0)
        for s in range(self.steps):
            work = self._grad(epoch, s)
            if s + 1 < self.steps:
                self._expand(epoch, s + 1)
            self._update(s, work)

    def batch_sizes(self):
        cfg = self.config
        return [min(cfg.batch_size, self.n - s * cfg.batch_size) for s in range(self.steps)]

    def epoch_loss(self) -> float:
        """Mean over steps of each step's mean loss (linear_model.py:218,222)."""
        sums = self.step_loss[:self.steps].cpu().numpy()
        sizes = np.asarray(self.batch_sizes(), dtype=np.float64)
        return float((sums / sizes).sum() / self.steps)

    def evaluate(self):
        """(accuracy, mean loss) on the test set (linear_model.py:226-239)."""
        torch = nat.require_cuda()
        nt = int(self.yt.shape[0])
        lo, hi = shard_range(nt, self.rank, self.ws)
        chunks = list(range(lo, hi, self.eval_chunk))
        acc = torch.zeros(max(len(chunks), 1), dtype=torch.float64, device=self.dev)
        hits = torch.zeros(max(len(chunks), 1), dtype=torch.int64, device=self.dev)
        for k, s0 in enumerate(chunks):
            m = min(self.eval_chunk, hi - s0)
            xs = self.Xt[s0:s0 + m]
            phi = self.featurize(xs, None, m)
            self.head.forward(phi, m, self.model, labels=self.yt[s0:s0 + m], delta=False,
                              loss_sum=acc.data_ptr() + 8 * k, hits=hits.data_ptr() + 8 * k)
        tot = torch.stack([acc.sum(), hits.sum().to(torch.float64)])
        if self.ws > 1:
            import torch.distributed as dist
            dist.all_reduce(tot)
        tot = tot.cpu().numpy()
        return float(tot[1]) / nt, float(tot[0]) / nt


def train(spec, train_ds, test_ds, config: TrainConfig, *, variant: str = "fast",
          eval_chunk: int = 4096):
    """Mini-batch SGD over shuffled epochs; returns (model, metrics) (linear_model.py:191-223)."""
    tr = Trainer(spec, train_ds, test_ds, config, variant=variant, eval_chunk=eval_chunk)
    metrics = RunMetrics()
    for epoch in range(config.epochs):
        tr.run_epoch(epoch)
        acc, _ = tr.evaluate()
        metrics.records.append(EpochRecord(epoch, tr.epoch_loss(), acc))
    return tr.model, metrics


def evaluate(model: SoftmaxModel, spec, ds, *, chunk: int = 4096):
    """Argmax accuracy and mean unregularised loss (linear_model.py:242-245)."""
    torch = nat.require_cuda()
    dev = model.w.device
    X = _feat_tensor(ds.features, dev)
    y = _labels_tensor(ds.labels, dev)
    _check_labels(y, model.num_classes)
    n = int(y.shape[0])
    F = model.num_features
    blocks = fastfood.build_blocks(spec, dev) if spec is not None else None
    phi = torch.empty((min(chunk, max(n, 1)), F), dtype=torch.float32, device=dev)
    head = _Head(phi.shape[0], F, model.num_classes, dev)
    nchunks = max((n + chunk - 1) // chunk, 1)
    ls = torch.zeros(nchunks, dtype=torch.float64, device=dev)
    hs = torch.zeros(nchunks, dtype=torch.int64, device=dev)
    for k, s0 in enumerate(range(0, n, chunk)):
        m = min(chunk, n - s0)
        if spec is None:
            phi[:m].copy_(X[s0:s0 + m])
        else:
            fastfood.feature_map_batch(spec, blocks, X[s0:s0 + m], normalize=False, out=phi)
        head.forward(phi, m, model, labels=y[s0:s0 + m], delta=False,
                     loss_sum=ls.data_ptr() + 8 * k, hits=hs.data_ptr() + 8 * k)
    return int(hs.sum().item()) / n, float(ls.sum().item()) / n


# -- checkpoints (MCKMODL1, linear_model.py:248-272) ------------------------

MODEL_MAGIC = b"MCKMODL1"


def save_model(path, model: SoftmaxModel, spec) -> None:
    """Magic, spec text, then W and b float64 records -- readable by the reference's load_model."""
    from . import dataio
    config = fastfood.spec_to_config(spec) if spec is not None else "kernel=none\n"
    payload = config.encode("utf-8")
    w, b = model.numpy()
    with open(path, "wb") as f:
        f.write(MODEL_MAGIC)
        f.write(len(payload).to_bytes(4, "little"))
        f.write(payload)
        dataio.write_matrix_record(f, np.ascontiguousarray(w, dtype=np.float64))
        dataio.write_matrix_record(f, np.ascontiguousarray(b, dtype=np.float64)[None, :])


def read_model_arrays(path):
    """(W, b, spec) from an MCKMODL1 file, host-side (no GPU needed)."""
    from . import dataio
    with open(path, "rb") as f:
        magic = f.read(8)
        if magic != MODEL_MAGIC:
            raise ValueError(f"{path}: not a model checkpoint (magic {magic!r})")
        size = int.from_bytes(f.read(4), "little")
        config = f.read(size).decode("utf-8")
        w = dataio.read_matrix_record(f)
        b = dataio.read_matrix_record(f)[0]
    spec = None if "kernel=none" in config else fastfood.spec_from_config(config)
    return w, b, spec


def load_model(path, device=None):
    """Inverse of :func:`save_model`; the model is placed on the GPU."""
    w, b, spec = read_model_arrays(path)
    return SoftmaxModel(w, b, device), spec
