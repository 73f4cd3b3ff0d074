"""Oracle restatement of the reference softmax head and SGD trainer.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Follows ``pkg/src/mckernel/linear_model.py``:

* ``softmax_rows``  -- linear_model.py:79-83
* ``forward_batch`` -- linear_model.py:95-97 (float64 logits on fp32 features)
* ``loss``          -- linear_model.py:105-115
* ``gradients``     -- linear_model.py:118-131
* ``sgd_step``      -- linear_model.py:134-142
* ``train``         -- linear_model.py:191-223 (shuffle stream ("shuffle", epoch))
* ``evaluate``      -- linear_model.py:226-239 (512-row chunks)
"""

from __future__ import annotations

import numpy as np

from . import detrand
from . import fastfood as off


def softmax_rows(logits: np.ndarray) -> np.ndarray:
    z = logits - logits.max(axis=1, keepdims=True)
    np.exp(z, out=z)
    z /= z.sum(axis=1, keepdims=True)
    return z


def forward_batch(w, b, x):
    return softmax_rows(np.asarray(x @ w.T + b, dtype=np.float64))


def loss(w, b, x, y, l2=0.0) -> float:
    p = forward_batch(w, b, x)
    ce = float(-np.log(np.maximum(p[np.arange(len(y)), y], 1e-300)).mean())
    if l2:
        ce += l2 * float((w * w).sum())
    return ce


def gradients(w, b, x, y, l2=0.0):
    x = np.asarray(x, dtype=np.float64)
    m = x.shape[0]
    d = forward_batch(w, b, x)
    d[np.arange(m), y] -= 1.0
    d /= m
    dw = d.T @ x
    if l2:
        dw += 2.0 * l2 * w
    return dw, d.sum(axis=0)


def sgd_step(w, b, x, y, lr, l2=0.0):
    dw, db = gradients(w, b, x, y, l2)
    w -= lr * dw
    b -= lr * db


def epoch_order(shuffle_seed: int, epoch: int, n: int) -> np.ndarray:
    """linear_model.py:210-211."""
    return detrand.fisher_yates(detrand.Stream(shuffle_seed, "shuffle", epoch), n)


def evaluate(w, b, featurize, x, y, chunk=512):
    hits, tot = 0, 0.0
    for s in range(0, len(y), chunk):
        p = forward_batch(w, b, featurize(x[s:s + chunk]))
        yy = y[s:s + chunk]
        hits += int((p.argmax(axis=1) == yy).sum())
        tot += float(-np.log(np.maximum(p[np.arange(len(yy)), yy], 1e-300)).sum())
    return hits / len(y), tot / len(y)


def train(spec, x, y, xt, yt, num_classes, lr, batch, epochs, l2=0.0, shuffle_seed=0,
          blocks=None):
    """linear_model.py:191-223; returns (w, b, [(epoch, mean_loss, test_acc)])."""
    if spec is None:
        featurize = lambda a: a                      # noqa: E731
        fdim = x.shape[1]
    else:
        blocks = blocks if blocks is not None else off.build_blocks(spec)
        featurize = lambda a: off.feature_map_batch(spec, blocks, a, normalize=False)  # noqa: E731
        fdim = 2 * spec.n * spec.expansions
    w = np.zeros((num_classes, fdim))
    b = np.zeros(num_classes)
    hist = []
    n = len(y)
    for ep in range(epochs):
        order = epoch_order(shuffle_seed, ep, n)
        tot, nb = 0.0, 0
        for s in range(0, n, batch):
            idx = order[s:s + batch]
            xb = featurize(x[idx])
            yb = y[idx]
            tot += loss(w, b, xb, yb, l2)
            sgd_step(w, b, xb, yb, lr, l2)
            nb += 1
        acc, _ = evaluate(w, b, featurize, xt, yt)
        hist.append((ep, tot / nb, acc))
    return w, b, hist
