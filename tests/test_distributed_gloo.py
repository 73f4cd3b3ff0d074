"""Multi-process data-parallel plumbing on CPU (gloo, world_size 2).

Each rank takes its contiguous shard of every global mini-batch
(distributed.shard_range), forms its partial [dW | db | loss_sum] with
delta normalised by the GLOBAL batch size -- the convention of
mck_head_forward(m_total=...) -- packs it into a GradBucket and all-reduces.
The reduced gradient must equal the single-process gradient of the whole
batch, and both ranks must hold identical weights after every SGD step.
The per-rank arithmetic here is the oracle's (numpy); on GPUs the same
plumbing wraps the CUDA kernels (linear_model.Trainer.step).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import fastfood as off
from oracle import linear_model as olm
from paper_1702_08159_b200 import synthetic
from paper_1702_08159_b200.distributed import GradBucket, shard_range

WORLD = 2


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem():
    spec = off.OSpec(20, 2, "rbf", 1.0, 0, 5)
    blocks = off.build_blocks(spec)
    x, y = synthetic.class_images(120, 20, 10, seed=8, sample_seed=9, noise=0.2)
    phi = off.feature_map_batch(spec, blocks, x, normalize=False).astype(np.float64)
    return phi, y


def _local_partial(w, b, phi, y, lo, hi, m_total):
    """Rank-local [dW | db | loss_sum] with delta / m_total (mck_head_forward convention)."""
    p = olm.forward_batch(w, b, phi[lo:hi])
    loss_sum = float(-np.log(np.maximum(p[np.arange(hi - lo), y[lo:hi]], 1e-300)).sum())
    d = p.copy()
    d[np.arange(hi - lo), y[lo:hi]] -= 1.0
    d /= m_total
    return d.T @ phi[lo:hi], d.sum(axis=0), loss_sum


def _worker(rank, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    phi, y = _problem()
    C, F = 10, phi.shape[1]
    w, b = np.zeros((C, F)), np.zeros(C)
    order = olm.epoch_order(3, 0, len(y))
    lr, batch = 0.05, 50
    losses = []
    for s0 in range(0, len(y), batch):                    # last batch partial (20 rows)
        idx = order[s0:s0 + batch]
        mg = len(idx)
        lo, hi = shard_range(mg, rank, WORLD)
        bucket = GradBucket.empty(C, F, "cpu")
        dw, db, ls = _local_partial(w, b, phi[idx], y[idx], lo, hi, mg)
        bucket.dw.copy_(torch.from_numpy(dw))
        bucket.db.copy_(torch.from_numpy(db))
        bucket.loss_sum.fill_(ls)
        bucket.allreduce()
        # reference: full-batch gradient in one process
        rdw, rdb = olm.gradients(w, b, phi[idx], y[idx])
        assert np.allclose(bucket.dw.numpy(), rdw, rtol=1e-12, atol=1e-15)
        assert np.allclose(bucket.db.numpy(), rdb, rtol=1e-12, atol=1e-15)
        rl = olm.loss(w, b, phi[idx], y[idx])
        assert abs(float(bucket.loss_sum) / mg - rl) <= 1e-12 * abs(rl)
        losses.append(float(bucket.loss_sum) / mg)
        w -= lr * bucket.dw.numpy()
        b -= lr * bucket.db.numpy()
    # identical replicas on every rank
    chk = torch.tensor([w.sum(), (w * w).sum(), b.sum()], dtype=torch.float64)
    gathered = [torch.zeros(3, dtype=torch.float64) for _ in range(WORLD)]
    dist.all_gather(gathered, chk)
    assert all(torch.equal(g, gathered[0]) for g in gathered)
    np.save(os.path.join(out_dir, f"rank{rank}_w.npy"), w)
    np.save(os.path.join(out_dir, f"rank{rank}_losses.npy"), np.array(losses))
    dist.destroy_process_group()


def test_two_rank_allreduce_matches_single_process(tmp_path):
    port = _free_port()
    mp.start_processes(_worker, args=(port, str(tmp_path)), nprocs=WORLD, join=True,
                       start_method="spawn")
    w0 = np.load(tmp_path / "rank0_w.npy")
    w1 = np.load(tmp_path / "rank1_w.npy")
    assert np.array_equal(w0, w1)
    # and the replicated trajectory equals single-process SGD to roundoff
    phi, y = _problem()
    w, b = np.zeros((10, phi.shape[1])), np.zeros(10)
    order = olm.epoch_order(3, 0, len(y))
    for s0 in range(0, len(y), 50):
        idx = order[s0:s0 + 50]
        olm.sgd_step(w, b, phi[idx], y[idx], 0.05)
    np.testing.assert_allclose(w0, w, rtol=1e-11, atol=1e-14)


def test_shards_cover_every_row_once():
    for mg in (1, 2, 49, 50, 1000):
        covered = []
        for r in range(WORLD):
            lo, hi = shard_range(mg, r, WORLD)
            covered.extend(range(lo, hi))
        assert covered == list(range(mg))
