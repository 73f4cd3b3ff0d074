"""Multi-rank training paths on the GPU: two processes, world size 2.

Only one GPU is available to the tests, so both ranks share cuda:0 and the
process group is gloo (its all-reduce of CUDA tensors goes through host
memory; the kernels of one rank never wait on the other's).  The code under
test is the product's own multi-rank path -- ``linear_model.train`` /
``Trainer.run_epoch`` (batch shards, float64 [dW | db | loss] all-reduce
overlapped with the next batch's expansion) and ``FusedClassifier.step``
(bucketed float32 dW all-reduce) -- compared with the single-process run of
the same problem:

* both ranks end with bit-identical weights (the update is replicated);
* Trainer (float64 head): W within 1e-10 relative of single-process training
  (the two partial sums of each gradient are added in a different order);
* FusedClassifier (float32 W): W within 1e-6 relative.

Reference semantics: linear_model.py:191-223 (batch order, one update per
global batch), linear_model.py:118-142 (gradient and update).
"""

import os
import socket

import numpy as np
import pytest

from paper_1702_08159_b200 import synthetic

pytestmark = pytest.mark.gpu

WORLD = 2


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _trainer_problem():
    import paper_1702_08159_b200 as P
    spec = P.FeatureMapSpec(784, 2, P.RBF(1.0), 1234)
    x, y = synthetic.class_images(1100, 784, 10, seed=3, sample_seed=4, noise=0.25)
    xt, yt = synthetic.class_images(300, 784, 10, seed=3, sample_seed=5, noise=0.25)
    cfg = P.TrainConfig(0.05, 200, 2, shuffle_seed=9)        # 6 steps/epoch, the last 100 rows
    return spec, P.Dataset(x, y, 10), P.Dataset(xt, yt, 10), cfg


def _fused_problem():
    import paper_1702_08159_b200 as P
    spec = P.FeatureMapSpec(1000, 5, P.RBF(2.0), 17)          # n = 1024; buckets of 2, 2, 1 blocks
    x = np.random.default_rng(2).standard_normal((96, 1000)).astype(np.float32)
    y = np.random.default_rng(3).integers(0, 10, 96).astype(np.int32)
    return spec, x, y


def _run_fused(spec, x, y, rank, ws, steps=4, batch=48):
    import torch
    from paper_1702_08159_b200.large_scale import FusedClassifier
    from paper_1702_08159_b200.distributed import shard_range
    fc = FusedClassifier(spec, 10, batch, bucket_blocks=2)
    X = torch.from_numpy(x).cuda()
    Y = torch.from_numpy(y).cuda()
    losses = []
    for s in range(steps):
        g0 = (s * batch) % len(y)
        lo, hi = shard_range(batch, rank, ws)
        rows = torch.arange(g0 + lo, g0 + hi, dtype=torch.int32, device="cuda")
        fc.step(X, Y, rows=rows, m_total=batch, lr=0.02, l2=1e-4)
        losses.append(fc.loss_sum.item() / batch)
    return fc.w.cpu().numpy(), fc.b.cpu().numpy(), np.array(losses)


def _worker(rank, port, out_dir):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    import paper_1702_08159_b200 as P
    spec, tr, te, cfg = _trainer_problem()
    model, metrics = P.train(spec, tr, te, cfg)
    w, b = model.numpy()
    np.save(os.path.join(out_dir, f"tr_w{rank}.npy"), w)
    np.save(os.path.join(out_dir, f"tr_b{rank}.npy"), b)
    np.save(os.path.join(out_dir, f"tr_hist{rank}.npy"),
            np.array([[r.train_loss, r.test_acc] for r in metrics.records]))
    fspec, x, y = _fused_problem()
    fw, fb, fl = _run_fused(fspec, x, y, rank, WORLD)
    np.save(os.path.join(out_dir, f"fu_w{rank}.npy"), fw)
    np.save(os.path.join(out_dir, f"fu_b{rank}.npy"), fb)
    np.save(os.path.join(out_dir, f"fu_l{rank}.npy"), fl)
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_match_single_process(cuda, tmp_path):
    import torch.multiprocessing as mp
    import paper_1702_08159_b200 as P
    mp.start_processes(_worker, args=(_free_port(), str(tmp_path)), nprocs=WORLD, join=True,
                       start_method="spawn")
    ld = lambda k: np.load(tmp_path / f"{k}.npy")              # noqa: E731
    # replicas are identical bit for bit
    for k in ("tr_w", "tr_b", "tr_hist", "fu_w", "fu_b", "fu_l"):
        assert np.array_equal(ld(k + "0"), ld(k + "1")), k
    # Trainer: the sharded run equals single-process training
    spec, tr, te, cfg = _trainer_problem()
    model, metrics = P.train(spec, tr, te, cfg)
    w, b = model.numpy()
    np.testing.assert_allclose(ld("tr_w0"), w, rtol=0, atol=1e-10 * np.abs(w).max())
    np.testing.assert_allclose(ld("tr_b0"), b, rtol=0, atol=1e-10 * np.abs(b).max())
    hist = np.array([[r.train_loss, r.test_acc] for r in metrics.records])
    np.testing.assert_allclose(ld("tr_hist0")[:, 0], hist[:, 0], rtol=1e-10)
    assert np.array_equal(ld("tr_hist0")[:, 1], hist[:, 1])
    # FusedClassifier: bucketed all-reduce vs the fused single-rank update
    fspec, x, y = _fused_problem()
    fw, fb, fl = _run_fused(fspec, x, y, 0, 1)
    assert np.abs(ld("fu_w0") - fw).max() <= 1e-6 * np.abs(fw).max()
    np.testing.assert_allclose(ld("fu_b0"), fb, rtol=1e-6, atol=1e-9)
    np.testing.assert_allclose(ld("fu_l0"), fl, rtol=1e-5, atol=1e-12)
