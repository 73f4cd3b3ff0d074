"""K6 (config 4): fused expansion -> classifier against the materialised path.

The materialised path is the parity-tested expansion (test_gpu_parity.py)
followed by the same softmax arithmetic in float64 (linear_model.py:95-131):
logits = phi W^T, delta = (softmax(logits + b) - onehot)/m, dW = delta^T phi.
Tolerances: the fused contraction accumulates in float32 within 512-feature
chunks and in float64 across chunks -> logits within 1e-5 of max|logits|,
dW within 1e-4 of max|dW|.
"""

import numpy as np
import pytest

from paper_1702_08159_b200 import synthetic

pytestmark = pytest.mark.gpu


def _case(cuda, spec, m, seed, engine="ffma2", keep_z=True):
    import paper_1702_08159_b200 as P
    from paper_1702_08159_b200.large_scale import FusedClassifier
    torch = cuda
    g = torch.Generator(device="cuda").manual_seed(seed)
    if spec.input_dim == 784:
        x = torch.from_numpy(synthetic.image_rows(m, 784, seed)).cuda()
    else:
        x = torch.randn((m, spec.input_dim), generator=g, device="cuda")
    y = torch.randint(0, 10, (m,), generator=g, device="cuda", dtype=torch.int32)
    fc = FusedClassifier(spec, 10, m, engine=engine, keep_z=keep_z)
    fc.w.copy_(torch.randn(fc.w.shape, generator=g, device="cuda") * 0.01)
    fc.b.copy_(torch.randn(10, generator=g, device="cuda", dtype=torch.float64) * 0.1)
    phi = P.feature_map_batch(spec, fc.blocks, x, normalize=False).double()
    return fc, x, y, phi


@pytest.mark.parametrize("keep_z", [True, False], ids=["keep_z", "recompute_z"])
@pytest.mark.parametrize("engine", ["ffma2", "tcgen05", "reference"])
@pytest.mark.parametrize("which", ["small", "ragged", "c4"])
def test_fused_forward_backward(cuda, which, engine, keep_z):
    import paper_1702_08159_b200 as P
    torch = cuda
    if which == "small":
        spec, m = P.FeatureMapSpec(784, 4, P.RBF(1.0), 3), 96
    elif which == "ragged":  # m*C not a multiple of 4, partial row tile / stage
        spec, m = P.FeatureMapSpec(300, 2, P.RBF(1.0), 8), 37
    else:
        spec, m = P.FeatureMapSpec(16384, 32, P.RBF(4.0), 4), 8
    fc, x, y, phi = _case(cuda, spec, m, 11, engine, keep_z)
    logits = torch.empty((m, 10), dtype=torch.float64, device="cuda")
    probs = torch.empty((m, 10), dtype=torch.float64, device="cuda")
    fc.forward(x, y, logits=logits, probs=probs)
    want = phi @ fc.w.double().T
    err = (logits - want).abs().max().item()
    assert err <= 1e-5 * want.abs().max().item(), err
    p = torch.softmax(want + fc.b, dim=1)
    # |dp| <= max|d logits| (softmax is 1-Lipschitz in the max norm up to a factor 1/2)
    assert (probs - p).abs().max().item() <= max(1e-6, 1.0 * err)
    loss = -torch.log(p[torch.arange(m), y.long()]).sum().item()
    assert abs(fc.loss_sum.item() - loss) <= 1e-5 * abs(loss)
    delta = p.clone()
    delta[torch.arange(m), y.long()] -= 1.0
    delta /= m
    assert (fc.delta[:m] - delta).abs().max().item() <= max(1e-7, err / m)
    dw, db = fc.backward()
    dw = dw.double()
    dw_ref = delta.T @ phi
    assert (dw - dw_ref).abs().max().item() <= 1e-4 * dw_ref.abs().max().item()
    assert torch.allclose(db, fc.delta[:m].sum(0), rtol=1e-12, atol=1e-15)
    assert torch.allclose(db, delta.sum(0), rtol=1e-5, atol=max(1e-8, err))


@pytest.mark.parametrize("engine", ["ffma2", "tcgen05", "reference"])
def test_fused_sgd_update_and_gather(cuda, engine):
    import paper_1702_08159_b200 as P
    torch = cuda
    spec = P.FeatureMapSpec(784, 4, P.RBF(1.0), 3)
    fc, x, y, phi = _case(cuda, spec, 128, 5, engine)
    rows = torch.tensor(list(range(0, 128, 2)), dtype=torch.int32, device="cuda")
    w0, b0 = fc.w.clone(), fc.b.clone()
    fc.forward(x, y, rows=rows, m_total=64)
    ph = phi[rows.long()]
    p = torch.softmax(ph @ w0.double().T + b0, dim=1)
    d = p.clone()
    d[torch.arange(64), y[rows.long()].long()] -= 1.0
    d /= 64
    assert (fc.delta[:64] - d).abs().max().item() <= 1e-7
    fc.backward(lr=0.5)
    w_ref = w0.double() - 0.5 * (d.T @ ph)
    assert (fc.w.double() - w_ref).abs().max().item() <= 1e-6
    assert torch.allclose(fc.b, b0 - 0.5 * d.sum(0), rtol=1e-6, atol=1e-9)


@pytest.mark.parametrize("engine", ["ffma2", "tcgen05", "reference"])
def test_bucketed_backward_equals_plain(cuda, engine):
    """The multi-rank backward (one all-reduce bucket per block range) writes
    the same float32 dW as the single-rank backward, bit for bit, and the
    bucket update equals the fused update."""
    import paper_1702_08159_b200 as P
    from paper_1702_08159_b200 import _native as nat
    torch = cuda
    spec = P.FeatureMapSpec(1000, 5, P.RBF(1.0), 21)        # n = 1024, ragged last bucket
    fc, x, y, _ = _case(cuda, spec, 70, 13, engine)
    fc.bucket_blocks = 2
    m = fc.forward(x, y)
    dw, db = fc.backward()
    n, D = spec.padded_dim, spec.padded_dim * spec.expansions
    fc._alloc_buckets()
    st = nat.stream_handle(fc.dev)
    for (e0, cnt), buf in zip(fc.bucket_ranges(), fc._buckets):
        nat.call("mck_fused_backward_bucket", *fc._bwd_args(), e0, cnt, nat.ptr(buf),
                 nat.ptr(fc.scratch), fc.variant, st)
        want = torch.cat([dw[:, e0 * n:(e0 + cnt) * n], dw[:, D + e0 * n:D + (e0 + cnt) * n]], dim=1)
        assert torch.equal(buf, want), (e0, cnt)
    nat.call("mck_fused_bias_grad", nat.ptr(fc.delta), m, 10, nat.ptr(fc._tail), st)
    assert torch.equal(fc._tail[:10], db)
    w0, b0 = fc.w.clone(), fc.b.clone()
    for k, ((e0, cnt), buf) in enumerate(zip(fc.bucket_ranges(), fc._buckets)):
        last = k == len(fc._buckets) - 1
        nat.call("mck_fused_apply_bucket", nat.ptr(fc.w), spec.input_dim, spec.expansions, 10, e0,
                 cnt, nat.ptr(buf), 0.3, 1e-3, nat.ptr(fc.b) if last else None,
                 nat.ptr(fc._tail) if last else None, st)
    w_bucket, b_bucket = fc.w.clone(), fc.b.clone()
    fc.w.copy_(w0)
    fc.b.copy_(b0)
    fc.forward(x, y)
    fc.backward(lr=0.3, l2=1e-3)
    assert torch.equal(w_bucket, fc.w)
    assert torch.equal(b_bucket, fc.b)


def test_fused_training_trajectory_vs_oracle(cuda):
    """Twenty-plus SGD steps of the fused classifier (float32 W, 3xTF32
    tensor-core contractions) against the float64 reference trainer
    (oracle.linear_model.train = linear_model.py:191-223) on the same
    shuffles: per-epoch mean loss within 1e-4 relative, test accuracy within
    0.2 percentage points, and the float32-W drift bounded."""
    import paper_1702_08159_b200 as P
    from oracle import fastfood as off
    from oracle import linear_model as olm
    from paper_1702_08159_b200.detrand import fisher_yates_permutations
    from paper_1702_08159_b200.large_scale import FusedClassifier
    torch = cuda
    spec = P.FeatureMapSpec(3000, 4, P.RBF(4.0), 77)          # n = 4096, 32768 features
    # noisy classes and a small step: the loss goes 2.07 -> 0.19 and test
    # accuracy stays near 87 % (neither saturated nor degenerate)
    x, y = synthetic.class_images(1200, 3000, 10, seed=5, sample_seed=6, noise=1.0)
    # 1,000 test rows: 0.2 percentage points = 2 rows
    xt, yt = synthetic.class_images(1000, 3000, 10, seed=5, sample_seed=7, noise=1.0)
    lr, batch, epochs = 0.02, 100, 2                          # 12 steps/epoch, 24 steps
    ospec = off.OSpec.of(spec)
    ob = off.build_blocks(ospec)
    w_ref, b_ref, hist = olm.train(ospec, x, y, xt, yt, 10, lr, batch, epochs, blocks=ob)
    fc = FusedClassifier(spec, 10, batch)
    X = torch.from_numpy(x).cuda()
    Y = torch.from_numpy(y.astype(np.int32)).cuda()
    orders = fisher_yates_permutations(0, "shuffle", 0, epochs, len(y), fc.dev)
    losses = []
    for ep in range(epochs):
        tot = 0.0
        for s0 in range(0, len(y), batch):
            rows = orders[ep, s0:s0 + batch]
            fc.step(X, Y, rows=rows, m_total=rows.shape[0], lr=lr)
            tot += fc.loss_sum.item() / rows.shape[0]
        losses.append(tot / ((len(y) + batch - 1) // batch))
    for (ep, want_loss, want_acc), got in zip(hist, losses):
        assert abs(got - want_loss) <= 1e-4 * abs(want_loss), (ep, got, want_loss)
    logits = torch.empty((len(yt), 10), dtype=torch.float64, device="cuda")
    fc2 = FusedClassifier(spec, 10, len(yt))
    fc2.w.copy_(fc.w)
    fc2.b.copy_(fc.b)
    fc2.forward(torch.from_numpy(xt).cuda(), logits=logits)
    acc = float((logits.argmax(1).cpu().numpy() == yt).mean())
    assert abs(acc - hist[-1][2]) <= 0.002 + 1e-12, (acc, hist[-1][2])
    # float32 W vs the float64 reference W: relative drift after 24 steps
    drift = np.abs(fc.w.double().cpu().numpy() - w_ref).max() / np.abs(w_ref).max()
    print(f"fused training: losses {losses} vs {[h[1] for h in hist]}; float32-W drift {drift:.3e}")
    assert drift <= 1e-4, drift
    np.testing.assert_allclose(fc.b.cpu().numpy(), b_ref, rtol=1e-4, atol=1e-7)


def test_kernel_check_bench_wht_and_feature_dump(cuda, tmp_path):
    # next-ranked items of SURVEY.md section 8f, on the GPU path
    import paper_1702_08159_b200 as P
    from paper_1702_08159_b200 import dataio
    from paper_1702_08159_b200.exact_kernel import kernel_check
    from paper_1702_08159_b200.wht import bench_wht, bench_wht_csv
    rng = np.random.default_rng(7)
    spec = P.FeatureMapSpec(64, 8, P.RBF(1.0), 31)
    pairs = [(rng.standard_normal(64) * 0.3, rng.standard_normal(64) * 0.3) for _ in range(100)]
    st = kernel_check(spec, pairs)
    assert st.D == 512 and st.pairs == 100 and st.mean_err <= 0.05      # test_fastfood.py:247-258
    recs = bench_wht([1024, 4096, 1 << 16, 1 << 20], repetitions=3)
    csv = bench_wht_csv(recs).splitlines()
    assert csv[0] == "size,impl,median_ms,reps" and len(csv) == 1 + 4 + 3
    assert all(r.fast_ms > 0 for r in recs) and recs[3].naive_ms is None
    assert recs[2].naive_ms is not None                      # naive oracle up to 2^16 (wht.py:187)
    import torch
    from paper_1702_08159_b200.wht import _naive_gpu, wht_fast
    v = torch.randn(4096, device="cuda", dtype=torch.float32)
    nv = _naive_gpu(torch, v)
    fv = wht_fast(v.clone()).double()
    assert (nv - fv).abs().max().item() <= 1e-6 * nv.abs().max().item()
    x = synthetic.image_rows(300, 784, 3)
    spec2 = P.FeatureMapSpec(784, 2, P.RBF(1.0), 9)
    bs = P.build_blocks(spec2)
    path = tmp_path / "f.mckmat"
    assert dataio.features_to_file(spec2, bs, x, path, batch_rows=128) == (300, 4096)
    got = dataio.read_matrix(path)
    np.testing.assert_array_equal(got, P.feature_map_batch(spec2, bs, x))


def test_checkpoint_round_trip_gpu(cuda, tmp_path):
    import paper_1702_08159_b200 as P
    from paper_1702_08159_b200.linear_model import load_model, save_model
    spec = P.FeatureMapSpec(20, 2, P.RBF(1.0), 5)
    m = P.SoftmaxModel(np.random.default_rng(0).standard_normal((10, 128)), np.arange(10.0))
    save_model(tmp_path / "m", m, spec)
    m2, spec2 = load_model(tmp_path / "m")
    assert spec2 == spec
    assert torch_equal(m2.w, m.w) and torch_equal(m2.b, m.b)


def torch_equal(a, b):
    return bool((a == b).all().item())


def test_bench_line_on_gpu(cuda, tmp_path):
    """bench.py's JSON contract on a GPU (short run): headline keys, the
    roofline / e2e / clocks objects and one leg per other config, each with
    a roofline."""
    import json
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    r = subprocess.run([sys.executable, str(root / "bench.py"), "--steps", "2", "--warmup", "3",
                        "--no-cpu", "--no-e2e"], cwd=root, capture_output=True, text=True,
                       timeout=900, env=dict(os.environ))
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "dtype", "config", "roofline", "clocks",
                "gpu_launches", "extras"):
        assert key in line, key
    assert line["n_gpus"] == 1 and line["gpu_launches"] == 2 * 15 and line["value"] > 0
    rf = line["roofline"]
    assert rf["bound"] == "hbm" and 0 < rf["frac"] < 1.2 and rf["peak"] > 0
    ex = line["extras"]
    for leg in ("c0", "c1_fwht_sweep", "c3_train", "c4_fused_step"):
        assert leg in ex, leg
    for leg in ("c0", "c3_train", "c4_fused_step"):
        assert ex[leg]["roofline"]["frac"] > 0
    assert len(ex["c1_fwht_sweep"]) == 11
    assert ex["c3_train"]["final_test_acc"] >= 0.9
