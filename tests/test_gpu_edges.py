"""Edge cases of the drop-in API on the GPU: empty and single-row batches,
empty row gathers, unaligned input widths, a rank shard with no rows, and
the error behaviour the reference's callers rely on (fastfood.py:170-183,
wht.py:152-158)."""

import numpy as np
import pytest

from oracle import fastfood as off
from paper_1702_08159_b200 import synthetic

pytestmark = pytest.mark.gpu


def test_empty_and_single_row_batches(cuda):
    import paper_1702_08159_b200 as P
    torch = cuda
    spec = P.FeatureMapSpec(784, 2, P.RBF(1.0), 3)
    bs = P.build_blocks(spec)
    # numpy in -> numpy out, empty batch
    out = P.feature_map_batch(spec, bs, np.zeros((0, 784), dtype=np.float32))
    assert isinstance(out, np.ndarray) and out.shape == (0, P.feature_dim(spec))
    z = P.apply_zhat_batch(spec, bs, torch.zeros((0, 784), device="cuda"))
    assert tuple(z.shape) == (0, spec.padded_dim * spec.expansions)
    # empty row gather
    x = torch.from_numpy(synthetic.image_rows(5, 784, 1)).cuda()
    e = P.feature_map_batch(spec, bs, x, rows=torch.zeros(0, dtype=torch.int64, device="cuda"))
    assert tuple(e.shape) == (0, P.feature_dim(spec))
    # single row (1-D input, feature_map) against the oracle
    ospec = off.OSpec.of(spec)
    ob = off.build_blocks(ospec)
    v = synthetic.image_rows(1, 784, 2)[0]
    got = P.feature_map(spec, bs, v)
    np.testing.assert_allclose(np.asarray(got), off.feature_map_batch(ospec, ob, v[None])[0],
                               rtol=1e-5, atol=1e-6)


def test_empty_transform_and_errors(cuda):
    import paper_1702_08159_b200 as P
    torch = cuda
    a = torch.zeros((0, 1024), device="cuda")
    assert P.wht_fast_batch(a) is a                     # returns its argument (wht.py:147)
    with pytest.raises(ValueError, match="not a power of two"):
        P.wht_fast_batch(torch.zeros((2, 1000), device="cuda"))
    spec = P.FeatureMapSpec(30, 1, P.RBF(1.0), 1)
    bs = P.build_blocks(spec)
    with pytest.raises(ValueError, match="features"):
        P.feature_map_batch(spec, bs, np.zeros((2, 31), dtype=np.float32))
    with pytest.raises(ValueError, match="rows must lie in"):
        P.feature_map_batch(spec, bs, np.zeros((2, 30), dtype=np.float32),
                            rows=torch.tensor([0, 2], device="cuda"))
    with pytest.raises(ValueError, match="float32"):
        P.feature_map_batch(spec, bs, torch.zeros((2, 30), device="cuda"),
                            out=torch.zeros((2, 64), dtype=torch.float16, device="cuda"))


@pytest.mark.parametrize("d", [1, 3, 783, 1023])
def test_unaligned_widths_match_oracle(cuda, d):
    """Row widths that are not a multiple of 4 take the scalar input path:
    z within 2e-6 * max|z| of the oracle, normalised features within rtol
    1e-5 / atol 1e-6 (inputs scaled like the configs' rows, |z| of order 1-10)."""
    import paper_1702_08159_b200 as P
    spec = P.FeatureMapSpec(d, 3, P.RBF(1.0), 40 + d)
    bs = P.build_blocks(spec)
    x = (0.1 * np.random.default_rng(d).standard_normal((9, d))).astype(np.float32)
    ospec = off.OSpec.of(spec)
    ob = off.build_blocks(ospec)
    zg = P.apply_zhat_batch(spec, bs, x)
    zo = off.apply_zhat_batch(ospec, ob, x)
    assert np.abs(zg - zo).max() <= 2e-6 * np.abs(zo).max()
    np.testing.assert_allclose(P.feature_map_batch(spec, bs, x), off.feature_map_batch(ospec, ob, x),
                               rtol=1e-5, atol=1e-6)


def test_fused_step_with_an_empty_shard(cuda):
    """A rank whose shard of the global batch is empty leaves W and b alone
    (its partial gradient is zero) -- the single-rank update path with 0 rows."""
    import paper_1702_08159_b200 as P
    from paper_1702_08159_b200.large_scale import FusedClassifier
    torch = cuda
    spec = P.FeatureMapSpec(256, 2, P.RBF(1.0), 5)
    fc = FusedClassifier(spec, 10, 16)
    fc.w.normal_()
    w0, b0 = fc.w.clone(), fc.b.clone()
    x = torch.randn((16, 256), device="cuda")
    y = torch.randint(0, 10, (16,), device="cuda", dtype=torch.int32)
    fc.step(x, y, m_total=32, lr=0.1)                       # a non-empty step first
    w0, b0 = fc.w.clone(), fc.b.clone()
    fc.step(x, y, rows=torch.zeros(0, dtype=torch.int32, device="cuda"), m_total=32, lr=0.1)
    assert torch.equal(fc.w, w0) and torch.equal(fc.b, b0)
    assert fc.loss_sum.item() == 0.0 and fc.hits.item() == 0   # no stale loss from the last step


def test_wht_naive_and_scalar_draws(cuda):
    """wht_naive (wht.py:67-87) against the oracle's float64 product, and the
    scalar draws of RandomStream (detrand.py:136-153) against its arrays."""
    import paper_1702_08159_b200 as P
    from oracle import wht as ow
    v = np.random.default_rng(3).standard_normal((256, 3))
    got = P.wht_naive(v)
    np.testing.assert_allclose(got, ow.wht_naive(v), rtol=1e-12, atol=1e-10)
    assert P.wht_naive(v[:, 0]).shape == (256,)
    a, b = P.RandomStream(42, "u", 3), P.RandomStream(42, "u", 3)
    arr = a.uniform01_array(5).cpu().numpy()
    assert [b.uniform01() for _ in range(5)] == arr.tolist()
    a, b = P.RandomStream(7, "g"), P.RandomStream(7, "g")
    arr = a.gaussian_array(5).cpu().numpy()         # pair cache shared with gaussian()
    assert [b.gaussian() for _ in range(5)] == arr.tolist()
    a, b = P.RandomStream(9, "s"), P.RandomStream(9, "s")
    assert [b.sign_pm1() for _ in range(4)] == a.sign_array(4).cpu().numpy().tolist()
