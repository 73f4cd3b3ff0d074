"""C-ABI surface and host-side logic (no GPU needed)."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT, load_npz

HEADER = ROOT / "include" / "mckernel_b200.h"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mck_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_1702_08159_b200 import _native
    if not _native.LIB_PATH.exists():
        pytest.fail("libmckernel_b200.so is not built (run __graft_entry__.build())")
    return _native.lib()


def test_library_exports_every_declared_symbol(lib):
    names = declared_functions()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), f"{name} declared in the header but not exported"


def test_ctypes_signatures_cover_header():
    from paper_1702_08159_b200 import _native
    assert sorted(_native.SIGNATURES) == declared_functions()


def test_stream_key_matches_reference_golden(lib):
    import json
    z = load_npz("detrand.npz")
    cases = json.loads(str(z["cases"][0]))
    from paper_1702_08159_b200.detrand import stream_key
    for k, (seed, label, block) in enumerate(cases):
        assert stream_key(seed, label, block) == int(z[f"key{k}"][0])


def test_validation_errors_without_gpu(lib):
    from paper_1702_08159_b200 import _native as nat
    with pytest.raises(ValueError, match="not a power of two"):
        nat.call("mck_fwht_f32", None, 1, 12, 0, None)
    with pytest.raises(ValueError, match="sigma must be positive"):
        nat.call("mck_tables_build", None, 784, 8, 0, 0.0, 0, 1, None)
    with pytest.raises(ValueError, match="t must be a positive integer"):
        nat.call("mck_tables_build", None, 784, 8, 1, 1.0, 0, 1, None)
    with pytest.raises(ValueError, match="expansions must be positive"):
        nat.call("mck_tables_build", None, 784, 0, 0, 1.0, 0, 1, None)
    with pytest.raises(ValueError, match="empty permutation"):
        nat.call("mck_fisher_yates", 1, b"x", 0, 1, 0, None, None)
    assert lib.mck_abi_version() == 1
    assert lib.mck_tables_bytes(1024, 8) > 28 * 1024 * 8


class TestSpec:
    def test_padding_and_dims(self):
        from paper_1702_08159_b200 import RBF, FeatureMapSpec, feature_dim, param_count
        assert FeatureMapSpec(3, 1, RBF(1.0), 0).padded_dim == 4
        assert FeatureMapSpec(784, 1, RBF(1.0), 0).padded_dim == 1024
        assert FeatureMapSpec(1024, 1, RBF(1.0), 0).padded_dim == 1024
        s = FeatureMapSpec(784, 8, RBF(1.0), 1234)
        assert feature_dim(s) == 16384
        assert param_count(s, 10) == 10 * 16385
        with pytest.raises(ValueError):
            param_count(s, 1)

    def test_validation_messages(self):
        from paper_1702_08159_b200 import RBF, FeatureMapSpec, RBFMatern
        with pytest.raises(ValueError, match="input_dim must be positive"):
            FeatureMapSpec(0, 1, RBF(1.0), 0)
        with pytest.raises(ValueError, match="expansions must be positive"):
            FeatureMapSpec(4, 0, RBF(1.0), 0)
        with pytest.raises(ValueError, match="sigma must be positive"):
            RBF(0.0)
        with pytest.raises(ValueError, match="t must be a positive integer"):
            RBFMatern(1.0, 0)

    def test_train_config_validation(self):
        from paper_1702_08159_b200 import TrainConfig
        for kw in (dict(learning_rate=0.0, batch_size=1, epochs=1),
                   dict(learning_rate=0.1, batch_size=0, epochs=1),
                   dict(learning_rate=0.1, batch_size=1, epochs=-1),
                   dict(learning_rate=0.1, batch_size=1, epochs=1, l2_lambda=-1.0)):
            with pytest.raises(ValueError):
                TrainConfig(**kw)

    def test_wht_shape_errors_before_device(self):
        from paper_1702_08159_b200 import wht_fast, wht_fast_batch
        with pytest.raises(ValueError, match="not a power of two"):
            wht_fast(np.ones(12, dtype=np.float32))
        with pytest.raises(ValueError, match="1-D"):
            wht_fast(np.ones((4, 4), dtype=np.float32))
        with pytest.raises(ValueError, match=r"\(m, n\)"):
            wht_fast_batch(np.ones(4, dtype=np.float32))


class TestSharding:
    def test_shard_range_partitions(self):
        from paper_1702_08159_b200.distributed import shard_range
        for m in (0, 1, 7, 125, 1000, 1001):
            for ws in (1, 2, 3, 4, 8):
                parts = [shard_range(m, r, ws) for r in range(ws)]
                assert parts[0][0] == 0 and parts[-1][1] == m
                for (a, b), (c, d) in zip(parts, parts[1:]):
                    assert b == c
                sizes = [b - a for a, b in parts]
                assert max(sizes) - min(sizes) <= 1
        with pytest.raises(ValueError):
            shard_range(10, 2, 2)

    def test_grad_bucket_views(self):
        import torch
        from paper_1702_08159_b200.distributed import GradBucket
        b = GradBucket.empty(3, 5, "cpu")
        b.dw.fill_(1.0)
        b.db.fill_(2.0)
        b.loss_sum.fill_(3.0)
        b.hits.fill_(4.0)
        assert b.flat.shape == (3 * 5 + 3 + 2,)
        assert b.flat[:15].sum() == 15 and b.flat[15:18].sum() == 6
        assert float(b.flat[-2]) == 3.0 and float(b.flat[-1]) == 4.0
        assert b.dw.data_ptr() == b.flat.data_ptr()
        assert isinstance(b.flat, torch.Tensor)


@pytest.mark.parametrize("m,kind", [(32, "random"), (512, "random"), (32, "parallel"), (64, "strided")])
def test_edge_colouring_of_permutation_graphs(lib, m, kind):
    # the layout of Pi in shared memory (perm_color.cu): every scatter group
    # and every gather group must see 32 distinct banks
    n = 32 * m
    rng = np.random.default_rng(m)
    left = (np.arange(n) // 32).astype(np.int32)
    if kind == "random":
        right = (rng.permutation(n) // 32).astype(np.int32)
    elif kind == "parallel":      # identity permutation: 32 parallel edges per pair
        right = left.copy()
    else:                         # transpose-like permutation
        right = (np.arange(n) % m).astype(np.int32)
    col = np.zeros(n, dtype=np.uint8)
    def ptr(a):
        return a.ctypes.data
    rc = lib.mck_diag_edge_color32(m, ptr(left), ptr(right), ptr(col))
    assert rc == 0
    assert col.max() < 32
    for side in (left, right):
        pairs = side.astype(np.int64) * 32 + col
        assert len(np.unique(pairs)) == n


def test_edge_colouring_rejects_irregular_graph(lib):
    def ptr(a):
        return a.ctypes.data
    m = 4
    left = (np.arange(128) // 32).astype(np.int32)
    right = np.zeros(128, dtype=np.int32)          # right node 0 has degree 128
    col = np.zeros(128, dtype=np.uint8)
    assert lib.mck_diag_edge_color32(m, ptr(left), ptr(right), ptr(col)) == 1
