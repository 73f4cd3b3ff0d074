"""Pin the CPU oracle against the reference's golden vectors (no GPU).

The fixtures were produced by the reference itself (tests/golden/make_golden.py);
the constants in TestReferenceConstants are the reference tests' own goldens
(pkg/tests/test_detrand.py:22-32, pkg/tests/test_fastfood.py:28-36).
"""

import json

import numpy as np
import pytest

from conftest import load_json, load_npz
from oracle import detrand as od
from oracle import fastfood as off
from oracle import linear_model as olm
from oracle import wht as ow
from paper_1702_08159_b200 import synthetic


class TestReferenceConstants:
    def test_hash_goldens(self):
        want = {(42, "B", 0): 0x1E33DE85387EAE97, (42, "G", 0): 0xCE29D5FF2B3CD5DA,
                (43, "B", 0): 0xD3E8DB5D9D65A34D}
        for (seed, label, block), h in want.items():
            assert od.Stream(seed, label, block).hash_at(0) == h

    def test_stream_goldens_seed7(self):
        # labels "u", "g", "s" as in pkg/tests/test_detrand.py:74,107,128
        np.testing.assert_array_equal(od.Stream(7, "u", 0).uniforms(4), [0.19681970807755012, 0.3875403325733868,
                                                      0.9742781761190904, 0.6916958472993927])
        np.testing.assert_allclose(od.Stream(7, "g", 0).gaussians(4),
                                   [0.1577956022387008, -1.074844538017888,
                                    0.5536515769773818, -0.3044021609698588], rtol=1e-12)
        np.testing.assert_array_equal(od.Stream(7, "s", 0).signs(6), [-1, 1, -1, -1, 1, 1])

    def test_perm_golden(self):
        assert od.fisher_yates(od.Stream(42, "Pi", 0), 4).tolist() == [2, 0, 3, 1]

    def test_block_goldens(self):
        spec = off.OSpec(4, 2, "rbf", 1.0, 0, 42)
        b0 = off.build_block(spec, 0)
        assert b0.b_signs.tolist() == [-1.0, 1.0, -1.0, 1.0]
        assert b0.permutation.tolist() == [2, 0, 3, 1]
        assert b0.g_diag.tolist() == [0.6566604375839233, -0.04258674010634422,
                                      0.2037200927734375, 1.5018609762191772]
        assert b0.c_diag.tolist() == [1.5748388767242432, 0.5051615834236145,
                                      1.2349847555160522, 0.8342806696891785]
        assert off.build_block(spec, 1).g_diag.tolist() == [
            -1.41425621509552, -0.8420379757881165, -0.24285130202770233, -0.7654402852058411]


class TestDetrand:
    def test_streams_bit_exact(self):
        z = load_npz("detrand.npz")
        cases = json.loads(str(z["cases"][0]))
        for k, (seed, label, block) in enumerate(cases):
            assert od.stream_key(seed, label, block) == int(z[f"key{k}"][0])
            np.testing.assert_array_equal(od.Stream(seed, label, block).hashes(64), z[f"hash{k}"])
            np.testing.assert_array_equal(od.Stream(seed, label, block).uniforms(64), z[f"uni{k}"])
            np.testing.assert_array_equal(od.Stream(seed, label, block).signs(64), z[f"sign{k}"])
            s = od.Stream(seed, label, block)
            g = np.concatenate([s.gaussians(5), s.gaussians(60)])
            np.testing.assert_array_equal(g, z[f"gauss{k}"])
            assert s.counter == int(z[f"gauss_counter{k}"][0])

    def test_permutations_bit_exact(self):
        z = load_npz("detrand.npz")
        np.testing.assert_array_equal(od.fisher_yates(od.Stream(3, "Pi", 1), 1000), z["perm_n1000_s3"])
        for ep in (0, 1):
            np.testing.assert_array_equal(olm.epoch_order(0, ep, 60000), z[f"shuffle60000_e{ep}"])

    def test_unit_ball(self):
        z = load_npz("detrand.npz")
        np.testing.assert_array_equal(od.unit_ball(od.Stream(11, "ball", 0), 5, 6, 1.0), z["ball_n6"])
        np.testing.assert_array_equal(od.unit_ball(od.Stream(11, "ball", 1), 4, 3, 2.0), z["ball_n3"])


def _spec_from_json(js):
    c = json.loads(js)
    return off.OSpec(c["d"], c["E"], c["kind"], c["sigma"], c["t"], c["seed"])


class TestBlocks:
    def _check(self, spec, z, prefix=""):
        blocks = off.build_blocks(spec)
        np.testing.assert_array_equal(np.stack([b.b_signs for b in blocks]), z[prefix + "b"])
        np.testing.assert_array_equal(np.stack([b.permutation for b in blocks]), z[prefix + "perm"])
        np.testing.assert_array_equal(np.stack([b.g_diag for b in blocks]), z[prefix + "g"])
        np.testing.assert_array_equal(np.stack([b.c_diag for b in blocks]), z[prefix + "c"])
        return blocks

    @pytest.mark.parametrize("name", ["rbf_d4", "matern_d13", "rbf_d1", "matern_d1", "rbf_d100",
                                      "rbf_d1000", "matern_d700", "matern_d2048"])
    def test_small_specs(self, name):
        z = load_npz("blocks_small.npz")
        spec = _spec_from_json(str(z[f"{name}.spec"][0]))
        blocks = self._check(spec, z, name + ".")
        x = np.random.default_rng(spec.seed).standard_normal((5, spec.input_dim)).astype(np.float32)
        np.testing.assert_array_equal(off.apply_zhat_batch(spec, blocks, x), z[f"{name}.z"])
        np.testing.assert_array_equal(off.feature_map_batch(spec, blocks, x), z[f"{name}.feat"])

    def test_config0(self):
        z = load_npz("c0.npz")
        meta = json.loads(str(z["meta"][0]))
        spec = off.OSpec(meta["d"], meta["E"], meta["kind"], meta["sigma"], meta["t"], meta["seed"])
        blocks = self._check(spec, z)
        x = synthetic.image_rows(meta["m"], meta["d"], meta["xseed"])[z["rows"]]
        got = off.apply_zhat_batch(spec, blocks, x)
        np.testing.assert_array_equal(got, z["z"])
        # BLAS-independent restatement: bit-exact as well
        np.testing.assert_array_equal(off.apply_zhat_batch(spec, blocks, x, wht="sequential"), z["z"])
        feat = off.feature_map_batch(spec, blocks, x)[:, z["feat_cols"]]
        np.testing.assert_array_equal(feat, z["feat"])

    def test_config2_factors(self):
        z = load_npz("c2.npz")
        meta = json.loads(str(z["meta"][0]))
        spec = off.OSpec(meta["d"], meta["E"], meta["kind"], meta["sigma"], meta["t"], meta["seed"])
        # Matern calibration of 2 of 16 blocks (the full set takes ~45 s on CPU)
        for e in (0, 15):
            blk = off.build_block(spec, e)
            np.testing.assert_array_equal(blk.b_signs, z["b"][e])
            np.testing.assert_array_equal(blk.permutation, z["perm"][e])
            np.testing.assert_array_equal(blk.g_diag, z["g"][e])
            np.testing.assert_array_equal(blk.c_diag, z["c"][e])

    def test_config4_partial(self):
        z = load_npz("c4_blocks.npz")
        meta = json.loads(str(z["meta"][0]))
        spec = off.OSpec(meta["d"], meta["E"], meta["kind"], meta["sigma"], meta["t"], meta["seed"])
        n = spec.n
        for e in (0, 31):
            np.testing.assert_array_equal(od.Stream(spec.seed, "B", e).signs(n).astype(np.float32),
                                          z[f"b{e}"])
            np.testing.assert_array_equal(od.fisher_yates(od.Stream(spec.seed, "Pi", e), n),
                                          z[f"perm{e}"])
            np.testing.assert_array_equal(
                od.Stream(spec.seed, "G", e).gaussians(n).astype(np.float32), z[f"g{e}"])
        entries = np.array([0, 1, 777, 16383])
        np.testing.assert_array_equal(off.rbf_c_entries(spec, 0, entries), z["c0"][entries])


class TestWht:
    def test_reference_bits(self):
        z = load_npz("wht.npz")
        for k in range(0, 15):
            x = synthetic.gaussian_rows(3, 1 << k, seed=100 + k)
            np.testing.assert_array_equal(ow.wht_fast_batch(x.copy()), z[f"n{k}"])
            if k >= 1:
                np.testing.assert_array_equal(ow.wht_sequential(x), z[f"n{k}"])

    def test_large_sizes(self):
        z = load_npz("wht.npz")
        for k in (15, 16, 18, 20):
            x = synthetic.gaussian_rows(1, 1 << k, seed=100 + k)
            y = ow.wht_sequential(x)
            np.testing.assert_array_equal(y[0, :2048], z[f"n{k}.head"])
            np.testing.assert_array_equal(y[0, -2048:], z[f"n{k}.tail"])

    def test_naive_oracle(self):
        assert ow.wht_naive(np.array([1.0, 2.0, 3.0, 4.0])).tolist() == [10.0, -2.0, -4.0, 0.0]
        rng = np.random.default_rng(0)
        for k in range(0, 11):
            v = rng.standard_normal((2, 1 << k))
            np.testing.assert_allclose(ow.wht_butterfly_f64(v), ow.wht_naive(v.T).T, rtol=1e-10,
                                       atol=1e-10)


class TestLinearModel:
    def test_train_history_tiny(self):
        g = load_json("train_tiny.json")
        c = g["config"]
        x, y = synthetic.class_images(c["m"], c["d"], 10, seed=c["data_seed"],
                                      sample_seed=c["train_sample_seed"], noise=c["noise"])
        xt, yt = synthetic.class_images(c["m_test"], c["d"], 10, seed=c["data_seed"],
                                        sample_seed=c["test_sample_seed"], noise=c["noise"])
        spec = off.OSpec(c["d"], c["E"], "rbf", c["sigma"], 0, c["seed"])
        _, b, hist = olm.train(spec, x, y, xt, yt, 10, c["lr"], c["batch"], c["epochs"],
                               shuffle_seed=c["shuffle_seed"])
        for (e, l, a), (e2, l2, a2) in zip(hist, g["history"]):
            assert e == e2 and a == a2
            assert abs(l - l2) <= 1e-12 * abs(l2)
        np.testing.assert_allclose(b, g["b"], rtol=1e-10, atol=1e-12)

    def test_gradients_match_finite_differences(self):
        rng = np.random.default_rng(1)
        x = rng.standard_normal((7, 5))
        y = rng.integers(0, 3, 7)
        w = rng.standard_normal((3, 5)) * 0.1
        b = rng.standard_normal(3) * 0.1
        dw, db = olm.gradients(w, b, x, y, 0.01)
        eps = 1e-6
        for i in range(3):
            for j in range(5):
                wp = w.copy(); wp[i, j] += eps
                wm = w.copy(); wm[i, j] -= eps
                fd = (olm.loss(wp, b, x, y, 0.01) - olm.loss(wm, b, x, y, 0.01)) / (2 * eps)
                assert abs(fd - dw[i, j]) < 1e-5
