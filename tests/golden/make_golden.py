"""Generate the golden fixtures by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src:/root/repo python tests/golden/make_golden.py [--only NAME ...]

Every array below is produced by the reference's own public functions
(``mckernel`` 0.1.0); the tests compare the oracle restatement (CPU) and the
CUDA library (GPU) against these files.  Inputs are regenerated in the tests
from the seeds recorded here (paper_1702_08159_b200.synthetic), so only
outputs are stored.  The GPU box never needs /root/reference.
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)
HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))

import mckernel  # noqa: E402  (the reference)
from mckernel import detrand as rd  # noqa: E402
from mckernel import fastfood as rf  # noqa: E402
from mckernel import wht as rw  # noqa: E402
from mckernel import linear_model as rl  # noqa: E402
from mckernel.dataio import Dataset  # noqa: E402

from paper_1702_08159_b200 import synthetic  # noqa: E402

C0 = dict(d=784, E=8, kind="rbf", sigma=1.0, t=0, seed=1234, m=1000, xseed=1234)
C2 = dict(d=784, E=16, kind="matern", sigma=2.0, t=40, seed=42, m=60000, xseed=42)
C4 = dict(d=16384, E=32, kind="rbf", sigma=4.0, t=0, seed=4, xseed=7)
C3 = dict(d=784, E=8, sigma=1.0, seed=1234, m=60000, m_test=10000, data_seed=1234,
          test_sample_seed=99, noise=0.1, lr=0.01, batch=1000, epochs=20, shuffle_seed=0)
TINY = dict(d=20, E=2, sigma=1.0, seed=5, m=300, m_test=100, data_seed=8, train_sample_seed=9,
            test_sample_seed=10, noise=0.2, lr=0.05, batch=64, epochs=2, shuffle_seed=3)
C3H = dict(d=784, E=8, sigma=1.0, seed=1234, m=6000, m_test=2000, data_seed=1,
           train_sample_seed=2, test_sample_seed=3, noise=0.25, lr=0.01, batch=100, epochs=2,
           shuffle_seed=0)


def spec_of(c):
    k = rf.RBF(c["sigma"]) if c["kind"] == "rbf" else rf.RBFMatern(c["sigma"], c["t"])
    return rf.FeatureMapSpec(c["d"], c["E"], k, c["seed"])


def blocks_arrays(blocks):
    return dict(
        b=np.stack([b.b_signs for b in blocks]).astype(np.int8),
        perm=np.stack([b.permutation for b in blocks]).astype(np.int32),
        g=np.stack([b.g_diag for b in blocks]),
        c=np.stack([b.c_diag for b in blocks]),
    )


def gen_detrand():
    out = {}
    cases = [(42, "B", 0), (42, "G", 0), (43, "B", 0), (7, "x", 0), (1234, "C", 5),
             (0, "shuffle", 3), (2**64 - 1, "Pi", 2**40)]
    for k, (seed, label, block) in enumerate(cases):
        s = rd.RandomStream(seed, label, block)
        out[f"key{k}"] = np.array([rd.stream_key(seed, label, block)], dtype=np.uint64)
        out[f"hash{k}"] = s._hash_block(64)
        s = rd.RandomStream(seed, label, block)
        out[f"uni{k}"] = s.uniform01_array(64)
        s = rd.RandomStream(seed, label, block)
        out[f"sign{k}"] = s.sign_array(64)
        s = rd.RandomStream(seed, label, block)
        g1 = s.gaussian_array(5)          # odd count -> cached variate
        g2 = s.gaussian_array(60)
        out[f"gauss{k}"] = np.concatenate([g1, g2])
        out[f"gauss_counter{k}"] = np.array([s.counter])
    out["cases"] = np.array([json.dumps(cases)])
    out["perm_n4_s42"] = rd.fisher_yates_permutation(rd.RandomStream(42, "Pi", 0), 4)
    out["perm_n1000_s3"] = rd.fisher_yates_permutation(rd.RandomStream(3, "Pi", 1), 1000)
    for ep in (0, 1):
        out[f"shuffle60000_e{ep}"] = rd.fisher_yates_permutation(
            rd.RandomStream(0, "shuffle", ep), 60000).astype(np.int32)
    s = rd.RandomStream(11, "ball", 0)
    out["ball_n6"] = rd.unit_ball_batch(s, 5, 6, 1.0)
    s = rd.RandomStream(11, "ball", 1)
    out["ball_n3"] = rd.unit_ball_batch(s, 4, 3, 2.0)
    np.savez_compressed(HERE / "detrand.npz", **out)


def gen_blocks_small():
    out = {}
    small = {
        "rbf_d4": dict(d=4, E=2, kind="rbf", sigma=1.0, t=0, seed=42),
        "matern_d13": dict(d=13, E=3, kind="matern", sigma=1.0, t=2, seed=5),
        "rbf_d1": dict(d=1, E=2, kind="rbf", sigma=1.0, t=0, seed=3),
        "matern_d1": dict(d=1, E=2, kind="matern", sigma=1.5, t=3, seed=3),
        "rbf_d100": dict(d=100, E=2, kind="rbf", sigma=0.7, t=0, seed=9),
        "rbf_d1000": dict(d=1000, E=2, kind="rbf", sigma=1.3, t=0, seed=10),
        "matern_d700": dict(d=700, E=2, kind="matern", sigma=1.0, t=5, seed=11),
        "matern_d2048": dict(d=2048, E=1, kind="matern", sigma=3.0, t=2, seed=12),
    }
    for name, c in small.items():
        blocks = rf.build_blocks(spec_of(c))
        for k, v in blocks_arrays(blocks).items():
            out[f"{name}.{k}"] = v
        out[f"{name}.spec"] = np.array([json.dumps(c)])
        # z / features for a few inputs of this spec
        x = np.random.default_rng(c["seed"]).standard_normal((5, c["d"])).astype(np.float32)
        out[f"{name}.z"] = rf.apply_zhat_batch(spec_of(c), blocks, x)
        out[f"{name}.feat"] = rf.feature_map_batch(spec_of(c), blocks, x)
    np.savez_compressed(HERE / "blocks_small.npz", **out)


def gen_config(name, c, rows):
    spec = spec_of(c)
    t0 = time.time()
    blocks = rf.build_blocks(spec)
    build_s = time.time() - t0
    out = blocks_arrays(blocks)
    x = synthetic.image_rows(c["m"], c["d"], c["xseed"])[rows]
    t0 = time.time()
    out["z"] = rf.apply_zhat_batch(spec, blocks, x)
    out["feat"] = rf.feature_map_batch(spec, blocks, x)[:, ::7]   # every 7th feature
    out["feat_cols"] = np.arange(0, 2 * spec.padded_dim * c["E"], 7)
    out["raw"] = rf.feature_map_batch(spec, blocks, x[:2], normalize=False)
    out["rows"] = np.asarray(rows)
    out["meta"] = np.array([json.dumps(dict(c, build_s=build_s))])
    np.savez_compressed(HERE / f"{name}.npz", **out)


def gen_c4():
    """Config 4 spec (n = 16384): full block 0 and block 31 (30 s / 8.5 GB each)."""
    spec = spec_of(C4)
    out = {}
    for e in (0, 31):
        t0 = time.time()
        b = rf.build_block(spec, e)
        out[f"b{e}"] = b.b_signs.astype(np.int8)
        out[f"perm{e}"] = b.permutation.astype(np.int32)
        out[f"g{e}"] = b.g_diag
        out[f"c{e}"] = b.c_diag
        out[f"build_s{e}"] = np.array([time.time() - t0])
    out["meta"] = np.array([json.dumps(C4)])
    np.savez_compressed(HERE / "c4_blocks.npz", **out)


def gen_wht():
    out = {}
    for k in range(0, 15):
        n = 1 << k
        x = synthetic.gaussian_rows(3, n, seed=100 + k)
        out[f"n{k}"] = rw.wht_fast_batch(x.copy())
    for k in (15, 16, 18, 20):
        n = 1 << k
        x = synthetic.gaussian_rows(1, n, seed=100 + k)
        y = rw.wht_fast_batch(x.copy())
        out[f"n{k}.head"] = y[0, :2048]
        out[f"n{k}.tail"] = y[0, -2048:]
        out[f"n{k}.sumsq"] = np.array([float((y.astype(np.float64) ** 2).sum())])
    np.savez_compressed(HERE / "wht.npz", **out)


def gen_train(name, c):
    if name == "train_c3":
        x, y = synthetic.class_images(c["m"], c["d"], 10, seed=c["data_seed"], noise=c["noise"])
        xt, yt = synthetic.class_images(c["m_test"], c["d"], 10, seed=c["data_seed"],
                                        sample_seed=c["test_sample_seed"], noise=c["noise"])
    else:
        x, y = synthetic.class_images(c["m"], c["d"], 10, seed=c["data_seed"],
                                      sample_seed=c["train_sample_seed"], noise=c["noise"])
        xt, yt = synthetic.class_images(c["m_test"], c["d"], 10, seed=c["data_seed"],
                                        sample_seed=c["test_sample_seed"], noise=c["noise"])
    spec = rf.FeatureMapSpec(c["d"], c["E"], rf.RBF(c["sigma"]), c["seed"])
    cfg = rl.TrainConfig(c["lr"], c["batch"], c["epochs"], shuffle_seed=c["shuffle_seed"])
    t0 = time.time()
    model, met = rl.train(spec, Dataset(x, y, 10), Dataset(xt, yt, 10), cfg)
    wall = time.time() - t0
    hist = [[r.epoch, r.train_loss, r.test_acc] for r in met.records]
    (HERE / f"{name}.json").write_text(json.dumps(
        dict(config=c, history=hist, wall_s=wall,
             w_norm=float(np.sqrt((model.w ** 2).sum())), b=model.b.tolist()), indent=1))


def gen_formats():
    """Byte-level fixtures of the reference's on-disk formats."""
    from mckernel import dataio as rdio
    spec = rf.FeatureMapSpec(5, 2, rf.RBFMatern(1.5, 3), 77)
    m = rl.SoftmaxModel(np.arange(3 * 20, dtype=np.float64).reshape(3, 20) / 7.0,
                        np.array([0.5, -1.25, 3.0]))
    rl.save_model(HERE / "model_small.mckmodl", m, spec)
    rdio.write_matrix(HERE / "matrix_small.mckmat",
                      (np.arange(12, dtype=np.float32).reshape(3, 4) - 5) / 3)


JOBS = {
    "detrand": gen_detrand,
    "blocks_small": gen_blocks_small,
    "c0": lambda: gen_config("c0", C0, list(range(8)) + list(range(992, 1000))),
    "c2": lambda: gen_config("c2", C2, list(range(4)) + [30000, 59999]),
    "c4": gen_c4,
    "wht": gen_wht,
    "train_c3h": lambda: gen_train("train_c3h", C3H),
    "train_c3": lambda: gen_train("train_c3", C3),
    "train_tiny": lambda: gen_train("train_tiny", TINY),
    "formats": gen_formats,
}

if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", nargs="*", default=list(JOBS))
    args = ap.parse_args()
    for name in args.only:
        t0 = time.time()
        JOBS[name]()
        print(f"{name}: {time.time() - t0:.1f}s", flush=True)

