"""On-disk formats shared with the reference (no GPU): MCKMAT records and
MCKMODL1 checkpoints, byte-compared with files the reference itself wrote
(tests/golden/make_golden.py, job "formats")."""

import io

import numpy as np

from conftest import GOLDEN
from paper_1702_08159_b200 import dataio, fastfood
from paper_1702_08159_b200.linear_model import read_model_arrays


def test_matrix_record_bytes_match_reference():
    want = (GOLDEN / "matrix_small.mckmat").read_bytes()
    arr = (np.arange(12, dtype=np.float32).reshape(3, 4) - 5) / 3
    buf = io.BytesIO()
    dataio.write_matrix_record(buf, arr)
    assert buf.getvalue() == want
    np.testing.assert_array_equal(dataio.read_matrix(GOLDEN / "matrix_small.mckmat"), arr)


def test_matrix_record_errors(tmp_path):
    import pytest
    with pytest.raises(ValueError, match="unsupported record dtype"):
        dataio.write_matrix_record(io.BytesIO(), np.zeros((2, 2), np.int16))
    with pytest.raises(ValueError, match="2-D"):
        dataio.write_matrix_record(io.BytesIO(), np.zeros(3, np.float32))
    p = tmp_path / "bad"
    p.write_bytes(b"MCKMAT4\n" + (5).to_bytes(4, "little") + (5).to_bytes(4, "little") + b"\0" * 8)
    with pytest.raises(ValueError, match="truncated"):
        dataio.read_matrix(p)


def test_checkpoint_reads_reference_file_and_spec_text_round_trips():
    w, b, spec = read_model_arrays(GOLDEN / "model_small.mckmodl")
    np.testing.assert_array_equal(w, np.arange(60, dtype=np.float64).reshape(3, 20) / 7.0)
    np.testing.assert_array_equal(b, [0.5, -1.25, 3.0])
    assert spec == fastfood.FeatureMapSpec(5, 2, fastfood.RBFMatern(1.5, 3), 77)
    for s in (spec, fastfood.FeatureMapSpec(784, 8, fastfood.RBF(1.0), 1398239763)):
        assert fastfood.spec_from_config(fastfood.spec_to_config(s)) == s


def test_checkpoint_bytes_match_reference(tmp_path):
    # write with our writer (host arrays via a stand-in model object) and compare
    from paper_1702_08159_b200 import linear_model as lm

    class HostModel:
        def numpy(self):
            return (np.arange(60, dtype=np.float64).reshape(3, 20) / 7.0,
                    np.array([0.5, -1.25, 3.0]))

    out = tmp_path / "m.mckmodl"
    lm.save_model(out, HostModel(), fastfood.FeatureMapSpec(5, 2, fastfood.RBFMatern(1.5, 3), 77))
    assert out.read_bytes() == (GOLDEN / "model_small.mckmodl").read_bytes()
