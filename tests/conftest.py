"""Shared fixtures.  `-m gpu` tests need a B200 and the built library;
everything else runs on CPU (oracle vs golden vectors, host logic, ABI
symbols, gloo multi-process plumbing)."""

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libmckernel_b200.so")
    config.addinivalue_line("markers", "slow: long-running")


def load_npz(name):
    path = GOLDEN / name
    if not path.exists():
        pytest.skip(f"golden fixture {name} missing")
    return np.load(path, allow_pickle=False)


def load_json(name):
    path = GOLDEN / name
    if not path.exists():
        pytest.skip(f"golden fixture {name} missing")
    return json.loads(path.read_text())


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1702_08159_b200 import _native
    _native.lib()
    return torch
