import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running (large sizes)")


@pytest.fixture
def rng():
    # same seed as the reference's fixture (pkg/tests/conftest.py:7-9)
    return np.random.default_rng(1234)


@pytest.fixture(scope="session")
def golden_index():
    with open(os.path.join(GOLDEN, "golden_index.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def bitmask_golden():
    return np.load(os.path.join(GOLDEN, "bitmask_golden.npz"))


@pytest.fixture(scope="session")
def quant_golden():
    return np.load(os.path.join(GOLDEN, "quant_golden.npz"))


@pytest.fixture(scope="session")
def checkpoint_golden():
    return np.load(os.path.join(GOLDEN, "checkpoint_golden.npz"))


def cuda_ok():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def dev():
    if not cuda_ok():
        pytest.skip("no CUDA device")
    import torch
    return torch.device("cuda:0")
