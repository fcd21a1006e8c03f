import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libvxb.so")
    config.addinivalue_line("markers", "slow: full-size parity against the host oracle (minutes)")


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


@pytest.fixture(scope="session")
def golden_ops():
    return dict(np.load(os.path.join(GOLDEN, "ops.npz")))


@pytest.fixture(scope="session")
def golden_nets():
    return dict(np.load(os.path.join(GOLDEN, "nets.npz")))


def cuda_ready():
    try:
        import torch
        from paper_1903_07525_b200 import _lib
        return torch.cuda.is_available() and _lib.library_available()
    except Exception:
        return False
