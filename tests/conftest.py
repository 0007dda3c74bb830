import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA sm_100 device (B200)")
    config.addinivalue_line("markers", "slow: long-running (full BASELINE sizes)")


@pytest.fixture(scope="session")
def orc():
    from oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle import RefLib
    if not RefLib.available():
        pytest.skip("reference library (oracle/_ref) not built here")
    return RefLib()


@pytest.fixture(scope="session")
def F():
    import paper_2407_10960_b200 as F
    return F


def f16_bits(orc, a: np.ndarray) -> np.ndarray:
    """Round float array to binary16 with the oracle's RNE rule, return u16 bits."""
    a = np.asarray(a, np.float32)
    return a.astype(np.float16).view(np.uint16).reshape(a.shape)


@pytest.fixture(scope="session")
def gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)
    return torch
