import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: full-size BASELINE shapes")


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN, allow_pickle=False)


@pytest.fixture(scope="session")
def coracle():
    from oracle.oracle import c_oracle
    return c_oracle()


@pytest.fixture(scope="session")
def reforacle():
    from oracle.oracle import ref_available, ref_oracle
    if not ref_available():
        pytest.skip("oracle/_ref not built (reference tree absent)")
    return ref_oracle()


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a CUDA device")
    from paper_2504_19449_b200 import lib
    lib()  # the native library must load: there is no fallback
    return torch.device("cuda:0")
