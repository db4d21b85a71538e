import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

# the reference's own python tests, staged by tests/cpp/build_reftests.py, run
# in their own process through the `graphfuse` alias (test_reference_suites.py)
collect_ignore_glob = ["cpp/_reftests/*", "alias/*"]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def cuda():
    import torch

    assert torch.cuda.is_available(), "GPU test run without a CUDA device"
    from paper_2411_16127_b200 import _capi

    assert _capi.lib().gf_device_ok() == 1, "libgraphfuse_cuda cannot launch on this device"
    return torch.device("cuda:0")


def rel_err(a, b) -> float:
    """Reference parity metric |a-b| / max(|a|,|b|,1) (bench.cpp:106-115)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if a.size == 0:
        return 0.0
    return float(np.max(np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), 1.0)))
