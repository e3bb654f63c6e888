import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu on the GPU box)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def port():
    from oracle.oracle import Oracle
    return Oracle("port")


@pytest.fixture(scope="session")
def ref():
    """The reference compiled from /root/reference (oracle/_ref).  Built here;
    the prebuilt .so travels to the GPU box."""
    from oracle.oracle import REF_SO, Oracle
    if not REF_SO.exists() and not Path("/root/reference/proj").exists():
        pytest.skip("oracle/_ref not built and /root/reference absent")
    return Oracle("reference")


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a CUDA device")
    return torch.device("cuda:0")
