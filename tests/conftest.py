import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C ABI")
    config.addinivalue_line("markers", "slow: long-running")


def gpu_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def oracle_port():
    import pyoracle
    return pyoracle.load("port")


@pytest.fixture(scope="session")
def oracle_ref():
    import pyoracle
    if not pyoracle.available("reference"):
        pytest.skip("oracle/_ref not built (reference tree absent)")
    return pyoracle.load("reference")
