import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

REFERENCE_SRC = os.environ.get("DMLENS_SRC", "/root/reference/pkg/src")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs through libb2l.so")
    config.addinivalue_line("markers", "slow: long-running parity sweep")


def have_reference() -> bool:
    return os.path.isdir(os.path.join(REFERENCE_SRC, "dmlens"))


def import_reference():
    """The unmodified reference (build container only; absent on the GPU box)."""
    if not have_reference():
        pytest.skip("reference checkout not present (GPU box): golden fixtures cover parity")
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    import dmlens  # noqa: F401
    return dmlens


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test scheduled without a CUDA device")
    return torch.device("cuda:0")
