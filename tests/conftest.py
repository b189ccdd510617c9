import ctypes
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

ORACLE_SO = os.path.join(ROOT, "oracle", "_ref", "libswapsched_ref.so")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


@pytest.fixture(scope="session")
def oracle():
    """The compiled reference planner (oracle/_ref); test infrastructure only."""
    if not os.path.exists(ORACLE_SO):
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    from paper_1901_06773_b200 import _native
    lib = ctypes.CDLL(ORACLE_SO)
    _native.declare_planner_symbols(lib, "oracle_")
    return lib


@pytest.fixture(scope="session")
def cuda_dev():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")
