import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).resolve().parent))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) device")
    config.addinivalue_line("markers", "slow: long-running parity case")


def _have_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Build the product library and the oracle when missing (CPU-side check)."""
    from paper_2109_00485_b200 import build as b
    if not b.LIB.exists():
        b.build_lib()
    import oracle_lib
    if not oracle_lib.ORC_PATH.exists():
        oracle_lib.build()
    yield


@pytest.fixture(scope="session")
def ctx():
    if not _have_gpu():
        pytest.skip("no CUDA device")
    from paper_2109_00485_b200 import abi
    c = abi.Context(0)
    yield c
    c.close()
