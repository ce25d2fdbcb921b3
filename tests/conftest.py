import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path through the C-ABI)")


def _has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


HAS_GPU = _has_gpu()


@pytest.fixture(scope="session")
def built():
    """Build libffca.so and the oracle in-tree (no-op when up to date)."""
    from paper_2101_08563_b200 import build
    build.build_all()
    return True


@pytest.fixture(scope="session")
def gpu(built):
    if not HAS_GPU:
        pytest.fail("gpu-marked test run without a visible CUDA device")
    from paper_2101_08563_b200 import _lib
    return _lib.context(0)
