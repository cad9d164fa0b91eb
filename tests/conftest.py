import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def _has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


@pytest.fixture(scope="session", autouse=True)
def _native_built():
    """Build the product library and the CPU oracle in-tree (no-ops when fresh)."""
    from paper_1901_06363_b200 import build
    build.build()
    from oracle import oracle_py
    oracle_py.build(ref=True)
    yield


@pytest.fixture(scope="session")
def docker():
    if not _has_gpu():
        pytest.skip("no CUDA device")
    from paper_1901_06363_b200 import Docker
    d = Docker(int(os.environ.get("GD_TEST_DEVICE", "0")))
    yield d
    d.close()
