import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libdfno.so")


@pytest.fixture(scope="session")
def golden_dir():
    return GOLDEN


def gpu_ready() -> bool:
    try:
        import torch

        from paper_2211_12709_b200 import _lib
    except Exception:
        return False
    return torch.cuda.is_available() and _lib.LIB_PATH.exists()


def pytest_collection_modifyitems(config, items):
    # GPU tests must FAIL (not skip) on a GPU box without the library; they
    # only skip on a host with no CUDA device at all.
    import torch

    if torch.cuda.is_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device on this host")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)
