import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU; runs the CUDA path through the C-ABI")


@pytest.fixture(scope="session")
def ws():
    """The product package with libws.so loaded (built in-tree if missing)."""
    import paper_2510_14719_b200 as pkg
    from paper_2510_14719_b200 import build

    if not os.path.exists(build.LIB):
        build.build()
    pkg._lib.load()
    return pkg


@pytest.fixture(scope="session")
def dev():
    import torch

    assert torch.cuda.is_available(), "GPU tests need cuda:0"
    return torch.device("cuda:0")
