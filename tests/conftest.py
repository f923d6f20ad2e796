import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an sm_100 GPU and the built libmagfd_b200.so")
    config.addinivalue_line("markers", "slow: long-running (minutes)")


def _gpu_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _gpu_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session", autouse=True)
def _built_oracle():
    """Build the C restatement once (cheap); oracle/_ref is built by __graft_entry__.build()."""
    from oracle import oracle as O
    if not all(os.path.exists(p) for p in O.PORT_SO.values()):
        O.build(ref=False)
    yield
