import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run under gpurun)")
    config.addinivalue_line("markers", "slow: full-size parity (seconds to minutes)")


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


HAS_GPU = _has_gpu()


def pytest_collection_modifyitems(config, items):
    if HAS_GPU:
        return
    skip = pytest.mark.skip(reason="no GPU in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def ref():
    """The unmodified reference (oracle/_ref/_fastnn_ref), test-only."""
    from oracle import oracle
    return oracle.reference()


@pytest.fixture(scope="session")
def orc():
    """Our C restatement (oracle/_ref/liboracle.so), test-only."""
    from oracle import oracle
    oracle.lib()
    return oracle


@pytest.fixture(scope="session")
def fnl():
    import paper_2503_10017_b200 as f
    return f
