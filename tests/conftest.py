import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: larger sizes")


def _has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def orc():
    import oracle
    return oracle.restatement()


@pytest.fixture(scope="session")
def ref():
    import oracle
    r = oracle.reference()
    if r is None:
        pytest.skip("compiled reference (oracle/_ref) not available here")
    return r


@pytest.fixture(scope="session")
def gpulib():
    import os
    import paper_2311_14616_b200 as p
    from paper_2311_14616_b200 import _lib
    # the in-tree library ships with the snapshot (its objects do not):
    # build only when it is missing
    if not os.path.exists(_lib.LIB_PATH):
        p.build()
    return p.lib()
