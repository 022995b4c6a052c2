import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running")


def _has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


HAS_GPU = _has_gpu()


@pytest.fixture(scope="session")
def ctx():
    if not HAS_GPU:
        pytest.skip("no GPU")
    import paper_2604_08584_b200 as cs
    c = cs.Context(0)
    yield c
    c.close()


@pytest.fixture(scope="session")
def ref_ok():
    from oracle.bindings import ref_available
    if not ref_available():
        pytest.skip("oracle/_ref not built")
    return True
