import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def golden_dir():
    return ROOT / "tests" / "golden"


@pytest.fixture(scope="module", autouse=True)
def _release_device_memory():
    """After each module on a GPU box: return cached device memory (torch's
    allocator and the library's stream-ordered pool), so later tests that
    spawn processes sharing the GPU find it free."""
    yield
    import torch
    if torch.cuda.is_available() and torch.cuda.is_initialized():
        from paper_2412_11639_b200 import _capi as capi
        torch.cuda.empty_cache()
        capi.check(capi.lib().spk_release_memory())
