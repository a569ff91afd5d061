import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")
REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden():
    def load(name):
        return np.load(os.path.join(GOLDEN, name), allow_pickle=False)
    return load


def has_gpu():
    try:
        from paper_2402_13171_b200 import _lib
        return _lib.load().lbw_device_count() > 0
    except Exception:
        return False


@pytest.fixture(scope="session")
def gpu():
    """Skip-free guard: -m gpu tests must run on a GPU box; fail loudly."""
    from paper_2402_13171_b200 import _lib
    _lib.require_gpu()
    return _lib.load()


@pytest.fixture(scope="session")
def reference_lbwind():
    """The read-only reference package, importable only in the build
    container (used to cross-check the oracle beyond the golden vectors)."""
    if not os.path.isdir(REFERENCE_SRC):
        pytest.skip("reference source tree not present (GPU box)")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_lbw_tests")
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    import lbwind
    return lbwind
