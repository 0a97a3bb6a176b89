import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def golden():
    return np.load(os.path.join(ROOT, "tests", "golden", "ref_vectors.npz"))


@pytest.fixture(scope="session")
def O():
    from oracle import oracle

    oracle.lib()
    return oracle


def rel(a, b):
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


@pytest.fixture(autouse=True, scope="module")
def _trim_library_device_cache():
    """The library keeps large device blocks between refit sessions; hand
    them back after each module so torch allocations in later modules (and
    their memory-size assumptions) see a clean device."""
    yield
    mod = sys.modules.get("paper_1907_05884_b200._lib")
    if mod is not None and getattr(mod, "_LIB", None) is not None:
        mod.trim_device_cache(-1)
