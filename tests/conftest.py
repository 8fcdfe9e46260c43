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
def orc():
    import oracle
    oracle.build()
    return oracle.Oracle()


@pytest.fixture(scope="session")
def ref():
    import oracle
    if not oracle.reference_available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return oracle.Reference()


@pytest.fixture(scope="session")
def fmmlib():
    import paper_1203_0889_b200 as fb
    fb._capi.load()
    return fb


def sorted_pairs(pairs: np.ndarray) -> np.ndarray:
    """Canonical multiset form of (target, source) pairs."""
    p = np.ascontiguousarray(pairs, dtype=np.int64).reshape(-1, 2)
    keys = (p[:, 0] << 32) | p[:, 1]
    return np.sort(keys)
