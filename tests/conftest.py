import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

CASES = os.path.join(ROOT, "cases")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def port():
    from oracle import oracle as O
    return O.port()


@pytest.fixture(scope="session")
def ref():
    from oracle import oracle as O
    if not O.have_ref():
        pytest.skip("oracle/_ref not built (reference sources unavailable)")
    return O.ref()


@pytest.fixture(scope="session")
def ctx():
    from paper_1109_3524_b200 import ibm
    return ibm.Context.default()


def case_path(name: str) -> str:
    return os.path.join(CASES, name + ".cfg")


def rel_err(a, b):
    a = np.asarray(a, float)
    b = np.asarray(b, float)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300)) if a.size else 0.0
