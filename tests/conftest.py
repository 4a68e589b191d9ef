import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


@pytest.fixture(autouse=True)
def _fresh_counters():
    # exact-equality assertions on the global counters need a clean slate
    from paper_2306_11665_b200 import counting

    counting.reset_multiplication_count()
    counting.reset_allocation_ledger()
    yield


def golden(name):
    return np.load(os.path.join(GOLDEN, name))


def max_rel(got, ref):
    got = np.asarray(got)
    ref = np.asarray(ref)
    scale = np.max(np.abs(ref))
    if scale == 0.0:
        return float(np.max(np.abs(got)))
    return float(np.max(np.abs(got - ref)) / scale)
