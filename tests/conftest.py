import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libxpgb.so")
    config.addinivalue_line("markers", "slow: long-running (large shapes)")


@pytest.fixture(scope="session")
def golden():
    import json

    import numpy as np

    arrays = np.load(os.path.join(GOLDEN, "golden_v1.npz"))
    with open(os.path.join(GOLDEN, "golden_v1.json")) as fh:
        meta = json.load(fh)
    return arrays, meta
