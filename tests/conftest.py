import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(REPO, "tests", "golden")
if REPO not in sys.path:
    sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libgs_b200.so")
    config.addinivalue_line("markers", "slow: long-running (still part of the default suites)")


def cases(npz_name):
    """{case: {field: array}} from a golden npz written by tests/golden/make_golden.py."""
    z = np.load(os.path.join(GOLDEN, npz_name))
    out = {}
    for key in z.files:
        name, fld = key.split("__", 1)
        out.setdefault(name, {})[fld] = z[key]
    return out


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1510_03816_b200._native as N

    N.load()
    return torch
