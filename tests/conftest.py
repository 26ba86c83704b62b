import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def golden():
    with np.load(os.path.join(GOLDEN_DIR, "golden_v1.npz")) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture
def rng():
    return np.random.default_rng(1234)



@pytest.fixture(scope="session")
def golden_bf16():
    with np.load(os.path.join(GOLDEN_DIR, "golden_bf16.npz")) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def golden_reads():
    with np.load(os.path.join(GOLDEN_DIR, "golden_reads.npz")) as z:
        return {k: z[k] for k in z.files}
