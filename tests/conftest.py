import os
import sys

# The oracle's small dense algebra gains nothing from many BLAS threads, and OpenBLAS's
# spinning workers stall badly when the host is shared (e.g. with a long oracle run):
# cap them before numpy is imported (an explicit setting in the environment wins).
for _v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, "4")

import numpy as np  # noqa: E402
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu on the GPU box)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def rng():
    return np.random.default_rng(12345)
