import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

# the package maps its shim (and with it cuBLAS 12.9, whose BF16x9 FP32
# emulation the np.dot boundary uses) before any test module imports PyTorch,
# whose wheel carries an older libcublas.so.12
import paper_1901_03771_b200  # noqa: E402,F401


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture
def sess():
    """A fresh default session per test (GPU tests)."""
    import paper_1901_03771_b200 as gp
    s = gp.Session()
    old = gp.set_default_session(s)
    yield s
    gp.set_default_session(old)
