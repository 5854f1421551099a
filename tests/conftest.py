import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)


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
