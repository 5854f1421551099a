"""Drop-in module name from the paper: ``import grumpy as np``.

Re-exports the B200 implementation in ``paper_1901_03771_b200``.
"""
from paper_1901_03771_b200 import *  # noqa: F401,F403
from paper_1901_03771_b200 import distributed, errors, workloads  # noqa: F401
