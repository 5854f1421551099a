"""ORACLE — test infrastructure.  The BASELINE configs as plain NumPy programs.

The config programs live in ``paper_1901_03771_b200/workloads.py`` written over
a module ``xp`` (the paper's drop-in idea): with ``xp=numpy``
(+ ``scipy.special.erf``, pkg/pyproject.toml:13) each one is the reference's
eager NumPy baseline.  This module loads that
one file *by path*, so the product package's ``__init__`` never runs and the
native shim (``libgrumpy_rt.so``) is never mapped into a process that only
runs the CPU reference (``bench.py --impl reference``) or the checker.
"""

from __future__ import annotations

import importlib.util
import os
import sys

_PATH = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                     "paper_1901_03771_b200", "workloads.py")
_NAME = "_grumpy_numpy_programs"


def load():
    """The workloads module (NumPy-only imports), without the product package."""
    mod = sys.modules.get(_NAME)
    if mod is None:
        spec = importlib.util.spec_from_file_location(_NAME, _PATH)
        mod = importlib.util.module_from_spec(spec)
        sys.modules[_NAME] = mod
        spec.loader.exec_module(mod)
    return mod


def native_shim_mapped() -> bool:
    """True when libgrumpy_rt.so is mapped into this process (Linux)."""
    try:
        with open("/proc/self/maps") as f:
            return any("libgrumpy_rt" in line for line in f)
    except OSError:
        return False
