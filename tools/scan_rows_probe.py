"""Experiment: scans along the last axis of a matrix with few long lines —
the segmented TMA look-back scan against the warp-per-16-lines kernel — and
a 1-D scan whose length is not a multiple of a 128-byte line (TMA kernel with
a tail).
Run under ncu (--metrics gpu__time_duration.sum) for kernel times; prints the
kernel label per case.  usage: scan_rows_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1901_03771_b200 as gp  # noqa: E402
from paper_1901_03771_b200 import codegen, codegen_scan  # noqa: E402

sess = gp.default_session()
for shape in [(1024, 262144), (64, 1 << 22), (8192, 32768), (1024, 262147)]:
    x = gp.asarray(np.random.default_rng(1).standard_normal(shape, dtype=np.float32))
    for mode in ("tma", "rows"):
        codegen_scan.ROWS_T_MIN_LINES = 148 * 16 * 4 if mode == "tma" else 0
        codegen._GEN_CACHE.clear()
        sess._plan_cache.clear()
        for _ in range(3):
            y = gp.cumsum(x * 0.5 + 1.0, axis=1)
            gp.force(y)
        print(shape, mode, sess.executor.last_steps[-1].cache["ks"].meta.get("label"), flush=True)
        del y
x = gp.asarray(np.random.default_rng(2).standard_normal((1 << 28) + 7, dtype=np.float32))
for _ in range(3):
    y = gp.cumsum(x * 0.5 + 1.0)
    gp.force(y)
print("2^28+7", sess.executor.last_steps[-1].cache["ks"].meta.get("label"), flush=True)
x2 = gp.asarray(np.random.default_rng(3).standard_normal((16384, 16384), dtype=np.float32))
for _ in range(3):
    y = gp.cumsum(x2 * 0.5 + 1.0)          # flattened (axis=None) scan of a matrix
    gp.force(y)
print("16384x16384 flat", sess.executor.last_steps[-1].cache["ks"].meta.get("label"), flush=True)

