import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_1901_03771_b200 as gp
from paper_1901_03771_b200 import codegen, codegen_scan
sess = gp.default_session()
for shape in [(16384, 16384), (32768, 8192), (65536, 4096)]:
    x = gp.asarray(np.random.default_rng(1).standard_normal(shape, dtype=np.float32))
    for thr in (148 * 16 * 4, 1 << 30):
        codegen_scan.ROWS_T_MIN_LINES = thr
        codegen._GEN_CACHE.clear(); sess._plan_cache.clear()
        for _ in range(3):
            gp.force(gp.cumsum(x * 0.5 + 1.0, axis=1))
        print(shape, thr, sess.executor.last_steps[-1].cache["ks"].meta.get("label"), flush=True)
