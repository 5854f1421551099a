"""Experiment: per-step wall time of the end-to-end (host in, host out) path
of a bench workload, with the session counters that move in each step —
looking for outlier steps.  usage: e2e_probe.py [workload] [steps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_1901_03771_b200 as gp  # noqa: E402
from paper_1901_03771_b200 import runtime  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "mlp"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
w = bench.WORKLOADS[name]
n = bench.global_rows(name)
rt = runtime.get()
sess = gp.default_session()
host = bench.host_inputs(name, 0, n)
src = []
for x in host:
    p = rt.pinned_empty(x.shape, x.dtype)
    p[...] = x
    src.append(p)
outs0 = w["program"](gp, [gp.asarray(x) for x in src])
dst = [rt.pinned_empty(o.shape, o.dtype) for o in outs0]
del outs0
keys = ("kernels_executed", "library_calls", "streamed_chunks", "compile_ms", "h2d_bytes", "d2h_bytes")
for it in range(steps):
    s0 = {k: getattr(sess.stats, k) for k in keys}
    t0 = time.perf_counter()
    outs = w["program"](gp, [gp.asarray(x) for x in src])
    gp.materialize(*outs, out=dst)
    rt.sync()
    dt = time.perf_counter() - t0
    d = {k: round(getattr(sess.stats, k) - s0[k], 1) for k in keys}
    print(f"step {it:2d} {dt * 1e3:8.2f} ms {d}", flush=True)
    del outs
