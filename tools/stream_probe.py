"""Probe streamed to_external: per-step wall time and a host profile."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1901_03771_b200 as gp  # noqa: E402
from paper_1901_03771_b200 import runtime, workloads as wl  # noqa: E402

w = sys.argv[1] if len(sys.argv) > 1 else "listing1"
rt = runtime.get()
if w == "listing1":
    host = wl.listing1_inputs(n=1 << 24)
    prog = lambda *a: (wl.listing1(gp, *a),)
else:
    host = wl.blackscholes_inputs(n=1 << 28)
    prog = lambda *a: wl.blackscholes(gp, *a)
pin = []
for h in host:
    p = rt.pinned_empty(h.shape, h.dtype)
    p[...] = h
    pin.append(p)
outs0 = prog(*[gp.asarray(h) for h in host])
pout = [rt.pinned_empty(o.shape, o.dtype) for o in outs0]
del outs0


def step():
    outs = prog(*[gp.asarray(h) for h in pin])
    gp.materialize(*outs, out=pout)


for i in range(4):
    t0 = time.perf_counter()
    step()
    print("step", i, "%.2f ms" % ((time.perf_counter() - t0) * 1e3), flush=True)
pr = cProfile.Profile()
pr.enable()
step()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
