"""Host-side cost of a warm force on tiny arrays (the paper's small-size regime)."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1901_03771_b200 as gp  # noqa: E402
from paper_1901_03771_b200 import workloads as wl  # noqa: E402

S, X, T = wl.blackscholes_inputs(n=1024)
dS, dX, dT = gp.asarray(S), gp.asarray(X), gp.asarray(T)
gp.force(dS + 0, dX + 0, dT + 0)


def step():
    c, p = wl.blackscholes(gp, dS, dX, dT)
    return gp.materialize(c, p)


for _ in range(5):
    step()
n = 200
t0 = time.perf_counter()
for _ in range(n):
    step()
dt = (time.perf_counter() - t0) / n
print(f"warm force+D2H of BS on 1024 options: {dt * 1e6:.1f} us per step")
pr = cProfile.Profile()
pr.enable()
for _ in range(50):
    step()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
