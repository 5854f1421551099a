#!/usr/bin/env python
"""Host-side cost of one bench step: recording, planning, launch, pool traffic.

usage: python tools/hostprof.py [workload] [steps]
"""
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import bench  # noqa: E402
import paper_1901_03771_b200 as gp  # noqa: E402
from paper_1901_03771_b200 import runtime  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "blackscholes-f32"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    w = bench.WORKLOADS[name]
    rt = runtime.get()
    sess = gp.Session()
    gp.set_default_session(sess)
    host = bench.make_inputs(name, w["n"], 42)
    dev = [gp.asarray(x) for x in host]
    for d in dev:
        d.node.data.device = rt.upload(d.node.data.host)
    prog = bench.make_program(name)
    for _ in range(3):
        gp.force(*prog(gp, dev))
    rt.sync()
    p0 = rt.pool_stats()
    rec = frc = 0.0
    keep = []
    t_all = time.perf_counter()
    for _ in range(steps):
        t0 = time.perf_counter()
        outs = prog(gp, dev)
        t1 = time.perf_counter()
        gp.force(*outs)
        t2 = time.perf_counter()
        rec += t1 - t0
        frc += t2 - t1
        keep.append(outs)
        if len(keep) > 2:
            keep.pop(0)
    t_host = time.perf_counter() - t_all
    rt.sync()
    t_dev = time.perf_counter() - t_all
    p1 = rt.pool_stats()
    print(f"{name}: host/step {t_host / steps * 1e3:.3f} ms (record {rec / steps * 1e3:.3f}, force {frc / steps * 1e3:.3f}),"
          f" wall incl. device {t_dev / steps * 1e3:.3f} ms; cuMemAlloc calls during loop: "
          f"{p1['cuMemAlloc_calls'] - p0['cuMemAlloc_calls']}; pool {p1}")


if __name__ == "__main__":
    main()
