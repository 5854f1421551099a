#!/usr/bin/env python
"""Host-side cost of one bench step without a GPU: the runtime is replaced by
a stub whose launches, copies and allocations do nothing, so the timing is
recording + plan-cache lookup + executor bookkeeping + parameter packing.

usage: python tools/hostprof_cpu.py [workload] [steps] [--profile]
"""
import cProfile
import itertools
import os
import pstats
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402

import paper_1901_03771_b200 as gp  # noqa: E402
from paper_1901_03771_b200 import runtime  # noqa: E402


class _Buf:
    _ids = itertools.count(1 << 20)

    def __init__(self, nbytes):
        self.ptr = next(self._ids) * 256
        self.nbytes = nbytes


class _Kernel:
    def __init__(self):
        self.fn, self.module, self.blocks_per_sm, self.cache_hit, self.compile_ms = 1, 1, 8, 1, 0.0


class FakeRuntime:
    device, sm_count, gemm_math, name = 0, 148, "bf16x9", "stub"

    def alloc(self, n):
        return _Buf(n)

    def upload(self, a):
        return _Buf(a.nbytes)

    def kernel(self, *a, **k):
        return _Kernel()

    def function(self, *a):
        return 1

    def module_global(self, *a):
        return (4096, 0)

    def event(self):
        return 1

    def __getattr__(self, name):
        return lambda *a, **k: None


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    name = args[0] if args else "blackscholes-f32"
    steps = int(args[1]) if len(args) > 1 else 200
    runtime._rt = FakeRuntime()
    import bench
    w = bench.WORKLOADS[name]
    wl = bench._programs()
    n = wl.NAMED[name][1]          # one row block of inputs: shapes differ, host work does not
    host = wl.named_inputs(name, 0, n)
    sess = gp.Session()
    gp.set_default_session(sess)
    dev = [gp.asarray(x) for x in host]
    prog = w["program"]
    for _ in range(3):
        gp.force(*prog(gp, dev))

    def loop():
        keep = []
        for _ in range(steps):
            outs = prog(gp, dev)
            gp.force(*outs)
            keep.append(outs)
            if len(keep) > 2:
                keep.pop(0)

    t0 = time.perf_counter()
    loop()
    dt = (time.perf_counter() - t0) / steps
    print(f"{name}: host per step {dt * 1e6:.1f} us (stub runtime, {steps} steps)")
    if "--profile" in sys.argv:
        cProfile.runctx("loop()", globals(), locals(), "/tmp/hostprof.out")
        pstats.Stats("/tmp/hostprof.out").sort_stats("tottime").print_stats(25)


if __name__ == "__main__":
    main()
