"""PCIe copy bandwidth on this box: H2D alone, D2H alone, both concurrently
(pinned host buffers, 256 MB chunks on separate streams)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1901_03771_b200 import runtime  # noqa: E402

rt = runtime.get()
N = 3 << 30
h_in = rt.pinned_empty((N,), np.uint8)
h_out = rt.pinned_empty((N,), np.uint8)
h_in[:] = 1
d = rt.alloc(N)
d2 = rt.alloc(N)
s1, s2 = rt.stream_create(), rt.stream_create()
C = 256 << 20


def run(h2d, d2h, reps=3):
    best = 1e9
    for _ in range(reps):
        rt.sync()
        t0 = time.perf_counter()
        for off in range(0, N, C):
            if h2d:
                rt.set_stream(s1)
                rt.h2d_async(d.ptr + off, h_in[off:off + C])
            if d2h:
                rt.set_stream(s2)
                rt.d2h_async(h_out[off:off + C], d2.ptr + off)
        rt.set_stream(0)
        rt.sync()
        best = min(best, time.perf_counter() - t0)
    return best


for name, a, b in (("h2d", 1, 0), ("d2h", 0, 1), ("both", 1, 1)):
    t = run(a, b)
    print(f"{name}: {N * (a + b) / t / 1e9:.1f} GB/s aggregate ({t * 1e3:.1f} ms for {(a + b) * N / 2**30:.0f} GiB)")
