"""Skinny GEMM (the MLP's layer 2, 65536x1024 @ 1024x10): cuBLAS paths timed
with CUDA events (mean of 20 after 3 warm-ups)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1901_03771_b200 import runtime  # noqa: E402
from paper_1901_03771_b200.tensor import DType  # noqa: E402

rt = runtime.get()
m, k = 65536, 1024
for n in (10, 16, 64, 256):
    A = rt.upload(np.random.default_rng(0).random((m, k), dtype=np.float32))
    B = rt.upload(np.random.default_rng(1).random((k, n), dtype=np.float32))
    bias = rt.upload(np.ones(n, np.float32))
    C = rt.alloc(m * n * 4)

    def t(fn):
        for _ in range(3):
            fn()
        ev = []
        for _ in range(20):
            a, b = rt.event(), rt.event()
            rt.record(a)
            fn()
            rt.record(b)
            ev.append((a, b))
        return np.mean([rt.elapsed_ms(a, b) for a, b in ev]) * 1e3
    res = {}
    for mode in ("fp32", "bf16x9"):
        rt.set_gemm_math(mode)
        res["sgemm-" + mode] = t(lambda: rt.gemm(False, False, m, n, k, DType.f32, A.ptr, k, B.ptr, n, C.ptr, n))
    for emu in (False, True):
        res[f"lt-bias-{'x9' if emu else 'fp32'}"] = t(lambda: rt.gemm_epilogue(False, False, m, n, k, A.ptr, k, B.ptr,
                                                                              n, C.ptr, n, bias=bias.ptr,
                                                                              epilogue="bias", emulate=emu))
    rt.set_gemm_math("bf16x9")
    print(f"N={n}: " + "  ".join(f"{kk} {v:.1f}us" for kk, v in res.items()), flush=True)
