"""First-call cost of the cuBLAS paths in a fresh process (run it with
CUDA_CACHE_DISABLE=1 to include any driver JIT of library PTX)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1901_03771_b200 import runtime  # noqa: E402
from paper_1901_03771_b200.tensor import DType  # noqa: E402

rt = runtime.get()
m, k, n = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
mode = sys.argv[4]
A = rt.upload(np.ones((m, k), np.float32))
B = rt.upload(np.ones((k, n), np.float32))
bias = rt.upload(np.ones(n, np.float32))
C = rt.alloc(m * n * 4)
rt.sync()
for i in range(2):
    t = time.perf_counter()
    if mode in ("fp32", "bf16x9"):
        rt.set_gemm_math(mode)
        rt.gemm(False, False, m, n, k, DType.f32, A.ptr, k, B.ptr, n, C.ptr, n)
    else:
        rt.gemm_epilogue(False, False, m, n, k, A.ptr, k, B.ptr, n, C.ptr, n, bias=bias.ptr,
                         epilogue=mode, emulate=True)
    rt.sync()
    print(f"{mode} {m}x{k}x{n} call {i}: {time.perf_counter() - t:.3f} s", flush=True)
