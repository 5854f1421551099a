"""Probe: achievable DRAM bandwidth of pure streaming READS (1 GiB, LDG.128,
U loads in flight per thread, grid-stride) against a copy, on one B200 —
the ceiling a read-dominated kernel such as row-normalise's total can reach.
usage: read_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1901_03771_b200 import runtime  # noqa: E402

SRC = r'''
extern "C" __global__ void __launch_bounds__(256) rd(const float4* __restrict__ x, float* __restrict__ o, long long n4) {
  float s = 0.f;
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n4; i += U * stride) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldg(x + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) s += v[u].x + v[u].y + v[u].z + v[u].w;
  }
  for (; i < n4; i += stride) { float4 v = x[i]; s += v.x + v.y + v.z + v.w; }
  if (s == 123.f) o[0] = s;
}
extern "C" __global__ void __launch_bounds__(256) cp(const float4* __restrict__ x, float4* __restrict__ o, long long n4) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n4; i += U * stride) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldg(x + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) o[i + u * stride] = v[u];
  }
  for (; i < n4; i += stride) o[i] = x[i];
}
'''


def main():
    rt = runtime.get()
    n = 1 << 28
    x = rt.alloc(n * 4)
    o = rt.alloc(n * 4)
    rt.memset(x, 0)
    for U in (1, 2, 4, 8, 16):
        src = f"#define U {U}\n" + SRC
        for name, nbytes in (("rd", n * 4), ("cp", n * 8)):
            k = rt.kernel(src, name, 256)
            for mult in (1, 2):
                grid = rt.sm_count * k.blocks_per_sm * mult
                ms = []
                for i in range(10):
                    e0, e1 = rt.event(), rt.event()
                    rt.record(e0)
                    rt.launch(k, grid, 256, runtime.pack_params([x.ptr, o.ptr, n // 4]))
                    rt.record(e1)
                    rt.sync()
                    if i >= 2:
                        ms.append(rt.elapsed_ms(e0, e1))
                t = float(np.mean(ms))
                print(f"{name} U={U:2d} regs={k.num_regs} occ={k.blocks_per_sm} grid={grid}: {t:.4f} ms "
                      f"{nbytes / t / 1e6:.0f} GB/s", flush=True)


if __name__ == "__main__":
    main()
