// gr_map.cuh — hand-written fused-loop skeleton for Map regions (K1).
//
// Replaces the reference executor's run_map (/root/reference/SPEC.md:364-372:
// out[p] = point(p) over a blocked partition of the linearised space) and the
// paper's GPU map, which ran one point per thread with no vectorisation
// (PAPER.md:444-446, 646-651).  Here:
//   * the iteration space is linearised and cut into VEC-point groups; a group
//     is VEC consecutive points along the innermost axis, so contiguous leaves
//     and every output are moved with one 16-byte access per group;
//   * a persistent grid (a multiple of the SM count × occupancy) walks the
//     groups with a grid stride; U groups per thread per trip, loads of all U
//     groups issued before any compute, for memory-level parallelism;
//   * the group body K::group<U> is generated per region by codegen.py from the
//     region's point program; points are independent, so the output is
//     bit-identical for every grid (SPEC.md:402 determinism).
#pragma once

namespace gr {

// K must provide:
//   struct Params;                      kernel argument block (pointers)
//   static constexpr long long NGROUPS; number of full VEC-groups
//   static constexpr int U;             groups per thread per trip
//   template <int N> static void group(const Params&, long long g, long long stride);
//       processes groups g, g+stride, ..., g+(N-1)*stride (all valid)
//   static constexpr bool TAIL; static void tail(const Params&);
//       scalar points beyond NGROUPS*VEC (rank-1 spaces only)
template <class K> __device__ __forceinline__ void map_kernel(const typename K::Params& p) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (K::U > 1) {
    for (; g + (K::U - 1) * stride < K::NGROUPS; g += K::U * stride) K::template group<K::U>(p, g, stride);
  }
  for (; g < K::NGROUPS; g += stride) K::template group<1>(p, g, stride);
  if (K::TAIL && blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) K::tail(p);
}

}  // namespace gr
