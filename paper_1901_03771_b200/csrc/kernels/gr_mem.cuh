// gr_mem.cuh — vectorised global-memory access for the fused-loop skeletons.
//
// Leaves are read-only for the lifetime of a kernel (regions never write a
// buffer they read: outputs are fresh pool allocations), so loads go through
// the non-coherent path (__ldg / LDG.E.CONSTANT) and can be hoisted above the
// region's stores.  Vector width is chosen by the code generator so every
// access is one 16-byte LDG.128/STG.128 when the leaf is contiguous along the
// innermost iteration axis and 16-byte aligned (SURVEY.md §2.2 "128-bit-vector").
#pragma once

namespace gr {

template <int BYTES> struct RawVec;
template <> struct RawVec<1> { typedef unsigned char T; };
template <> struct RawVec<2> { typedef unsigned short T; };
template <> struct RawVec<4> { typedef unsigned int T; };
template <> struct RawVec<8> { typedef uint2 T; };
template <> struct RawVec<16> { typedef uint4 T; };

template <class T, int V> union VecU {
  typename RawVec<sizeof(T) * V>::T raw;
  T v[V];
};

// dst[0..V) = src[0..V); src aligned to sizeof(T)*V
#ifdef GR_LDG_NOALLOC   // experiments: streaming loads that do not allocate in L1
__device__ __forceinline__ uint4 ldg_na(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
template <class X> __device__ __forceinline__ X ldg_any(const X* p) { return __ldg(p); }
template <> __device__ __forceinline__ uint4 ldg_any(const uint4* p) { return ldg_na(p); }
#define GR_LDG ldg_any
#elif !defined(GR_LDG)   // a kernel may bring its own (e.g. reads of TMA-staged tiles)
#define GR_LDG __ldg
#endif
template <class T, int V> __device__ __forceinline__ void ldv(T (&dst)[V], const T* __restrict__ src) {
  VecU<T, V> u;
  u.raw = GR_LDG(reinterpret_cast<const typename RawVec<sizeof(T) * V>::T*>(src));
#pragma unroll
  for (int i = 0; i < V; ++i) dst[i] = u.v[i];
}
template <class T> __device__ __forceinline__ T ld(const T* __restrict__ src) { return __ldg(src); }

// Element i (a compile-time constant once the lane loop is unrolled) of the
// 2V-element window a ++ b: a vector at a constant misalignment (e.g. the
// x[j-1] and x[j+1] neighbours of a stencil) read as two aligned vectors.
template <class T, int V> __device__ __forceinline__ T pick(const T (&a)[V], const T (&b)[V], int i) {
  return i < V ? a[i] : b[i - V];
}
template <> __device__ __forceinline__ bool ld(const bool* __restrict__ src) {
  return __ldg(reinterpret_cast<const unsigned char*>(src)) != 0;
}

template <class T, int V> __device__ __forceinline__ void stv(T* __restrict__ dst, const T (&src)[V]) {
  VecU<T, V> u;
#pragma unroll
  for (int i = 0; i < V; ++i) u.v[i] = src[i];
  *reinterpret_cast<typename RawVec<sizeof(T) * V>::T*>(dst) = u.raw;
}
template <class T> __device__ __forceinline__ void st(T* __restrict__ dst, T x) { *dst = x; }

// the first n of V elements (the last partial group of a packed map body);
// lanes past n read element 0 and are never stored
template <class T, int V> __device__ __forceinline__ void ldv_part(T (&dst)[V], const T* __restrict__ src, int n) {
#pragma unroll
  for (int i = 0; i < V; ++i) dst[i] = src[i < n ? i : 0];
}
template <class T, int V> __device__ __forceinline__ void stv_part(T* __restrict__ dst, const T (&src)[V], int n) {
#pragma unroll
  for (int i = 0; i < V; ++i)
    if (i < n) dst[i] = src[i];
}

// L1 prefetch of the next grid-stride row's leaf data (row family): no
// register or scoreboard dependency, the row's own loads then hit L1
template <class T> __device__ __forceinline__ void prefetch_l1(const T* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

}  // namespace gr
