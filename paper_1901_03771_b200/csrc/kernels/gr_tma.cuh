// gr_tma.cuh — bulk asynchronous copies (TMA bulk engine) and mbarriers.
//
// The row-streaming family (codegen_wrow.py) moves each row of a region's
// inputs from HBM into a shared-memory ring with `cp.async.bulk` (SASS
// UBLKCP), completion signalled on an mbarrier (expect_tx / complete_tx), so
// the next rows are in flight while the current one is reduced — no register
// staging, no LSU traffic for the stream (PTX ISA: cp.async.bulk, mbarrier).
#pragma once

namespace gr {

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// order this thread's prior generic-proxy smem accesses before later
// async-proxy (bulk copy) writes to the same smem
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(unsigned long long* bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// global -> shared bulk copy; bytes % 16 == 0, both addresses 16-byte aligned
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// TMA tensor copies: the 128-byte CUtensorMap built on the host
// (grumpy_rt_tensor_map_2d) travels in the kernel's __grid_constant__
// parameter block; one instruction moves a whole box (e.g. a 16 KB row).
struct alignas(64) TMap {
  unsigned long long v[16];
};

__device__ __forceinline__ void tma_load_2d(void* dst, const TMap* map, int x, int y, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

// shared -> global tensor store of a whole box (bulk-group completion):
// commit, then wait_group.read before the smem is overwritten, wait_group
// before the kernel may exit
__device__ __forceinline__ void tma_store_2d(const TMap* map, int x, int y, const void* src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<unsigned long long>(map)),
               "r"(x), "r"(y), "r"(smem_u32(src))
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N> __device__ __forceinline__ void bulk_wait() { asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Element offset -> byte offset inside a [rows][128 B] box stored with the
// 128-byte swizzle: element e of an S-byte type sits in line e*S/128, 16-byte
// chunk (e*S%128)/16 xor (line % 8).
template <int S> __device__ __forceinline__ unsigned sw128_elem(unsigned e) {
  const unsigned b = e * S;
  return (b & ~127u) | ((((b >> 4) & 7u) ^ ((b >> 7) & 7u)) << 4) | (b & 15u);
}
// V consecutive elements (one 16-byte chunk) of a swizzled box <-> registers
template <class T, int V> __device__ __forceinline__ void lds_sw(T (&d)[V], const unsigned char* base, unsigned e) {
  static_assert(sizeof(T) * V == 16, "one 16-byte chunk");
  VecU<T, V> u;
  u.raw = *reinterpret_cast<const uint4*>(base + sw128_elem<sizeof(T)>(e));
#pragma unroll
  for (int i = 0; i < V; ++i) d[i] = u.v[i];
}
template <class T, int V> __device__ __forceinline__ void sts_sw(unsigned char* base, unsigned e, const T (&s)[V]) {
  static_assert(sizeof(T) * V == 16, "one 16-byte chunk");
  VecU<T, V> u;
#pragma unroll
  for (int i = 0; i < V; ++i) u.v[i] = s[i];
  *reinterpret_cast<uint4*>(base + sw128_elem<sizeof(T)>(e)) = u.raw;
}

// Byte offset of 16-byte chunk `c` (0..7) of 128-byte line `L` inside a box
// stored with CU_TENSOR_MAP_SWIZZLE_128B (1024-byte aligned atoms).
__device__ __forceinline__ unsigned sw128(unsigned L, unsigned c) { return L * 128u + ((c ^ (L & 7u)) << 4); }

// Bulk prefetch of [src, src+bytes) into L2 (no shared memory, no completion):
// later LDGs of that range hit L2 instead of HBM.
__device__ __forceinline__ void prefetch_l2(const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// Per-thread asynchronous 16-byte global->shared copies (LDGSTS).  Each thread
// stages exactly the elements it will read back, so completion needs only the
// thread's own wait_group — no CTA barrier — and the copies of the next work
// item stay in flight while this one computes from registers.
__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sdst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// V consecutive elements (16 bytes) from shared memory into registers
template <class T, int V> __device__ __forceinline__ void ldsv(T (&d)[V], const T* s) {
  VecU<T, V> u;
  u.raw = *reinterpret_cast<const typename RawVec<sizeof(T) * V>::T*>(s);
#pragma unroll
  for (int i = 0; i < V; ++i) d[i] = u.v[i];
}

// 8 consecutive elements from shared memory (16-byte aligned) into registers
template <class T> __device__ __forceinline__ void lds8(T (&d)[8], const T* s) {
  static_assert(sizeof(T) == 4 || sizeof(T) == 8, "lds8");
  if constexpr (sizeof(T) == 4) {
    const uint4 a = reinterpret_cast<const uint4*>(s)[0];
    const uint4 b = reinterpret_cast<const uint4*>(s)[1];
    d[0] = __uint_as_float(a.x); d[1] = __uint_as_float(a.y); d[2] = __uint_as_float(a.z); d[3] = __uint_as_float(a.w);
    d[4] = __uint_as_float(b.x); d[5] = __uint_as_float(b.y); d[6] = __uint_as_float(b.z); d[7] = __uint_as_float(b.w);
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const double2 a = reinterpret_cast<const double2*>(s)[i];
      d[2 * i] = a.x;
      d[2 * i + 1] = a.y;
    }
  }
}
template <> __device__ __forceinline__ void lds8<int>(int (&d)[8], const int* s) {
  const int4 a = reinterpret_cast<const int4*>(s)[0];
  const int4 b = reinterpret_cast<const int4*>(s)[1];
  d[0] = a.x; d[1] = a.y; d[2] = a.z; d[3] = a.w; d[4] = b.x; d[5] = b.y; d[6] = b.z; d[7] = b.w;
}
template <> __device__ __forceinline__ void lds8<long long>(long long (&d)[8], const long long* s) {
#pragma unroll
  for (int i = 0; i < 8; ++i) d[i] = s[i];
}

// 8 consecutive elements to global memory (32/64-byte aligned run)
template <class T> __device__ __forceinline__ void st8(T* dst, const T (&v)[8]) {
  constexpr int V = 16 / sizeof(T);
#pragma unroll
  for (int i = 0; i < 8; i += V) {
    T tmp[V];
#pragma unroll
    for (int k = 0; k < V; ++k) tmp[k] = v[i + k];
    stv<T, V>(dst + i, tmp);
  }
}

}  // namespace gr
