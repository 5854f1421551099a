#include "gr_ops.cuh"
#include "gr_mem.cuh"
#include "gr_pair.cuh"

#include "gr_reduce.cuh"

__constant__ float gr_cin1[256];

struct K {
  struct Params {
    const float* __restrict__ in0;
    const float* __restrict__ in1;
    long long* __restrict__ out0;
    double* __restrict__ out1;
    double* __restrict__ out2;
    double* __restrict__ out3;
    double* __restrict__ out4;
    long long* __restrict__ out5;
    void* __restrict__ scratch;
    unsigned int* ticket;
  };
  static constexpr long long NROWS = 67108864LL;
  static __device__ __forceinline__ void row(const Params& p, const long long r, const bool valid, double* khist0, double* khist1, double* khist2, double* khist3, long long* khist4) {
    (void)valid;
    int gz; asm volatile("mov.u32 %0, 0;" : "=r"(gz));
    float a1 = 0;
    long long a2 = 0;
    float L7[4];
    gr::ldv<float, 4>(L7, p.in0 + (4*r));
    gr::f2 a11 = gr::splat(0.0f);
  #pragma unroll
    for (long long i12 = 0; i12 < 32LL; ++i12) {
      gr::f2 a13 = gr::splat(gr::f32_bits(0x00000000u));
      gr::f2 a14 = gr::splat(gr::f32_bits(0x80000000u));
  #pragma unroll
      for (long long i15 = 0; i15 < 4LL; ++i15) {
        const gr::f2 t16 = gr::f2{*reinterpret_cast<const unsigned long long*>(&gr_cin1[(i12 * 4 + i15) * 2 + gz])};
        const gr::f2 t17 = gr::p2::sub(gr::splat(L7[i15]), t16);
        const gr::f2 t18 = gr::p2::square_nc(t17);
        a14 = gr::p2::add(a14, t18);
      }
      a13 = gr::p2::add(a13, a14);
      { const float vlo = gr::lo(a13), vhi = gr::hi(a13); if (i12 == 0 || vlo < a1) { a1 = vlo; a2 = 2 * i12; } if (vhi < a1) { a1 = vhi; a2 = 2 * i12 + 1; } }
      a11 = gr::p2::add(a11, a13);
    }
    if (gr::lo(a11) != gr::lo(a11) || gr::hi(a11) != gr::hi(a11)) {
      for (long long i19 = 0; i19 < 64LL; ++i19) {
        float a20 = gr::f32_bits(0x00000000u);
        float a21 = gr::f32_bits(0x80000000u);
  #pragma unroll
        for (long long i22 = 0; i22 < 4LL; ++i22) {
          const float t23 = gr_cin1[(4*i19 + i22)];
          const float t24 = gr::sub<float>(L7[i22], t23);
          const float t25 = gr::square<float>(t24);
          a21 = gr::add<float>(a21, t25);
        }
        a20 = gr::add<float>(a20, a21);
        if (a20 != a20) { a1 = a20; a2 = i19; break; }
      }
    }
    gr::st<long long>(p.out0 + r, a2);
    const long long kkey = valid ? a2 : -1LL;
    const float t26 = gr::ld<float>(p.in0 + (4*r));
    const double t27 = gr::cast<double, float>(t26);
    const double kw0 = t27;
    const float t28 = gr::ld<float>(p.in0 + (4*r + 1));
    const double t29 = gr::cast<double, float>(t28);
    const double kw1 = t29;
    const float t30 = gr::ld<float>(p.in0 + (4*r + 2));
    const double t31 = gr::cast<double, float>(t30);
    const double kw2 = t31;
    const float t32 = gr::ld<float>(p.in0 + (4*r + 3));
    const double t33 = gr::cast<double, float>(t32);
    const double kw3 = t33;
    const long long kw4 = 1LL;
    const unsigned kpeers = __match_any_sync(0xffffffffu, (unsigned long long)kkey);
    const unsigned klane = threadIdx.x & 31u;
    const bool klead = (kpeers & ((1u << klane) - 1u)) == 0u;
    unsigned krest = klead ? (kpeers & (kpeers - 1u)) : 0u;
    double ks0 = kw0;
    double ks1 = kw1;
    double ks2 = kw2;
    double ks3 = kw3;
    while (__any_sync(0xffffffffu, krest != 0u)) {
      const int ksrc = krest ? __ffs(krest) - 1 : (int)klane;
      const double kv0 = __shfl_sync(0xffffffffu, kw0, ksrc);
      const double kv1 = __shfl_sync(0xffffffffu, kw1, ksrc);
      const double kv2 = __shfl_sync(0xffffffffu, kw2, ksrc);
      const double kv3 = __shfl_sync(0xffffffffu, kw3, ksrc);
      if (krest) {
        ks0 += kv0;
        ks1 += kv1;
        ks2 += kv2;
        ks3 += kv3;
        krest &= krest - 1u;
      }
    }
    if (klead && kkey >= 0) {
      if (kkey < 64LL) khist0[(threadIdx.x >> 5) * 64 + kkey] += ks0;
      if (kkey < 64LL) khist1[(threadIdx.x >> 5) * 64 + kkey] += ks1;
      if (kkey < 64LL) khist2[(threadIdx.x >> 5) * 64 + kkey] += ks2;
      if (kkey < 64LL) khist3[(threadIdx.x >> 5) * 64 + kkey] += ks3;
      if (kkey < 64LL) khist4[(threadIdx.x >> 5) * 64 + kkey] += (long long)__popc(kpeers);
    }
  }
};
extern "C" __global__ void __launch_bounds__(128) gr_region(const K::Params p) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  __shared__ double khist0[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) khist0[i] = 0;
  __shared__ double khist1[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) khist1[i] = 0;
  __shared__ double khist2[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) khist2[i] = 0;
  __shared__ double khist3[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) khist3[i] = 0;
  __shared__ long long khist4[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) khist4[i] = 0;
  __syncthreads();
  for (long long base = (long long)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < K::NROWS; base += stride) {
    const long long r = base + (threadIdx.x & 31);
    K::row(p, r < K::NROWS ? r : K::NROWS - 1, r < K::NROWS, khist0, khist1, khist2, khist3, khist4);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < 64; b += blockDim.x) {
    double s = khist0[b];
    for (int w = 1; w < 4; ++w) s += khist0[w * 64 + b];
    reinterpret_cast<double*>(static_cast<char*>(p.scratch) + 0)[(long long)blockIdx.x * 64 + b] = s;
  }
  for (int b = threadIdx.x; b < 64; b += blockDim.x) {
    double s = khist1[b];
    for (int w = 1; w < 4; ++w) s += khist1[w * 64 + b];
    reinterpret_cast<double*>(static_cast<char*>(p.scratch) + 1212416)[(long long)blockIdx.x * 64 + b] = s;
  }
  for (int b = threadIdx.x; b < 64; b += blockDim.x) {
    double s = khist2[b];
    for (int w = 1; w < 4; ++w) s += khist2[w * 64 + b];
    reinterpret_cast<double*>(static_cast<char*>(p.scratch) + 2424832)[(long long)blockIdx.x * 64 + b] = s;
  }
  for (int b = threadIdx.x; b < 64; b += blockDim.x) {
    double s = khist3[b];
    for (int w = 1; w < 4; ++w) s += khist3[w * 64 + b];
    reinterpret_cast<double*>(static_cast<char*>(p.scratch) + 3637248)[(long long)blockIdx.x * 64 + b] = s;
  }
  for (int b = threadIdx.x; b < 64; b += blockDim.x) {
    long long s = khist4[b];
    for (int w = 1; w < 4; ++w) s += khist4[w * 64 + b];
    reinterpret_cast<long long*>(static_cast<char*>(p.scratch) + 4849664)[(long long)blockIdx.x * 64 + b] = s;
  }
  if (gr::last_block(p.ticket)) {
    for (int b = threadIdx.x; b < 64; b += blockDim.x) {
      double s = 0;
      for (unsigned c = 0; c < gridDim.x; ++c) s += reinterpret_cast<const double*>(static_cast<const char*>(p.scratch) + 0)[(long long)c * 64 + b];
      p.out1[b] = s;
    }
    for (int b = threadIdx.x; b < 64; b += blockDim.x) {
      double s = 0;
      for (unsigned c = 0; c < gridDim.x; ++c) s += reinterpret_cast<const double*>(static_cast<const char*>(p.scratch) + 1212416)[(long long)c * 64 + b];
      p.out2[b] = s;
    }
    for (int b = threadIdx.x; b < 64; b += blockDim.x) {
      double s = 0;
      for (unsigned c = 0; c < gridDim.x; ++c) s += reinterpret_cast<const double*>(static_cast<const char*>(p.scratch) + 2424832)[(long long)c * 64 + b];
      p.out3[b] = s;
    }
    for (int b = threadIdx.x; b < 64; b += blockDim.x) {
      double s = 0;
      for (unsigned c = 0; c < gridDim.x; ++c) s += reinterpret_cast<const double*>(static_cast<const char*>(p.scratch) + 3637248)[(long long)c * 64 + b];
      p.out4[b] = s;
    }
    for (int b = threadIdx.x; b < 64; b += blockDim.x) {
      long long s = 0;
      for (unsigned c = 0; c < gridDim.x; ++c) s += reinterpret_cast<const long long*>(static_cast<const char*>(p.scratch) + 4849664)[(long long)c * 64 + b];
      p.out5[b] = s;
    }
  }
}
