#include "gr_ops.cuh"
#include "gr_mem.cuh"
#include "gr_pair.cuh"

#include "gr_reduce.cuh"
#include "gr_tma.cuh"

struct K {
  struct Params {
    const float* __restrict__ in0;
    float* __restrict__ out0;
    void* __restrict__ scratch;
    unsigned int* ticket;
  };
  static constexpr long long NROWS = 65536LL;
  static constexpr long long NG = 16384LL;
  template <bool FAST> static __device__ __forceinline__ bool rows(const Params& p, const long long rb, unsigned char* stage, unsigned long long* bar, const long long gnext) {
    const int tr = threadIdx.x % 64;
    const int ri = threadIdx.x / 64;
    const bool valid = rb + ri < NROWS;
    const long long r = valid ? rb + ri : NROWS - 1;
    const long long cb = (long long)(tr / 2) * 128 + (tr % 2) * 4;
    (void)stage; (void)bar; (void)gnext;
    bool bad = false;
    const float k10 = gr::f32_bits(0x45800000u);  // 4096.0
    const gr::DivShared<float> t11 = gr::div_prep<float>(k10);
    float S1[16][4];
    #pragma unroll
    for (int mm = 0; mm < 16; ++mm) gr::ldv<float, 4>(S1[mm], p.in0 + r * 4096LL + cb + 8 * mm);
    gr::f2 a5[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) a5[h] = gr::pk(S1[0][2*h], S1[0][2*h+1]);
#pragma unroll
    for (int i = 1; i < 16; ++i)
#pragma unroll
      for (int h = 0; h < 2; ++h) a5[h] = gr::p2::add(a5[h], gr::pk(S1[i][2*h], S1[i][2*h+1]));
    float acc5[4] = {gr::lo(a5[0]), gr::hi(a5[0]), gr::lo(a5[1]), gr::hi(a5[1])};
    __shared__ float sh1[8];
    const float t8 = gr::row_sum<float, 4, 2, 64>(acc5, sh1, ri);
    const float t9 = gr::add<float>(gr::f32_bits(0x00000000u), t8);
    const float t12 = gr::div_sh<FAST, float>(t9, t11, bad);
    const gr::f2 m2 = gr::splat(t12);
    gr::f2 a14[2];
#pragma unroll
    for (int i = 0; i < 16; ++i)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const gr::f2 t = gr::p2::sub(gr::pk(S1[i][2*h], S1[i][2*h+1]), m2);
        const gr::f2 sq = gr::p2::mul_nc(t, t);
        a14[h] = i == 0 ? sq : gr::p2::add(a14[h], sq);
      }
    float acc14[4] = {gr::lo(a14[0]), gr::hi(a14[0]), gr::lo(a14[1]), gr::hi(a14[1])};
    __shared__ float sh2[8];
    const float t20 = gr::row_sum<float, 4, 2, 64>(acc14, sh2, ri);
    const float t21 = gr::add<float>(gr::f32_bits(0x00000000u), t20);
    const float t22 = gr::div_sh<FAST, float>(t21, t11, bad);
    const float t23 = gr::sqrt_(t22);
    const gr::DivShared<float> t24 = gr::div_prep<float>(t23);
    const gr::f2 r2 = gr::splat(t24.r), ns2 = gr::splat(-t24.s);
    gr::f2 a2[2];
#pragma unroll
    for (int i = 0; i < 16; ++i)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const gr::f2 t = gr::p2::sub(gr::pk(S1[i][2*h], S1[i][2*h+1]), m2);
        gr::f2 q;
        if constexpr (FAST) {
          const gr::f2 q0 = gr::p2::mul(t, r2);
          const gr::f2 e = gr::p2::fma(q0, ns2, t);
          q = gr::p2::fma(e, r2, q0);
          const float x0 = fabsf(gr::lo(t)), x1 = fabsf(gr::hi(t));
          bad |= !(x0 >= t24.xlo && x0 <= t24.xhi) || !(x1 >= t24.xlo && x1 <= t24.xhi);
        } else {
          q = gr::pk(gr::div_shared<float>(gr::lo(t), t24), gr::div_shared<float>(gr::hi(t), t24));
        }
        a2[h] = i == 0 ? q : gr::p2::add(a2[h], q);
      }
    float acc2[4] = {gr::lo(a2[0]), gr::hi(a2[0]), gr::lo(a2[1]), gr::hi(a2[1])};
    __shared__ float sh3[8];
    const float t26 = gr::row_sum<float, 4, 2, 64>(acc2, sh3, ri);
    if (valid && tr == 0) reinterpret_cast<float*>(static_cast<char*>(p.scratch) + 0)[r] = t26;
    return bad;
  }
};
extern "C" __global__ void __launch_bounds__(256, 3) gr_region(const K::Params p) {
  for (long long g = blockIdx.x; g < K::NG; g += gridDim.x)
    if (__syncthreads_or(K::rows<true>(p, g * 4, nullptr, nullptr, 0)))
      K::rows<false>(p, g * 4, nullptr, nullptr, 0);
  if (gr::last_block(p.ticket)) {
    const float v0 = gr::block_tree<gr::OpSum, float>(reinterpret_cast<const float*>(static_cast<const char*>(p.scratch) + 0), K::NROWS, gr::f32_bits(0x00000000u));
    if (threadIdx.x == 0) p.out0[0] = gr::add<float>(gr::f32_bits(0x00000000u), v0);
  }
}
