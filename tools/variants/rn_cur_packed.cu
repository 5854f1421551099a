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
    unsigned int* redo;
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
    float acc2[4];
    float acc5[4];
    {
      gr::f2 a0 = gr::pk(S1[0][0], S1[0][1]), a1 = gr::pk(S1[0][2], S1[0][3]);
  #pragma unroll
      for (int i = 1; i < 16; ++i) { a0 = gr::p2::add(a0, gr::pk(S1[i][0], S1[i][1])); a1 = gr::p2::add(a1, gr::pk(S1[i][2], S1[i][3])); }
      acc5[0] = gr::lo(a0); acc5[1] = gr::hi(a0); acc5[2] = gr::lo(a1); acc5[3] = gr::hi(a1);
    }
    __shared__ float sh1[8];
    const float t8 = gr::row_sum<float, 4, 2, 64>(acc5, sh1, ri);
    const float t9 = gr::add<float>(gr::f32_bits(0x00000000u), t8);
    const float t12 = gr::div_sh<FAST, float>(t9, t11, bad);
    float acc14[4];
    const float t17 = gr::div_sh<FAST, float>(t9, t11, bad);
    {
      const gr::f2 m2 = gr::splat(t17);
      gr::f2 a0, a1;
  #pragma unroll
      for (int i = 0; i < 16; ++i) {
        const gr::f2 d0 = gr::p2::sub(gr::pk(S1[i][0], S1[i][1]), m2), d1 = gr::p2::sub(gr::pk(S1[i][2], S1[i][3]), m2);
        const gr::f2 q0 = gr::p2::mul_nc(d0, d0), q1 = gr::p2::mul_nc(d1, d1);
        if (i == 0) { a0 = q0; a1 = q1; } else { a0 = gr::p2::add(a0, q0); a1 = gr::p2::add(a1, q1); }
      }
      acc14[0] = gr::lo(a0); acc14[1] = gr::hi(a0); acc14[2] = gr::lo(a1); acc14[3] = gr::hi(a1);
    }
    __shared__ float sh2[8];
    const float t20 = gr::row_sum<float, 4, 2, 64>(acc14, sh2, ri);
    const float t21 = gr::add<float>(gr::f32_bits(0x00000000u), t20);
    const float t22 = gr::div_sh<FAST, float>(t21, t11, bad);
    const float t23 = gr::sqrt_(t22);
    const gr::DivShared<float> t24 = gr::div_prep<float>(t23);
    gr::DivRange<float> w25 = gr::div_range_init<float>();
    if constexpr (FAST) {
      const gr::f2 m2 = gr::splat(t12), r2 = gr::splat(t24.r), ns2 = gr::splat(-t24.s);
      gr::f2 a0, a1;
  #pragma unroll
      for (int i = 0; i < 16; ++i) {
        const gr::f2 d0 = gr::p2::sub(gr::pk(S1[i][0], S1[i][1]), m2), d1 = gr::p2::sub(gr::pk(S1[i][2], S1[i][3]), m2);
        const gr::f2 e0 = gr::p2::mul(d0, r2), e1 = gr::p2::mul(d1, r2);
        const gr::f2 f0 = gr::p2::fma(e0, ns2, d0), f1 = gr::p2::fma(e1, ns2, d1);
        const gr::f2 q0 = gr::p2::fma(f0, r2, e0), q1 = gr::p2::fma(f1, r2, e1);
        w25.amin = fminf(w25.amin, fminf(fminf(fabsf(gr::lo(d0)), fabsf(gr::hi(d0))), fminf(fabsf(gr::lo(d1)), fabsf(gr::hi(d1)))));
        w25.amax = fmaxf(w25.amax, fmaxf(fmaxf(fabsf(gr::lo(d0)), fabsf(gr::hi(d0))), fmaxf(fabsf(gr::lo(d1)), fabsf(gr::hi(d1)))));
        if (i == 0) { a0 = q0; a1 = q1; } else { a0 = gr::p2::add(a0, q0); a1 = gr::p2::add(a1, q1); }
      }
      acc2[0] = gr::lo(a0); acc2[1] = gr::hi(a0); acc2[2] = gr::lo(a1); acc2[3] = gr::hi(a1);
    } else {
  #pragma unroll
    for (long long i3 = 0; i3 < 16LL; ++i3) {
  #pragma unroll
      for (long long i4 = 0; i4 < 4LL; ++i4) {
        const float t13 = gr::sub<float>(S1[i3][i4], t12);
        const float t26 = gr::div_shr<FAST, float>(t13, t24, w25);
        acc2[i4] = (i3 == 0) ? t26 : gr::add<float>(acc2[i4], t26);
      }
    }
    }
    __shared__ float sh3[8];
    const float t27 = gr::row_sum<float, 4, 2, 64>(acc2, sh3, ri);
    if (valid && tr == 0) reinterpret_cast<float*>(static_cast<char*>(p.scratch) + 0)[r] = t27;
    bad |= gr::div_range_bad<float>(w25, t24);
    return bad;
  }
};
extern "C" __global__ void __launch_bounds__(256, 3) gr_region(const K::Params p) {
  for (long long g = blockIdx.x; g < K::NG; g += gridDim.x) {
    if (K::rows<true>(p, g * 4, nullptr, nullptr, 0)) atomicOr(p.redo + ((g * 4 + threadIdx.x / 64) >> 5), 1u << ((g * 4 + threadIdx.x / 64) & 31));
  }
  __syncthreads();
  for (long long g = blockIdx.x; g < K::NG; g += gridDim.x) {
    const unsigned bits = (__ldcg(p.redo + ((g * 4) >> 5)) >> ((g * 4) & 31)) & 15u;
    if (bits) {
      __syncthreads();
      if (threadIdx.x == 0) atomicAnd(p.redo + ((g * 4) >> 5), ~(15u << ((g * 4) & 31)));
      K::rows<false>(p, g * 4, nullptr, nullptr, K::NG);
    }
  }
  if (gr::last_block(p.ticket)) {
    const float v0 = gr::block_tree<gr::OpSum, float>(reinterpret_cast<const float*>(static_cast<const char*>(p.scratch) + 0), K::NROWS, gr::f32_bits(0x00000000u));
    if (threadIdx.x == 0) p.out0[0] = gr::add<float>(gr::f32_bits(0x00000000u), v0);
  }
}
