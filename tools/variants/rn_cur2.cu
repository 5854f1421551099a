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
  #pragma unroll
    for (long long i6 = 0; i6 < 16LL; ++i6) {
  #pragma unroll
      for (long long i7 = 0; i7 < 4LL; ++i7) {
        acc5[i7] = (i6 == 0) ? S1[i6][i7] : gr::add<float>(acc5[i7], S1[i6][i7]);
      }
    }
    __shared__ float sh1[8];
    const float t8 = gr::row_sum<float, 4, 2, 64, false>(acc5, sh1, ri);
    const float t9 = gr::add<float>(gr::f32_bits(0x00000000u), t8);
    const float t12 = gr::div_sh<FAST, float>(t9, t11, bad);
    float acc14[4];
    const float t17 = gr::div_sh<FAST, float>(t9, t11, bad);
  #pragma unroll
    for (long long i15 = 0; i15 < 16LL; ++i15) {
  #pragma unroll
      for (long long i16 = 0; i16 < 4LL; ++i16) {
        const float t18 = gr::sub<float>(S1[i15][i16], t17);
        const float t19 = gr::mul<float>(t18, t18);
        acc14[i16] = (i15 == 0) ? t19 : gr::add<float>(acc14[i16], t19);
      }
    }
    __shared__ float sh2[8];
    const float t20 = gr::row_sum<float, 4, 2, 64, false>(acc14, sh2, ri);
    const float t21 = gr::add<float>(gr::f32_bits(0x00000000u), t20);
    const float t22 = gr::div_sh<FAST, float>(t21, t11, bad);
    const float t23 = gr::sqrt_(t22);
    const gr::DivShared<float> t24 = gr::div_prep<float>(t23);
    gr::DivRange<float> w25 = gr::div_range_init<float>();
  #pragma unroll
    for (long long i3 = 0; i3 < 16LL; ++i3) {
  #pragma unroll
      for (long long i4 = 0; i4 < 4LL; ++i4) {
        const float t13 = gr::sub<float>(S1[i3][i4], t12);
        const float t26 = gr::div_shr<FAST, float>(t13, t24, w25);
        acc2[i4] = (i3 == 0) ? t26 : gr::add<float>(acc2[i4], t26);
      }
    }
    __shared__ float sh3[8];
    const float t27 = gr::row_sum<float, 4, 2, 64, false>(acc2, sh3, ri);
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
