#include "gr_ops.cuh"
#include "gr_mem.cuh"
#include "gr_pair.cuh"

#include "gr_reduce.cuh"
#include "gr_tma.cuh"

struct K {
  struct Params {
    const float* __restrict__ in0;
    float* __restrict__ out0;
    float* __restrict__ out1;
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
    const float k11 = gr::f32_bits(0x45800000u);  // 4096.0
    const gr::DivShared<float> t12 = gr::div_prep<float>(k11);
    float S1[16][4];
    #pragma unroll
    for (int mm = 0; mm < 16; ++mm) gr::ldv<float, 4>(S1[mm], p.in0 + r * 4096LL + cb + 8 * mm);
    float acc3[4];
    float acc6[4];
  #pragma unroll
    for (long long i7 = 0; i7 < 16LL; ++i7) {
  #pragma unroll
      for (long long i8 = 0; i8 < 4LL; ++i8) {
        acc6[i8] = (i7 == 0) ? S1[i7][i8] : gr::add<float>(acc6[i8], S1[i7][i8]);
      }
    }
    __shared__ float sh1[8];
    const float t9 = gr::row_sum<float, 4, 2, 64, true>(acc6, sh1, ri);
    const float t10 = gr::add<float>(gr::f32_bits(0x00000000u), t9);
    const float t13 = gr::div_sh<FAST, float>(t10, t12, bad);
    float acc15[4];
    const float t18 = gr::div_sh<FAST, float>(t10, t12, bad);
  #pragma unroll
    for (long long i16 = 0; i16 < 16LL; ++i16) {
  #pragma unroll
      for (long long i17 = 0; i17 < 4LL; ++i17) {
        const float t19 = gr::sub<float>(S1[i16][i17], t18);
        const float t20 = gr::mul<float>(t19, t19);
        acc15[i17] = (i16 == 0) ? t20 : gr::add<float>(acc15[i17], t20);
      }
    }
    __shared__ float sh2[8];
    const float t21 = gr::row_sum<float, 4, 2, 64, true>(acc15, sh2, ri);
    const float t22 = gr::add<float>(gr::f32_bits(0x00000000u), t21);
    const float t23 = gr::div_sh<FAST, float>(t22, t12, bad);
    const float t24 = gr::sqrt_(t23);
    const gr::DivShared<float> t25 = gr::div_prep<float>(t24);
    gr::DivRange<float> w26 = gr::div_range_init<float>();
  #pragma unroll
    for (long long i4 = 0; i4 < 16LL; ++i4) {
      float O2[4];
  #pragma unroll
      for (long long i5 = 0; i5 < 4LL; ++i5) {
        const float t14 = gr::sub<float>(S1[i4][i5], t13);
        const float t27 = gr::div_shr<FAST, float>(t14, t25, w26);
        O2[i5] = t27;
        acc3[i5] = (i4 == 0) ? t27 : gr::add<float>(acc3[i5], t27);
      }
      if (valid) gr::stv<float, 4>(p.out0 + r * 4096LL + cb + 8 * i4, O2);
    }
    __shared__ float sh3[8];
    const float t28 = gr::row_sum<float, 4, 2, 64, true>(acc3, sh3, ri);
    if (valid && tr == 0) reinterpret_cast<float*>(static_cast<char*>(p.scratch) + 0)[r] = t28;
    bad |= gr::div_range_bad<float>(w26, t25);
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
    const float v1 = gr::block_tree<gr::OpSum, float>(reinterpret_cast<const float*>(static_cast<const char*>(p.scratch) + 0), K::NROWS, gr::f32_bits(0x00000000u));
    if (threadIdx.x == 0) p.out1[0] = gr::add<float>(gr::f32_bits(0x00000000u), v1);
  }
}
