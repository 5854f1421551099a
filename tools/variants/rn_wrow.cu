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
  static __device__ __forceinline__ void rows(const Params& p, const unsigned char* stage, const long long g, const int lane) {
    const int q = lane / 32;
    const int lr = lane % 32;
    const long long r0 = g * 1 + q;
    const bool valid = r0 < NROWS;
    const long long r = valid ? r0 : NROWS - 1;
    const int lf0 = lr * 1;
    const long long lfb = (long long)lf0 * 128;
    const unsigned char* sst0 = stage + 0 + (long long)q * 16896;
    const float k16 = gr::f32_bits(0x45800000u);  // 4096.0
    const gr::DivShared<float> t17 = gr::div_prep<float>(k16);
    float ls1[1];
    float ls7[1];
  #pragma unroll
    for (long long i9 = 0; i9 < 1LL; ++i9) {
      float acc8[8];
  #pragma unroll
      for (long long i10 = 0; i10 < 16LL; ++i10) {
        float L12[8];
        gr::lds8<float>(L12, reinterpret_cast<const float*>(sst0) + (lf0 + i9) * 132 + 8 * i10);
  #pragma unroll
        for (long long i11 = 0; i11 < 8LL; ++i11) {
          acc8[i11] = (i10 == 0) ? L12[i11] : gr::add<float>(acc8[i11], L12[i11]);
        }
      }
      ls7[i9] = gr::leaf_local<float, 8>(acc8);
    }
    const float t13 = gr::lane_tree<gr::OpSum, float, 1>(ls7);
    const float t14 = gr::warp_tree<gr::OpSum, float>(t13, 32);
    const float t15 = gr::add<float>(gr::f32_bits(0x00000000u), t14);
    const float t18 = gr::div_shared<float>(t15, t17);
    float ls20[1];
    const float t26 = gr::div_shared<float>(t15, t17);
  #pragma unroll
    for (long long i22 = 0; i22 < 1LL; ++i22) {
      float acc21[8];
  #pragma unroll
      for (long long i23 = 0; i23 < 16LL; ++i23) {
        float L25[8];
        gr::lds8<float>(L25, reinterpret_cast<const float*>(sst0) + (lf0 + i22) * 132 + 8 * i23);
  #pragma unroll
        for (long long i24 = 0; i24 < 8LL; ++i24) {
          const float t27 = gr::sub<float>(L25[i24], t26);
          const float t28 = gr::mul<float>(t27, t27);
          acc21[i24] = (i23 == 0) ? t28 : gr::add<float>(acc21[i24], t28);
        }
      }
      ls20[i22] = gr::leaf_local<float, 8>(acc21);
    }
    const float t29 = gr::lane_tree<gr::OpSum, float, 1>(ls20);
    const float t30 = gr::warp_tree<gr::OpSum, float>(t29, 32);
    const float t31 = gr::add<float>(gr::f32_bits(0x00000000u), t30);
    const float t32 = gr::div_shared<float>(t31, t17);
    const float t33 = gr::sqrt_(t32);
    const gr::DivShared<float> t34 = gr::div_prep<float>(t33);
  #pragma unroll
    for (long long i3 = 0; i3 < 1LL; ++i3) {
      float acc2[8];
  #pragma unroll
      for (long long i4 = 0; i4 < 16LL; ++i4) {
        float L6[8];
        gr::lds8<float>(L6, reinterpret_cast<const float*>(sst0) + (lf0 + i3) * 132 + 8 * i4);
  #pragma unroll
        for (long long i5 = 0; i5 < 8LL; ++i5) {
          const float t19 = gr::sub<float>(L6[i5], t18);
          const float t35 = gr::div_shared<float>(t19, t34);
          acc2[i5] = (i4 == 0) ? t35 : gr::add<float>(acc2[i5], t35);
        }
      }
      ls1[i3] = gr::leaf_local<float, 8>(acc2);
    }
    const float t36 = gr::lane_tree<gr::OpSum, float, 1>(ls1);
    const float t37 = gr::warp_tree<gr::OpSum, float>(t36, 32);
    if (valid && lr == 0) reinterpret_cast<float*>(static_cast<char*>(p.scratch) + 0)[r] = t37;
  }
  static __device__ __forceinline__ void issue(const Params& p, unsigned char* stage, unsigned long long* bar, const long long g, const int lane) {
    const long long nvalid = (g * 1 + 1 <= NROWS) ? 1 : (NROWS - g * 1);
    if (lane == 0) gr::mbar_arrive_expect_tx(bar, (unsigned)(nvalid * 16384));
    for (int c = lane; c < 32; c += 32) {
      const int qq = c / 32, lf = c % 32;
      if (qq < nvalid) gr::bulk_g2s(stage + 0 + (long long)qq * 16896 + (long long)lf * 528, p.in0 + (g * 1 + qq) * 4096LL + (long long)lf * 128, 512u, bar);
    }
  }
};
extern "C" __global__ void __launch_bounds__(128) gr_region(const K::Params p) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ unsigned long long bars[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { for (int s = 0; s < 2; ++s) gr::mbar_init(&bars[warp * 2 + s], 1); gr::fence_mbar_init(); }
  __syncwarp();
  const long long gw = (long long)blockIdx.x * 4 + warp, nwg = (long long)gridDim.x * 4;
  const long long NG = 65536LL;
  unsigned char* wbase = smem + (long long)warp * 33792;
  for (int s = 0; s < 1; ++s) { const long long g = gw + s * nwg; if (g < NG) K::issue(p, wbase + s * 16896, &bars[warp * 2 + s], g, lane); }
  int it = 0;
  for (long long g = gw; g < NG; g += nwg, ++it) {
    const int s = it % 2;
    {
      const long long gn = g + 1 * nwg;
      const int sn = (it + 1) % 2;
      __syncwarp();
      gr::fence_proxy_async();
      if (gn < NG) K::issue(p, wbase + sn * 16896, &bars[warp * 2 + sn], gn, lane);
    }
    gr::mbar_wait(&bars[warp * 2 + s], (unsigned)((it / 2) & 1));
    K::rows(p, wbase + s * 16896, g, lane);
  }
  if (gr::last_block(p.ticket)) {
    const float v0 = gr::block_tree<gr::OpSum, float>(reinterpret_cast<const float*>(static_cast<const char*>(p.scratch) + 0), K::NROWS, gr::f32_bits(0x00000000u));
    if (threadIdx.x == 0) p.out0[0] = gr::add<float>(gr::f32_bits(0x00000000u), v0);
  }
}
