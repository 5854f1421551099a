#define GR_LDG gr_generic_ld
template <class X> __device__ __forceinline__ X gr_generic_ld(const X* p) { return *p; }
#include "gr_ops.cuh"
#include "gr_mem.cuh"
#include "gr_pair.cuh"

#include "gr_map.cuh"

struct K {
  struct Params {
    const float* __restrict__ in0;
    const float* __restrict__ in1;
    const float* __restrict__ in2;
    float* __restrict__ out0;
    float* __restrict__ out1;
    void* __restrict__ scratch;
  };
  static constexpr long long NGROUPS = 67108864LL;
  static constexpr int U = 1;
  static constexpr bool TAIL = false;
  template <int N> static __device__ __forceinline__ void group(const Params& p, long long g0, long long stride) {
    const float k2 = gr::f32_bits(0x3f000000u);  // 0.5
    const float k3 = gr::f32_bits(0x3f800000u);  // 1.0
    const float k7 = gr::f32_bits(0x3d851eb8u);  // 0.06499999761581421
    const gr::f2 t9 = gr::splat(k7);
    const float k12 = gr::f32_bits(0x3e99999au);  // 0.30000001192092896
    const gr::f2 t14 = gr::splat(k12);
    const float k17 = gr::f32_bits(0x3f3504f3u);  // 0.7071067690849304
    const gr::f2 t18 = gr::splat(k17);
    const gr::f2 t21 = gr::splat(k3);
    const gr::f2 t23 = gr::splat(k2);
    const float k26 = gr::f32_bits(0xbca3d70au);  // -0.019999999552965164
    const gr::f2 t27 = gr::splat(k26);
    float L1[N][4];
    float L4[N][4];
    float L8[N][4];
  #pragma unroll
    for (int u = 0; u < N; ++u) {
      const int lin = (int)(g0 + u * stride) * 4; (void)lin;
      gr::ldv<float, 4>(L1[u], p.in0 + (lin));
      gr::ldv<float, 4>(L4[u], p.in1 + (lin));
      gr::ldv<float, 4>(L8[u], p.in2 + (lin));
    }
  #pragma unroll
    for (int u = 0; u < N; ++u) {
      const int lin = (int)(g0 + u * stride) * 4; (void)lin;
      float o0[4];
      float o1[4];
  #pragma unroll
      for (int v = 0; v < 2; ++v) {
        const gr::f2 t5 = gr::p2::div(gr::pk(L1[u][2 * v], L1[u][2 * v + 1]), gr::pk(L4[u][2 * v], L4[u][2 * v + 1]));
        const gr::f2 t6 = gr::p2::log_(t5);
        const gr::f2 t10 = gr::p2::mul_nc(t9, gr::pk(L8[u][2 * v], L8[u][2 * v + 1]));
        const gr::f2 t11 = gr::p2::add(t6, t10);
        const gr::f2 t13 = gr::p2::sqrt_(gr::pk(L8[u][2 * v], L8[u][2 * v + 1]));
        const gr::f2 t15 = gr::p2::mul_nc(t14, t13);
        const gr::f2 t16 = gr::p2::div(t11, t15);
        const gr::f2 t19 = gr::p2::mul(t16, t18);
        const gr::f2 t20 = gr::p2::erf_(t19);
        const gr::f2 t22 = gr::p2::add(t21, t20);
        const gr::f2 t24 = gr::p2::mul_nc(t23, t22);
        const gr::f2 t25 = gr::p2::mul_nc(gr::pk(L1[u][2 * v], L1[u][2 * v + 1]), t24);
        const gr::f2 t28 = gr::p2::mul(t27, gr::pk(L8[u][2 * v], L8[u][2 * v + 1]));
        const gr::f2 t29 = gr::p2::exp_(t28);
        const gr::f2 t30 = gr::p2::mul(gr::pk(L4[u][2 * v], L4[u][2 * v + 1]), t29);
        const gr::f2 t31 = gr::p2::sub(t16, t15);
        const gr::f2 t32 = gr::p2::mul(t31, t18);
        const gr::f2 t33 = gr::p2::erf_(t32);
        const gr::f2 t34 = gr::p2::add(t21, t33);
        const gr::f2 t35 = gr::p2::mul_nc(t23, t34);
        const gr::f2 t36 = gr::p2::mul_nc(t30, t35);
        const gr::f2 t37 = gr::p2::sub(t25, t36);
        const gr::f2 t38 = gr::p2::sub(t21, t35);
        const gr::f2 t39 = gr::p2::mul_nc(t30, t38);
        const gr::f2 t40 = gr::p2::sub(t21, t24);
        const gr::f2 t41 = gr::p2::mul_nc(gr::pk(L1[u][2 * v], L1[u][2 * v + 1]), t40);
        const gr::f2 t42 = gr::p2::sub(t39, t41);
        o0[2 * v] = gr::lo(t37); o0[2 * v + 1] = gr::hi(t37);
        o1[2 * v] = gr::lo(t42); o1[2 * v + 1] = gr::hi(t42);
      }
      gr::stv<float, 4>(p.out0 + lin, o0);
      gr::stv<float, 4>(p.out1 + lin, o1);
    }
  }
  static __device__ __forceinline__ void tail(const Params& p) {
  }
};
#include "gr_tma.cuh"
extern "C" __global__ void __launch_bounds__(256) gr_region(const K::Params p) {
  constexpr int S = 6, NL = 3, TILE = 1024;
  extern __shared__ __align__(128) unsigned char smraw[];
  float* sm = reinterpret_cast<float*>(smraw);
  __shared__ __align__(8) unsigned long long full[S];
  const long long ntiles = K::NGROUPS / 256;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) gr::mbar_init(&full[s], 1);
    gr::fence_mbar_init();
  }
  __syncthreads();
  const float* src[NL] = {p.in0, p.in1, p.in2};
  auto issue = [&](long long i) {
    const long long t = blockIdx.x + i * gridDim.x;
    if (t >= ntiles) return;
    const int s = (int)(i % S);
    gr::mbar_arrive_expect_tx(&full[s], NL * TILE * sizeof(float));
#pragma unroll
    for (int l = 0; l < NL; ++l) gr::bulk_g2s(sm + (s * NL + l) * TILE, src[l] + t * TILE, TILE * sizeof(float), &full[s]);
  };
  if (threadIdx.x == 0) for (int i = 0; i < S - 1; ++i) issue(i);
  for (long long i = 0;; ++i) {
    const long long t = blockIdx.x + i * gridDim.x;
    if (t >= ntiles) break;
    if (threadIdx.x == 0) issue(i + S - 1);
    const int s = (int)(i % S);
    gr::mbar_wait(&full[s], (unsigned)((i / S) & 1));
    K::Params q = p;
    q.in0 = sm + (s * NL + 0) * TILE - t * TILE;
    q.in1 = sm + (s * NL + 1) * TILE - t * TILE;
    q.in2 = sm + (s * NL + 2) * TILE - t * TILE;
    K::template group<1>(q, t * 256 + threadIdx.x, 0);
    __syncthreads();
  }
}
