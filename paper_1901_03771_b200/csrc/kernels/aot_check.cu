// aot_check.cu — build-time instantiation of every hand-written template.
//
// NVRTC instantiates the skeletons per region at run time; this translation
// unit instantiates them once with nvcc for sm_100a at build time
// (__graft_entry__.build()), over all element types, so a template error is a
// build error, and `cuobjdump -sass aot_check.cubin` shows the code shape of
// each skeleton without a GPU.
#include "gr_ops.cuh"
#include "gr_mem.cuh"
#include "gr_map.cuh"
#include "gr_reduce.cuh"
#include "gr_tma.cuh"
#include "gr_pair.cuh"

// reductions, packed pairs, bulk copies: one instantiation each
extern "C" __global__ void aot_reduce(const float* x, float* o, unsigned* ticket, long long* oi) {
  auto f = [&](long long i) -> float { return x[i]; };
  float s = gr::pairwise<float, 4096>(f, 0) + gr::pairwise<float, 1000>(f, 0);
  float acc[4] = {x[0], x[1], x[2], x[3]};
  __shared__ float sh[8];
  s += gr::row_sum<float, 4, 2, 64>(acc, sh, 0) + gr::row_tree<gr::OpMax, float, 64>(s, sh, 0);
  float ls[4] = {s, s, s, s};
  s += gr::lane_tree<gr::OpSum, float, 4>(ls) + gr::warp_tree<gr::OpSum, float>(s, 8);
  long long bi = gr::warp_arg<true, float>(s, threadIdx.x, 32);
  if (gr::last_block(ticket)) {
    o[0] = gr::block_tree<gr::OpSum, float>(o + 1, 1000, 0.0f);
    oi[0] = gr::block_arg<true, float>(o + 1, oi + 1, 1000) + bi;
  }
  const gr::DivShared<float> d = gr::div_prep<float>(s);
  o[threadIdx.x + 2000] = gr::div_shared<float>(x[threadIdx.x], d);
}

extern "C" __global__ void aot_pair(const float4* x, float4* o) {
  const float4 a = x[threadIdx.x];
  const gr::f2 p = gr::pk(a.x, a.y), q = gr::pk(a.z, a.w);
  const gr::f2 r = gr::p2::add(gr::p2::exp_(p), gr::p2::mul(gr::p2::log_(q), gr::p2::erf_(gr::p2::div(p, q))));
  o[threadIdx.x] = make_float4(gr::lo(r), gr::hi(r), gr::lo(gr::p2::sqrt_(q)), gr::hi(gr::p2::select(gr::p2::lt(p, q), p, q)));
}

extern "C" __global__ void aot_bulk(const float* x, float* o) {
  __shared__ __align__(128) float buf[128];
  __shared__ unsigned long long bar;
  if (threadIdx.x == 0) {
    gr::mbar_init(&bar, 1);
    gr::fence_mbar_init();
    gr::mbar_arrive_expect_tx(&bar, 512);
    gr::bulk_g2s(buf, x, 512, &bar);
    gr::prefetch_l2(x + 128, 512);
  }
  __syncthreads();
  gr::mbar_wait(&bar, 0);
  float v[8];
  gr::lds8<float>(v, buf + 8 * (threadIdx.x % 16));
  gr::st8<float>(o + 8 * threadIdx.x, v);
}


template <class T> __device__ T all_ops(T a, T b, bool c) {
  T r = gr::add<T>(a, b);
  r = gr::sub<T>(r, gr::mul<T>(a, b));
  r = gr::maximum<T>(r, gr::minimum<T>(a, b));
  r = gr::select<T>(gr::lt<T>(a, b) && gr::ge<T>(a, b) && c, r, gr::neg<T>(r));
  r = gr::add<T>(r, gr::floordiv<T>(a, b));
  r = gr::add<T>(r, gr::mod<T>(a, b));
  r = gr::add<T>(r, gr::pow_<T>(a, b));
  r = gr::add<T>(r, gr::abs_(a));
  return r;
}
template <class T> __device__ T float_ops(T a) {
  return gr::exp_(a) + gr::log_(a) + gr::sqrt_(a) + gr::erf_(a) + gr::tanh_(a) + gr::sin_(a) + gr::cos_(a) +
         gr::floor_(a) + gr::ceil_(a) + gr::div<T>(a, a);
}

// A Listing-1-shaped map region over f64, instantiated into the skeleton.
struct KCheck {
  struct Params {
    const double* __restrict__ in0;
    const double* __restrict__ in1;
    const double* __restrict__ in2;
    double* __restrict__ out0;
    void* __restrict__ scratch;
  };
  static constexpr long long NGROUPS = 1 << 23;
  static constexpr int U = 2;
  static constexpr bool TAIL = false;
  template <int N> static __device__ __forceinline__ void group(const Params& p, long long g0, long long stride) {
    double a[N][2], w[N][2], b[N][2];
#pragma unroll
    for (int u = 0; u < N; ++u) {
      const int lin = (int)(g0 + u * stride) * 2;
      gr::ldv<double, 2>(a[u], p.in0 + lin);
      gr::ldv<double, 2>(w[u], p.in1 + lin);
      gr::ldv<double, 2>(b[u], p.in2 + lin);
    }
#pragma unroll
    for (int u = 0; u < N; ++u) {
      const int lin = (int)(g0 + u * stride) * 2;
      double o[2];
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        double x = gr::mul<double>(a[u][v], w[u][v]);
        double y = gr::mul<double>(b[u][v], w[u][v]);
        o[v] = gr::add<double>(gr::add<double>(gr::mul<double>(gr::mul<double>(x, y), w[u][v]), a[u][v]), b[u][v]);
      }
      gr::stv<double, 2>(p.out0 + lin, o);
    }
  }
  static __device__ __forceinline__ void tail(const Params&) {}
};

extern "C" __global__ void aot_map_f64(const KCheck::Params p) { gr::map_kernel<KCheck>(p); }

extern "C" __global__ void aot_ops(const float* f, const double* d, const int* i, const long long* l,
                                   const bool* b, float* of, double* od, int* oi, long long* ol, bool* ob) {
  int t = threadIdx.x;
  of[t] = all_ops<float>(f[t], f[t + 1], b[t]) + float_ops<float>(f[t]) + gr::cast<float, long long>(l[t]);
  od[t] = all_ops<double>(d[t], d[t + 1], b[t]) + float_ops<double>(d[t]) + gr::cast<double, int>(i[t]);
  oi[t] = all_ops<int>(i[t], i[t + 1], b[t]) + gr::cast<int, float>(f[t]) + gr::cast<int, double>(d[t]);
  ol[t] = all_ops<long long>(l[t], l[t + 1], b[t]) + gr::cast<long long, double>(d[t]);
  ob[t] = gr::land<float>(f[t], f[t + 1]) || gr::lor<bool>(b[t], b[t + 1]) || gr::cast<bool, double>(d[t]) ||
          gr::isnan_<double>(d[t]) || gr::lnot<int>(i[t]);
}
