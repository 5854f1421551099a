// gr_nearest.cuh — certified nearest-centre search for argmin over squared
// distances to a small constant set of centres (k-means assignment, C5).
//
// The user program is NumPy's
//     d = ((P[:, None, :] - C[None]) ** 2).sum(-1);  lab = d.argmin(1)
// whose labels must match np.argmin over NumPy's float32 distances exactly
// (first index on ties, NaN extreme).  Evaluating d as written costs 4 sub,
// 4 mul and 3 add per centre plus the ordered compare.  Here each row instead
// ranks the centres by the expanded distance
//     key_j = (||c'_j||^2 + ||p'||^2) - 2 p'.c'_j     (p' = p - o, c' = c - o)
// one FADD2 and four FFMA2 per centre PAIR, with the centre index written into
// the key's low mantissa bits so that one FMNMX keeps both the best key and
// its index.  The two smallest keys are tracked (m1 < m2, FMNMX3); the label
// is certified when
//     m2 - m1 > 2.1 Dc + e (|m1| + |m2|) + g max(m1 + e |m1| + Dc, 0) + 1e-35
// with Dc = 24 u (||p'||^2 + 2 max_j ||c'_j||^2) bounding the chain's error
// against the exact distance D_j (origin shift 4.06u, ||c'||^2 and ||p'||^2
// roundings 5u, five roundings of terms <= 2R 10u; u = 2^-24), e = 1.01 *
// 2^(BITS-23) the index bits' relative perturbation (x - e|x| is increasing,
// so every key >= m2 bounds its distance below by m2 - e|m2| - Dc), and
// g = 2.1 (D + 2) u > 2.01 gamma_(D+1) NumPy's own rounding of the distances
// (at most D + 1 roundings of non-negative terms: |D^_j - D_j| <= gamma D_j).  Then D^_label < D^_j for
// every other centre: the label IS np.argmin.  A row that fails (near-ties,
// NaN or inf anywhere, magnitudes above 1e37 where the chain could overflow)
// returns false and the caller runs the exact NumPy-order scan for it.
//
// Table layout (written per launch by the region's one-CTA pack kernel from
// the centre leaf, in the constant bank): float2 tab[H + K/2 * S], records
// 16-byte aligned (H, S even) so each is whole LDCU.128 loads,
//   header (H float2): o[0..D-1] (origin, the centres' mean),
//   o[D] = CC = max_j ||c'_j||^2 rounded up (NaN when any centre is not
//   finite: every row then takes the exact scan), o[D+1] = ~MASK (bits);
//   pair jp: tab[H + jp*S + k] = (c'_{2jp,k}, c'_{2jp+1,k}), k < D, and
//   tab[H + jp*S + D] = (||c'_{2jp}||^2, ||c'_{2jp+1}||^2) (double, rounded),
//   tab[H + jp*S + D + 1] = the index pair (2jp, 2jp+1) as integer bits (a
//   uniform operand of the embedding LOP3 instead of a per-key immediate move).
#pragma once

namespace gr {

template <int K, int D>
struct Nearest {
  static_assert(K >= 2 && K % 2 == 0 && K <= 256, "centre count");
  static constexpr int H = (D + 3) / 2 + ((D + 3) / 2) % 2;   // 16-byte aligned records
  static constexpr int S = (D + 2) + (D + 2) % 2;              // float2 per centre pair (even)
  static constexpr int BITS = K <= 2 ? 1 : K <= 4 ? 2 : K <= 8 ? 3 : K <= 16 ? 4 : K <= 32 ? 5 : K <= 64 ? 6 : K <= 128 ? 7 : 8;
  static constexpr unsigned MASK = (1u << BITS) - 1u;
  static constexpr int WORDS = H + K / 2 * S;
};

__device__ __forceinline__ unsigned nn_embed(float v, unsigned keep, unsigned idx) {
  unsigned r;
  // (bits & keep) | idx in one LOP3 (keep held in a register)
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(__float_as_uint(v)), "r"(keep), "r"(idx));
  return r;
}
__device__ __forceinline__ float nn_min3(float a, float b, float c) {
  float r;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

// NPT points at once (each table record loaded once for all of them: the
// uniform loads and moves per point shrink with NPT); ok[i] / label[i] per
// point exactly as the one-point search below.
template <int K, int D, int NPT>
__device__ __forceinline__ void nearest_centre_n(const float (&p)[NPT][D], const float2* __restrict__ tab,
                                                 int (&label)[NPT], bool (&ok)[NPT]) {
  using N = Nearest<K, D>;
  const float* hdr = reinterpret_cast<const float*>(tab);
  float q[NPT][D];
  float pp[NPT];
#pragma unroll
  for (int i = 0; i < NPT; ++i) {
    pp[i] = 0.0f;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const float pk = __fsub_rn(p[i][k], hdr[k]);
      q[i][k] = -2.0f * pk;
      pp[i] = __fmaf_rn(pk, pk, pp[i]);
    }
  }
  // the mask as a register operand (a volatile read of the header word the
  // pack kernel wrote): the LOP3 then takes the index pair as its uniform
  // operand, no per-key index move or LDC
  const unsigned keep = *reinterpret_cast<const volatile unsigned*>(hdr + D + 1);
  const float inf = __int_as_float(0x7f800000);
  float m1[NPT], m2[NPT];
#pragma unroll
  for (int i = 0; i < NPT; ++i) m1[i] = m2[i] = inf;
#pragma unroll
  for (int jp = 0; jp < K / 2; ++jp) {
    const float2* c = tab + N::H + jp * N::S;
    // the record's index pair (2jp, 2jp+1) arrives with its centre words
    const float2 ix = c[D + 1];
#pragma unroll
    for (int i = 0; i < NPT; ++i) {
      float2 acc = __fadd2_rn(make_float2(pp[i], pp[i]), c[D]);
#pragma unroll
      for (int k = 0; k < D; ++k) acc = __ffma2_rn(make_float2(q[i][k], q[i][k]), c[k], acc);
      const float k0 = __uint_as_float(nn_embed(acc.x, keep, __float_as_uint(ix.x)));
      const float k1 = __uint_as_float(nn_embed(acc.y, keep, __float_as_uint(ix.y)));
      const float lo = fminf(k0, k1), hi = fmaxf(k0, k1);
      m2[i] = nn_min3(m2[i], fmaxf(m1[i], lo), hi);
      m1[i] = fminf(m1[i], lo);
    }
  }
  constexpr float E = 1.01f * (float)(1u << N::BITS) * 1.1920928955078125e-07f;
  // NumPy's own rounding: a term passes through at most D + 1 roundings (sub,
  // square, the D - 1 adds of the sequential fold; 5 for the n == 8 tree),
  // |D^_j - D_j| <= gamma_(D+1) D_j; 2.1 (D + 2) u covers 2.01 gamma_(D+1)
  constexpr float NP = 2.1f * (D + 2) * 5.9604644775390625e-08f;
#pragma unroll
  for (int i = 0; i < NPT; ++i) {
    label[i] = (int)(__float_as_uint(m1[i]) & N::MASK);
    const float R = pp[i] + 2.0f * hdr[D];
    const float dc = 24.0f * 5.9604644775390625e-08f * R;
    const float a1 = fabsf(m1[i]), a2 = fabsf(m2[i]);
    const float thr = 2.1f * dc + E * (a1 + a2) + NP * fmaxf(m1[i] + E * a1 + dc, 0.0f) + 1e-35f;
    // NaN anywhere (p, centres, keys) makes a comparison false: exact scan
    ok[i] = R < 1e37f && m2[i] - m1[i] > thr;
  }
}

template <int K, int D>
__device__ __forceinline__ bool nearest_centre(const float (&p)[D], const float2* __restrict__ tab, int& label) {
  float pa[1][D];
#pragma unroll
  for (int k = 0; k < D; ++k) pa[0][k] = p[k];
  int l[1];
  bool ok[1];
  nearest_centre_n<K, D, 1>(pa, tab, l, ok);
  label = l[0];
  return ok[0];
}

// np.argmin over NumPy's float32 distances, exactly: d_j = ((p0-c0)^2 +
// (p1-c1)^2) + ... (sub, square, then a left fold over the D < 8 terms —
// NumPy's pairwise sum is sequential below 8 elements; its 0.0 start changes
// only the sign of a zero sum, which no compare sees), first index on ties,
// the first NaN wins.  Out of line: the rows that need it are rare, and its
// registers stay out of the hot loop's allocation.
template <int D> struct Point { float v[D]; };   // passed by value: registers, no stack copy

template <int K, int D>
__device__ __noinline__ int nearest_exact_v(const Point<D> pt, const float* __restrict__ c) {
  const float* p = pt.v;
  static_assert(D <= 8, "NumPy's 8-accumulator block for 8 <= n <= 128 is written out for n == 8 only");
  float best = 0.0f;
  int bi = 0;
  for (int j = 0; j < K; ++j) {
    float sq[D];
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const float t = __fsub_rn(p[k], c[j * D + k]);
      sq[k] = __fmul_rn(t, t);
    }
    float d;
    if constexpr (D == 8) {
      // n == 8: eight accumulators, combined as a fixed tree
      d = __fadd_rn(__fadd_rn(__fadd_rn(sq[0], sq[1]), __fadd_rn(sq[2], sq[3])),
                    __fadd_rn(__fadd_rn(sq[4], sq[5]), __fadd_rn(sq[6], sq[7])));
    } else {
      d = sq[0];
#pragma unroll
      for (int k = 1; k < D; ++k) d = __fadd_rn(d, sq[k]);
    }
    if (d != d) return j;
    if (j == 0 || d < best) { best = d; bi = j; }
  }
  return bi;
}

template <int K, int D>
__device__ __forceinline__ int nearest_exact(const float (&p)[D], const float* __restrict__ c) {
  Point<D> pt;
#pragma unroll
  for (int k = 0; k < D; ++k) pt.v[k] = p[k];
  return nearest_exact_v<K, D>(pt, c);
}

// Pack kernel body (one CTA): origin, CC and the pair table from the row-major
// [K][D] centre leaf.
template <int K, int D>
__device__ __forceinline__ void nearest_pack(const float* __restrict__ src, float2* __restrict__ tab) {
  using N = Nearest<K, D>;
  __shared__ double o[D];
  __shared__ double cc[K];
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  if (threadIdx.x < D) {
    double s = 0.0;
    for (int j = 0; j < K; ++j) s += (double)src[j * D + threadIdx.x];
    o[threadIdx.x] = (double)(float)(s / K);
  }
  __syncthreads();
  for (int j = threadIdx.x; j < K; j += blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < D; ++k) {
      const float v = src[j * D + k];
      if (!isfinite(v)) bad = 1;
      const float cp = __fsub_rn(v, (float)o[k]);
      s += (double)cp * (double)cp;
      reinterpret_cast<float*>(tab + N::H + (j / 2) * N::S + k)[j & 1] = cp;
    }
    cc[j] = s;
    reinterpret_cast<float*>(tab + N::H + (j / 2) * N::S + D)[j & 1] = (float)s;
    reinterpret_cast<unsigned*>(tab + N::H + (j / 2) * N::S + D + 1)[j & 1] = (unsigned)j;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int j = 0; j < K; ++j) m = cc[j] > m ? cc[j] : m;
    float* hdr = reinterpret_cast<float*>(tab);
    for (int k = 0; k < D; ++k) hdr[k] = (float)o[k];
    hdr[D] = bad ? __int_as_float(0x7fffffff) : __double2float_ru(m * (1.0 + 1e-6));
    reinterpret_cast<unsigned*>(hdr)[D + 1] = ~N::MASK;
  }
}

}  // namespace gr
