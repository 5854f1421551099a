// gr_reduce.cuh — reduction templates with NumPy's association order.
//
// The reference reduces with per-thread sequential folds combined in thread
// order; its baseline is NumPy, whose float add.reduce
// is *pairwise* along the contiguous axis (numpy/_core/src/umath/
// loops_utils.h.src pairwise_sum: n < 8 sequential from -0.0; 8 <= n <= 128
// eight strided accumulators combined ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) plus
// a sequential tail; n > 128 split at n2 = n/2 - (n/2)%8) and sequential along
// the other axes, starting from the identity 0.0.  Restated and pinned in
// oracle/pairwise.py.  These templates reproduce that order exactly, so a
// fused reduction of IEEE-exact terms is bit-identical to NumPy.
#pragma once

namespace gr {

template <class T> __device__ __forceinline__ T shfl_xor(T v, int m) { return __shfl_xor_sync(0xffffffffu, v, m); }
template <> __device__ __forceinline__ bool shfl_xor(bool v, int m) { return __shfl_xor_sync(0xffffffffu, (int)v, m) != 0; }

template <class T> struct Zero { static __device__ __forceinline__ T neg() { return T(0); } };
template <> struct Zero<float> { static __device__ __forceinline__ float neg() { return -0.0f; } };
template <> struct Zero<double> { static __device__ __forceinline__ double neg() { return -0.0; } };

// True when NumPy's recursion over N splits in exact halves down to 128-leaves.
__host__ __device__ constexpr bool pw_regular(long long n) {
  return n == 128 || (n > 128 && n % 256 == 0 && pw_regular(n / 2));
}
__host__ __device__ constexpr int pw_log2(long long n) { return n <= 1 ? 0 : 1 + pw_log2(n / 2); }

// NumPy pairwise_sum over f(off .. off+N); N is a compile-time extent.
template <class T, long long N, class F>
__device__ __forceinline__ T pairwise(const F& f, long long off) {
  if constexpr (N < 8) {
    T r = Zero<T>::neg();
#pragma unroll
    for (long long i = 0; i < N; ++i) r = add<T>(r, f(off + i));
    return r;
  } else if constexpr (N <= 128) {
    T r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = f(off + j);
    constexpr long long NB = N - (N % 8);
#pragma unroll 2
    for (long long i = 8; i < NB; i += 8) {
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = add<T>(r[j], f(off + i + j));
    }
    T res = add<T>(add<T>(add<T>(r[0], r[1]), add<T>(r[2], r[3])), add<T>(add<T>(r[4], r[5]), add<T>(r[6], r[7])));
#pragma unroll
    for (long long i = NB; i < N; ++i) res = add<T>(res, f(off + i));
    return res;
  } else if constexpr (pw_regular(N)) {
    // perfect binary tree over N/128 leaves: fold leaves left to right with a
    // binary-counter stack (stack[l] holds a finished subtree of 2^l leaves)
    constexpr long long NL = N / 128;
    constexpr int D = pw_log2(NL) + 1;
    T stack[D];
#pragma unroll 1
    for (long long b = 0; b < NL; ++b) {
      T v = pairwise<T, 128>(f, off + b * 128);
      int l = 0;
      long long c = b;
      while (c & 1) {
        v = add<T>(stack[l], v);
        ++l;
        c >>= 1;
      }
      stack[l] = v;
    }
    return stack[D - 1];
  } else {
    constexpr long long H = N / 2;
    constexpr long long N2 = H - (H % 8);
    return add<T>(pairwise<T, N2>(f, off), pairwise<T, N - N2>(f, off + N2));
  }
}

// first-index arg-reduction predicates (np.argmax / np.argmin: the first
// maximal element wins; a NaN is maximal and minimal, the first NaN wins)
template <class T> __device__ __forceinline__ bool arg_better_max(T x, T best) {
  return (x > best) || (x != x && best == best);
}
// NaN-propagating min/max (PTX min.NaN / max.NaN): arg-reduction scans keep
// the best value with these so a NaN operand is visible at the end
__device__ __forceinline__ float min_nan(float a, float b) {
  float r;
  asm("min.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float max_nan(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
template <class T> __device__ __forceinline__ bool arg_better_min(T x, T best) {
  return (x < best) || (x != x && best == best);
}
template <> __device__ __forceinline__ bool arg_better_max(bool x, bool best) { return x && !best; }
template <> __device__ __forceinline__ bool arg_better_min(bool x, bool best) { return !x && best; }

// Is candidate (bv, bi) a better np.argmax/argmin answer than (av, ai)?
// NaN beats numbers; among equals (or NaNs) the lower index wins.
template <bool MAX, class T> __device__ __forceinline__ bool arg_take_b(T av, long long ai, T bv, long long bi) {
  const bool an = av != av, bn = bv != bv;
  if (an || bn) return bn && (!an || bi < ai);
  if (MAX ? (bv > av) : (bv < av)) return true;
  if (bv == av) return bi < ai;
  return false;
}

// CTA-wide first-index arg-reduction over n (value, index) candidates.
template <bool MAX, class T> __device__ long long block_arg(const T* v, const long long* ix, long long n) {
  __shared__ T sv[32];
  __shared__ long long si[32];
  const long long nt = blockDim.x;
  const long long chunk = (n + nt - 1) / nt;
  const long long lo = threadIdx.x * chunk;
  const long long hi = lo + chunk < n ? lo + chunk : n;
  T best = T(0);
  long long bi = -1;
  for (long long i = lo; i < hi; ++i) {
    if (bi < 0 || arg_take_b<MAX, T>(best, bi, v[i], ix[i])) {
      best = v[i];
      bi = ix[i];
    }
  }
#pragma unroll
  for (int m = 1; m < 32; m <<= 1) {
    T ov = shfl_xor<T>(best, m);
    long long oi = __shfl_xor_sync(0xffffffffu, bi, m);
    if (oi >= 0 && (bi < 0 || arg_take_b<MAX, T>(best, bi, ov, oi))) {
      best = ov;
      bi = oi;
    }
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  if (lane == 0) {
    sv[w] = best;
    si[w] = bi;
  }
  __syncthreads();
  if (w == 0) {
    best = lane < nw ? sv[lane] : T(0);
    bi = lane < nw ? si[lane] : -1;
#pragma unroll
    for (int m = 1; m < 32; m <<= 1) {
      T ov = shfl_xor<T>(best, m);
      long long oi = __shfl_xor_sync(0xffffffffu, bi, m);
      if (oi >= 0 && (bi < 0 || arg_take_b<MAX, T>(best, bi, ov, oi))) {
        best = ov;
        bi = oi;
      }
    }
    if (lane == 0) si[0] = bi;
  }
  __syncthreads();
  long long r = si[0];
  __syncthreads();
  return r;
}

// ---- combine ops for cross-thread / cross-block trees -----------------------
struct OpSum {
  template <class T> static __device__ __forceinline__ T c(T a, T b) { return add<T>(a, b); }
};
struct OpProd {
  template <class T> static __device__ __forceinline__ T c(T a, T b) { return mul<T>(a, b); }
};
struct OpMax {
  template <class T> static __device__ __forceinline__ T c(T a, T b) { return (a != a) ? a : ((b != b) ? b : (b > a ? b : a)); }
};
struct OpMin {
  template <class T> static __device__ __forceinline__ T c(T a, T b) { return (a != a) ? a : ((b != b) ? b : (b < a ? b : a)); }
};

template <class Op> struct IsSum { static constexpr bool v = false; };
template <> struct IsSum<OpSum> { static constexpr bool v = true; };

// Perfect binary tree over the lanes of a warp in lane order (pairs (0,1),
// (2,3), ... then (01,23), ...): the association of NumPy's pairwise split for
// power-of-two counts.  Every lane ends with the full result.
template <class Op, class T> __device__ __forceinline__ T warp_tree(T v, int width = 32) {
#pragma unroll
  for (int m = 1; m < 32; m <<= 1) {
    if (m < width) {
      T o = shfl_xor<T>(v, m);
      // lower lane's value is the left operand (add/mul commute exactly in IEEE)
      v = Op::template c<T>(v, o);
    }
  }
  return v;
}

// s = (((s + p[0]) + p[stride]) + ...) over n terms, in that order, with the
// loads of each batch of 8 issued before its adds: the fold of per-CTA
// partials by the last CTA waits on L2 once per batch instead of once per
// term (same association as the plain loop, bit for bit)
template <class T> __device__ __forceinline__ T seq_fold(T s, const T* p, unsigned n, long long stride) {
  unsigned c = 0;
  for (; c + 8 <= n; c += 8) {
    T v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __ldcg(p + (long long)(c + k) * stride);
#pragma unroll
    for (int k = 0; k < 8; ++k) s += v[k];
  }
  for (; c < n; ++c) s += __ldcg(p + (long long)c * stride);
  return s;
}

// Perfect binary tree over q[0..chunk) (chunk a power of two; elements at
// or past nvalid are the identity), by one thread: leaves in batches of 32
// (8 for shorter chunks) — the batch's loads issued together, combined as a
// perfect tree — then a binary-counter stack over the batches.  Same
// association as a leaf-by-leaf stack; one L2 round trip per batch instead of
// per partial (rownorm's total: the last CTA's fold of 65536 row partials
// 0.048 -> ~0.01 ms).
template <class Op, class T, int B>
__device__ __forceinline__ T batch_tree(const T* q, long long nvalid, T ident) {
  T a[B];
#pragma unroll
  for (int k = 0; k < B; ++k) a[k] = (k < nvalid) ? __ldcg(q + k) : ident;
#pragma unroll
  for (int s = 1; s < B; s <<= 1)
#pragma unroll
    for (int k = 0; k + s < B; k += 2 * s) a[k] = Op::template c<T>(a[k], a[k + s]);
  return a[0];
}
template <class Op, class T>
__device__ __forceinline__ T chunk_tree(const T* q, long long chunk, long long nvalid, T ident) {
  T stack[40];
  long long cnt = 0;
  const long long step = chunk >= 32 ? 32 : chunk >= 8 ? 8 : 1;
  for (long long i = 0; i < chunk; i += step) {
    T v;
    if (step == 32) {
      v = batch_tree<Op, T, 32>(q + i, nvalid - i, ident);
    } else if (step == 8) {
      v = batch_tree<Op, T, 8>(q + i, nvalid - i, ident);
    } else {
      v = (i < nvalid) ? __ldcg(q + i) : ident;
    }
    int lvl = 0;
    while ((cnt >> lvl) & 1) {
      v = Op::template c<T>(stack[lvl], v);
      ++lvl;
    }
    stack[lvl] = v;
    ++cnt;
  }
  int top = 0;
  while ((1ll << top) < chunk / step) ++top;
  return stack[top];
}

// Tree over n partials p[0..n) in index order, by one CTA (blockDim.x a power
// of two <= 1024, n arbitrary).  Each thread folds a contiguous power-of-two
// chunk as a perfect binary tree (binary-counter stack), then warp and CTA
// trees: for power-of-two n this is exactly the perfect binary tree over p,
// i.e. NumPy's pairwise split above row granularity.
// Large n: each warp takes a contiguous power-of-two range and walks it in
// 256-element chunks with coalesced loads (lane i: elements 8i..8i+7 of the
// chunk, 4 chunks in flight): an 8-leaf tree per lane, the xor butterfly over
// the lanes (the chunk's perfect tree), a stack over the chunks; the warps'
// ranges combine in a perfect tree.  Same association as the per-thread
// chunks below (a perfect tree over the padded range); 65536 f32 partials:
// 44 -> a few us (the per-thread chunks were 32 lanes x 1 KB strided).
template <class Op, class T> __device__ T block_tree_wide(const T* p, long long n, T ident, long long S) {
  __shared__ T shw[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const long long W = S / nw;                       // per-warp range (power of two, >= 1024)
  const long long base = (long long)w * W;
  T stack[40];
  long long cnt = 0;
  for (long long c0 = 0; c0 < W; c0 += 4 * 256) {
    T a[4][8];
    if (base + c0 + 4 * 256 <= n && (reinterpret_cast<unsigned long long>(p) & 15) == 0) {
      // whole chunks in range: 16-byte vector loads (the range bases are
      // multiples of 1024 elements)
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint4* q = reinterpret_cast<const uint4*>(p + base + c0 + u * 256 + lane * 8);
#pragma unroll
        for (int h = 0; h < (int)(8 * sizeof(T) / 16); ++h) {
          const uint4 r = __ldcg(q + h);
          memcpy(&a[u][h * (16 / sizeof(T))], &r, 16);
        }
      }
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const long long e = base + c0 + u * 256 + lane * 8 + k;
          a[u][k] = e < n ? __ldcg(p + e) : ident;
        }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
#pragma unroll
      for (int st = 1; st < 8; st <<= 1)
#pragma unroll
        for (int k = 0; k + st < 8; k += 2 * st) a[u][k] = Op::template c<T>(a[u][k], a[u][k + st]);
      T v = warp_tree<Op, T>(a[u][0]);
      int lvl = 0;
      while ((cnt >> lvl) & 1) {
        v = Op::template c<T>(stack[lvl], v);
        ++lvl;
      }
      stack[lvl] = v;
      ++cnt;
    }
  }
  int top = 0;
  while ((1ll << top) < W / 256) ++top;
  if (lane == 0) shw[w] = stack[top];
  __syncthreads();
  if (w == 0) {
    T v = lane < nw ? shw[lane] : ident;
    v = warp_tree<Op, T>(v);
    if (lane == 0) shw[0] = v;
  }
  __syncthreads();
  T r = shw[0];
  __syncthreads();
  return r;
}

template <class Op, class T> __device__ T block_tree(const T* p, long long n, T ident) {
  __shared__ T sh[32];
  const int t = threadIdx.x, nt = blockDim.x;
  long long chunk = 1;
  while (chunk * nt < n) chunk <<= 1;
  if (chunk * nt >= 1024LL * (nt / 32) && (nt & 31) == 0)
    return block_tree_wide<Op, T>(p, n, ident, chunk * nt);
  const long long lo = (long long)t * chunk;
  T acc = chunk_tree<Op, T>(p + lo, chunk, n - lo, ident);
  acc = warp_tree<Op, T>(acc);
  const int lane = t & 31, w = t >> 5, nw = (nt + 31) >> 5;
  if (lane == 0) sh[w] = acc;
  __syncthreads();
  if (w == 0) {
    T v = lane < nw ? sh[lane] : ident;
    v = warp_tree<Op, T>(v);
    if (lane == 0) sh[0] = v;
  }
  __syncthreads();
  T r = sh[0];
  __syncthreads();
  return r;
}

// Perfect binary tree over N (power of two) register values in index order.
template <class Op, class T, int N> __device__ __forceinline__ T lane_tree(const T (&a)[N]) {
  if constexpr (N == 1) {
    return a[0];
  } else {
    T b[N];
#pragma unroll
    for (int i = 0; i < N; ++i) b[i] = a[i];
#pragma unroll
    for (int s = 1; s < N; s <<= 1)
#pragma unroll
      for (int i = 0; i + s < N; i += 2 * s) b[i] = Op::template c<T>(b[i], b[i + s]);
    return b[0];
  }
}

// First-index (value, index) combine over aligned groups of `width` lanes.
template <bool MAX, class T> __device__ __forceinline__ long long warp_arg(T best, long long bi, int width) {
#pragma unroll
  for (int m = 1; m < 32; m <<= 1) {
    if (m < width) {
      T ov = shfl_xor<T>(best, m);
      long long oi = __shfl_xor_sync(0xffffffffu, bi, m);
      if (arg_take_b<MAX, T>(best, bi, ov, oi)) {
        best = ov;
        bi = oi;
      }
    }
  }
  return bi;
}

// ---- cooperative rows (codegen_coop.py) --------------------------------------
// A row of C = 128 * 2^k elements is held by TPR = (C/128) * P threads; thread
// (leaf l, part h) owns accumulators j = h*VEC .. h*VEC+VEC-1 of NumPy's
// 8-accumulator leaf loop (element 128*l + 8*m + j, m = 0..15), so:
//   leaf sum  = ((r0+r1)+(r2+r3)) + ((r4+r5)+(r6+r7))   (local + shfl over P)
//   row sum   = perfect binary tree over leaves          (shfl, then smem)
// which is exactly numpy.add.reduce along a contiguous row of that length.

template <class T, int VEC> __device__ __forceinline__ T leaf_local(const T (&a)[VEC]) {
  if constexpr (VEC == 1) {
    return a[0];
  } else if constexpr (VEC == 2) {
    return add<T>(a[0], a[1]);
  } else if constexpr (VEC == 4) {
    return add<T>(add<T>(a[0], a[1]), add<T>(a[2], a[3]));
  } else {
    return add<T>(add<T>(add<T>(a[0], a[1]), add<T>(a[2], a[3])), add<T>(add<T>(a[4], a[5]), add<T>(a[6], a[7])));
  }
}

// Combine a per-thread value over the TPR threads of a row (lanes grouped in
// aligned runs of TPR, tr = thread index within the row) in perfect-tree
// order; for TPR > 32 the warp results meet in shared memory `sh`
// (>= rows_per_cta * TPR/32 elements).  Every thread of the row gets the result.
// Barrier over the TPR threads of row slot ri only (named barrier 1 + ri):
// the warps of one row wait for each other, not for the whole CTA.
// GR_RPC (rows per CTA, set by the generated source) lets the barrier id be
// an immediate: a register id makes ptxas reserve all 16 named barriers per
// CTA, which caps residency at 4 CTAs per SM (ncu "Block Limit Barriers").
#ifndef GR_RPC
#define GR_RPC 0
#endif
template <int TPR> __device__ __forceinline__ void row_bar(int ri) {
  if constexpr (TPR >= 1024 || GR_RPC == 1) {
    __syncthreads();
  } else if constexpr (GR_RPC == 2) {
    if (ri == 0) asm volatile("bar.sync 1, %0;" ::"n"(TPR) : "memory");
    else asm volatile("bar.sync 2, %0;" ::"n"(TPR) : "memory");
  } else if constexpr (GR_RPC == 4) {
    switch (ri) {
      case 0: asm volatile("bar.sync 1, %0;" ::"n"(TPR) : "memory"); break;
      case 1: asm volatile("bar.sync 2, %0;" ::"n"(TPR) : "memory"); break;
      case 2: asm volatile("bar.sync 3, %0;" ::"n"(TPR) : "memory"); break;
      default: asm volatile("bar.sync 4, %0;" ::"n"(TPR) : "memory"); break;
    }
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + ri), "n"(TPR) : "memory");
  }
}

template <class Op, class T, int TPR> __device__ __forceinline__ T row_tree(T v, T* sh, int ri) {
  constexpr int W = TPR < 32 ? TPR : 32;
#pragma unroll
  for (int m = 1; m < W; m <<= 1) v = Op::template c<T>(v, shfl_xor<T>(v, m));
  if constexpr (TPR > 32) {
    constexpr int NW = TPR / 32;
    const int tr = threadIdx.x % TPR;
    if ((threadIdx.x & 31) == 0) sh[ri * NW + tr / 32] = v;
    row_bar<TPR>(ri);
    T buf[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w) buf[w] = sh[ri * NW + w];
#pragma unroll
    for (int s = 1; s < NW; s <<= 1)
#pragma unroll
      for (int w = 0; w + s < NW; w += 2 * s) buf[w] = Op::template c<T>(buf[w], buf[w + s]);
    row_bar<TPR>(ri);
    v = buf[0];
  }
  return v;
}

// Leaf-level combine over the P parts then the row tree (float sums).
// TRAIL: end with a second row barrier so ``sh`` may be rewritten at once;
// callers that pass another barrier of the row before reusing ``sh`` (a later
// row reduction with its own ``sh``, or the CTA barrier that ends a row group)
// skip it.
template <class T, int VEC, int P, int TPR, bool TRAIL = true>
__device__ __forceinline__ T row_sum(const T (&acc)[VEC], T* sh, int ri) {
  T s = leaf_local<T, VEC>(acc);
#pragma unroll
  for (int m = 1; m < P; m <<= 1) s = add<T>(s, shfl_xor<T>(s, m));
  // leaves: lanes P apart
  constexpr int W = TPR < 32 ? TPR : 32;
#pragma unroll
  for (int m = P; m < W; m <<= 1) s = add<T>(s, shfl_xor<T>(s, m));
  if constexpr (TPR > 32) {
    constexpr int NW = TPR / 32;
    const int tr = threadIdx.x % TPR;
    if ((threadIdx.x & 31) == 0) sh[ri * NW + tr / 32] = s;
    row_bar<TPR>(ri);
    T buf[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w) buf[w] = sh[ri * NW + w];
#pragma unroll
    for (int st = 1; st < NW; st <<= 1)
#pragma unroll
      for (int w = 0; w + st < NW; w += 2 * st) buf[w] = add<T>(buf[w], buf[w + st]);
    if constexpr (TRAIL) row_bar<TPR>(ri);
    s = buf[0];
  }
  return s;
}

// First-index arg combine over the row's threads.
template <bool MAX, class T, int TPR>
__device__ __forceinline__ long long row_arg(T best, long long bi, T* shv, long long* shi, int ri) {
  constexpr int W = TPR < 32 ? TPR : 32;
#pragma unroll
  for (int m = 1; m < W; m <<= 1) {
    T ov = shfl_xor<T>(best, m);
    long long oi = __shfl_xor_sync(0xffffffffu, bi, m);
    if (arg_take_b<MAX, T>(best, bi, ov, oi)) {
      best = ov;
      bi = oi;
    }
  }
  if constexpr (TPR > 32) {
    constexpr int NW = TPR / 32;
    const int tr = threadIdx.x % TPR;
    if ((threadIdx.x & 31) == 0) {
      shv[ri * NW + tr / 32] = best;
      shi[ri * NW + tr / 32] = bi;
    }
    row_bar<TPR>(ri);
    best = shv[ri * NW];
    bi = shi[ri * NW];
#pragma unroll
    for (int w = 1; w < NW; ++w) {
      if (arg_take_b<MAX, T>(best, bi, shv[ri * NW + w], shi[ri * NW + w])) {
        best = shv[ri * NW + w];
        bi = shi[ri * NW + w];
      }
    }
    row_bar<TPR>(ri);
  }
  return bi;
}

// ---- single-pass scan with decoupled look-back (codegen_scan.py) -------------
// Tile t publishes (flag, value): flag 1 = tile aggregate, 2 = inclusive prefix.
// Tile ids come from an atomic counter so earlier tiles are always scheduled
// first (forward progress); the look-back folds predecessors right to left.
template <class T> struct ScanState {
  unsigned long long* flags;   // per tile: 0 empty, 1 aggregate, 2 inclusive
  T* agg;
  T* inc;
};

template <class Op, class T>
__device__ __forceinline__ T scan_lookback(const ScanState<T>& st, long long tile, T tile_agg) {
  // called by one thread; returns the exclusive prefix of `tile`
  if (tile == 0) {
    st.inc[0] = tile_agg;
    __threadfence();
    atomicExch(&st.flags[0], 2ull);
    return T(0);
  }
  st.agg[tile] = tile_agg;
  __threadfence();
  atomicExch(&st.flags[tile], 1ull);
  T excl;
  bool have = false;
  long long p = tile - 1;
  while (true) {
    unsigned long long f;
    do {
      f = atomicAdd(&st.flags[p], 0ull);
    } while (f == 0ull);
    __threadfence();
    const T v = (f == 2ull) ? st.inc[p] : st.agg[p];
    excl = have ? Op::template c<T>(v, excl) : v;
    have = true;
    if (f == 2ull) break;
    --p;
  }
  st.inc[tile] = Op::template c<T>(excl, tile_agg);
  __threadfence();
  atomicExch(&st.flags[tile], 2ull);
  return excl;
}

// Single-pass tile scan with a warp-parallel, order-preserving look-back.
// Tile t publishes its aggregate (flag 1) and later its inclusive prefix
// (flag 2) with release stores.  Warp 0 of tile t walks back over windows of
// 32 predecessors (acquire loads) until a window holds an inclusive prefix,
// then folds LEFT TO RIGHT: that inclusive prefix, then the aggregates of every
// later tile up to t-1 (re-read from the aggregate array).  Each inclusive
// prefix is prefix + aggregate, so any such left fold equals the sequential
// chain of tile aggregates bit for bit: the result does not depend on timing.
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u32(unsigned* p, unsigned v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// padded shared-tile index: one spare word per 32 keeps both the striped
// (coalesced) and the blocked (per-thread run) accesses bank-conflict free
__device__ __forceinline__ long long spad(long long e) { return e + (e >> 5); }

// Publish a tile's aggregate (flag 1); tile 0 publishes its inclusive prefix
// from the look-back instead.
// Scan status words: a published value travels with its flag in the same
// 64-bit word (flag in the high half), so a reader that sees the flag sees the
// value — no fences on either side.  8-byte values use two words, each
// carrying one half and the flag.  Words are zeroed before the launch and
// written once (group prefixes may be written by several warps, always with
// the same bits).
template <class T> struct Stat { static constexpr int W = sizeof(T) <= 4 ? 1 : 2; };
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
template <class T> __device__ __forceinline__ unsigned long long stat_bits(T v) {
  union { T t; unsigned long long u; } x;
  x.u = 0;
  x.t = v;
  return sizeof(T) <= 4 ? (x.u & 0xffffffffull) : x.u;
}
template <class T> __device__ __forceinline__ void stat_put(unsigned long long* w, long long i, T v) {
  constexpr unsigned long long F = 1ull << 32;
  if constexpr (sizeof(T) <= 4) {
    st_relaxed_u64(w + i, F | stat_bits(v));
  } else {
    const unsigned long long b = stat_bits(v);
    st_relaxed_u64(w + 2 * i, F | (b & 0xffffffffull));
    st_relaxed_u64(w + 2 * i + 1, F | (b >> 32));
  }
}
// raw words of entry i (issue the loads; check with stat_ok / decode later)
template <class T> struct StatRaw { unsigned long long a, b; };
template <class T> __device__ __forceinline__ StatRaw<T> stat_ld(const unsigned long long* w, long long i) {
  StatRaw<T> r;
  if constexpr (sizeof(T) <= 4) { r.a = ld_relaxed_u64(w + i); r.b = 1ull << 32; }
  else { r.a = ld_relaxed_u64(w + 2 * i); r.b = ld_relaxed_u64(w + 2 * i + 1); }
  return r;
}
template <class T> __device__ __forceinline__ bool stat_ok(const StatRaw<T>& r) {
  if constexpr (sizeof(T) <= 4) return (r.a >> 32) != 0;
  else return (r.a >> 32) != 0 && (r.b >> 32) != 0;
}
template <class T> __device__ __forceinline__ T stat_val(const StatRaw<T>& r) {
  T v;
  union { T t; unsigned long long u; } x;
  x.u = sizeof(T) <= 4 ? (r.a & 0xffffffffull) : ((r.a & 0xffffffffull) | (r.b << 32));
  v = x.t;
  return v;
}

#ifdef GR_SCAN_STATS
__device__ unsigned long long gr_scan_stats[8];
#endif
// A look-back waits for other CTAs' tile aggregates; those CTAs are resident
// by construction (persistent grids sized by the occupancy calculator).  If
// that ever fails (another tenant holding SMs), fail loudly instead of
// hanging: ~2^24 polls of an L2 word is seconds, a normal wait microseconds.
__device__ __forceinline__ void spin_guard(unsigned& polls) {
  if (++polls == (1u << 24)) {
    printf("grumpy: scan look-back waited 2^24 polls for a predecessor tile (grid not co-resident?)\n");
    __trap();
  }
}
// Exclusive prefix of tile `tile` of a single-pass scan; one full warp calls
// it after the tile's aggregate was published (stat_put(agg, tile, .)), and it
// publishes the tile's inclusive prefix (stat_put(inc, tile, .)).
//
// Deterministic: incl(t) = incl(t-1) (+) agg(t), a left fold over the tile
// aggregates, so the prefix is the same bits whichever published inclusive
// prefix the walk starts from.  Values travel inside their status words (no
// fences): one L2 round trip reads the inclusive and aggregate words of the
// 256 nearest predecessors, the nearest published inclusive prefix starts the
// fold, and lane 0 folds the aggregates above it in tile order.
#ifndef GR_SCAN_J
#define GR_SCAN_J 2
#endif
#ifndef GR_SCAN_R
#define GR_SCAN_R 8
#endif
template <class T> struct __align__(16) LookbackBuf { T v[32 * GR_SCAN_J * GR_SCAN_R]; };

template <class Op, class T>
__device__ __forceinline__ T tile_lookback_buf(const unsigned long long* agg, unsigned long long* inc,
                                               long long tile, T tile_agg, T ident, T* lb, long long ls = 0);
template <class Op, class T>
__device__ __forceinline__ T tile_lookback(const unsigned long long* agg, unsigned long long* inc,
                                           long long tile, T tile_agg, T ident, long long ls = 0) {
  __shared__ LookbackBuf<T> lbs;
  return tile_lookback_buf<Op, T>(agg, inc, tile, tile_agg, ident, lbs.v, ls);
}
// lb: the calling warp's own staging array (32 * J * R values); several
// look-back warps of one CTA each pass their own.  ls: the first tile of the
// tile's segment (a line of a matrix scanned along its rows): the walk never
// goes below it, and the segment's first tile starts its own prefix chain.
template <class Op, class T>
__device__ __forceinline__ T tile_lookback_buf(const unsigned long long* agg, unsigned long long* inc,
                                               long long tile, T tile_agg, T ident, T* lb, long long ls) {
  const int lane = threadIdx.x & 31;
#ifdef GR_SCAN_NOLB
  return ident;   // experiment: streaming floor without any look-back (wrong results)
#endif
  if (tile == ls) {
    if (lane == 0) stat_put<T>(inc, tile, tile_agg);
    return ident;
  }
#ifdef GR_SCAN_STATS
  const long long c0 = clock64();
#endif
  constexpr int J = GR_SCAN_J;       // 32*J predecessors per round trip
  constexpr int R = GR_SCAN_R;       // windows staged before the slow path
  // lb: aggregates by distance, lb[tile-1-q]
  // walk back window by window: one round trip reads the inclusive and the
  // aggregate words of 32*J predecessors; aggregates above the nearest
  // published inclusive prefix are staged by distance
  long long found = -1;
  T base = ident;
  long long top = tile - 1;
  for (int w = 0; w < R && found < 0; ++w, top -= 32 * J) {
    StatRaw<T> ri[J], ra[J];
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const long long q = top - lane - 32 * j;
      ri[j] = q >= ls ? stat_ld<T>(inc, q) : StatRaw<T>{0, 0};
      ra[j] = q >= ls ? stat_ld<T>(agg, q) : StatRaw<T>{0, 0};
    }
    long long fw = -1;
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const unsigned m = __ballot_sync(0xffffffffu, stat_ok<T>(ri[j]));
      if (fw < 0 && m) fw = top - (__ffs(m) - 1) - 32 * j;
    }
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const long long q = top - lane - 32 * j;
      if (q >= ls && q > fw) {
        for (unsigned polls = 0; !stat_ok<T>(ra[j]); spin_guard(polls)) ra[j] = stat_ld<T>(agg, q);
        lb[tile - 1 - q] = stat_val<T>(ra[j]);
      }
      if (q == fw) base = stat_val<T>(ri[j]);
    }
    if (fw >= 0) {
      found = fw;
      base = __shfl_sync(0xffffffffu, base, (int)((top - fw) & 31));
    }
    if (top - 32 * J < ls && found < 0) { top = tile - 1 + 32 * J; w = -1; }   // nothing published down to the segment's start yet: poll again
  }
  __syncwarp();
  T pre = ident;
  if (found >= 0) {
    if (lane == 0) {
      pre = base;
      // left fold in tile order; the shared-memory reads of each batch of 8
      // are issued together (a read per add was an LDS latency per tile of
      // distance on every look-back's critical path)
      long long d = tile - 2 - found;
      for (; d >= 7; d -= 8) {
        T v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = lb[d - k];
#pragma unroll
        for (int k = 0; k < 8; ++k) pre = Op::template c<T>(pre, v[k]);
      }
      for (; d >= 0; --d) pre = Op::template c<T>(pre, lb[d]);
    }
  } else {
    // slow path (more than 32*J*R tiles in flight behind this one): walk the
    // inclusive words further back, then fold the aggregates in chunks
    while (found < 0) {
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const long long q = top - lane - 32 * j;
        const StatRaw<T> r = q >= ls ? stat_ld<T>(inc, q) : StatRaw<T>{0, 0};
        const unsigned m = __ballot_sync(0xffffffffu, stat_ok<T>(r));
        if (found < 0 && m) found = top - (__ffs(m) - 1) - 32 * j;
      }
      if (found < 0) {
        top -= 32 * J;
        if (top < ls) top = tile - 1;
      }
    }
    StatRaw<T> rf = stat_ld<T>(inc, found);
    pre = stat_val<T>(rf);
    for (long long b0 = found + 1; b0 <= tile - 1; b0 += 32 * J) {
      __syncwarp();
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const long long q = b0 + lane + 32 * j;
        if (q <= tile - 1) {
          StatRaw<T> r = stat_ld<T>(agg, q);
          for (unsigned polls = 0; !stat_ok<T>(r); spin_guard(polls)) r = stat_ld<T>(agg, q);
          lb[lane + 32 * j] = stat_val<T>(r);
        }
      }
      __syncwarp();
      if (lane == 0) {
        const int cnt = (int)((tile - b0) < 32 * J ? (tile - b0) : 32 * J);
        int l = 0;
        for (; l + 8 <= cnt; l += 8) {
          T v[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) v[k] = lb[l + k];
#pragma unroll
          for (int k = 0; k < 8; ++k) pre = Op::template c<T>(pre, v[k]);
        }
        for (; l < cnt; ++l) pre = Op::template c<T>(pre, lb[l]);
      }
    }
  }
  if (lane == 0) stat_put<T>(inc, tile, Op::template c<T>(pre, tile_agg));
#ifdef GR_SCAN_STATS
  if (lane == 0) { atomicAdd(&gr_scan_stats[0], (unsigned long long)(tile - found)); atomicAdd(&gr_scan_stats[1], 1ull);
                   atomicAdd(&gr_scan_stats[2], (unsigned long long)(clock64() - c0)); }
#endif
  return __shfl_sync(0xffffffffu, pre, 0);
}

// Look-back of a persistent grid whose G CTAs take the tiles round-robin
// (tile t on CTA t % G, in its round t / G).  The prefix of tile t > 0 is the
// left fold, in tile order, of the calling CTA's own inclusive prefix of tile
// t - G (in the first round: the aggregate of tile 0) and the aggregates of
// the tiles in between — the same left fold as tile_lookback_buf, so the same
// bits.  No inclusive prefix crosses CTAs: a look-back waits only for its
// predecessors' aggregates (published when their tiles are reduced), never
// for their look-backs, and one L2 round trip reads all G - 1 of them.
// One full warp calls it; lb: the warp's staging array (>= G - 1 values).
//
// Two halves, so that several look-back warps can overlap one tile's loads
// with the previous tile's fold: round_stage reads the aggregates into lb
// (padded to a multiple of 8 with a value the combine leaves unchanged:
// -0.0 for sums, x + -0.0 == x with signed zeros; the identity otherwise),
// round_fold folds them onto the CTA's previous inclusive prefix.
template <class Op, class T> __device__ __forceinline__ T round_pad(T ident) {
  if constexpr (IsSum<Op>::v) return Zero<T>::neg();
  return ident;
}
// ls: the first tile of the tile's segment (0 for one long scan; the first
// tile of its line for a scan along the rows of a matrix): the fold never
// reaches below it
template <class Op, class T, int J = 5>
__device__ __forceinline__ void round_stage(const unsigned long long* agg, long long tile, int G, long long ls,
                                            T ident, T* lb) {
#ifdef GR_SCAN_NOLB
  return;           // experiment: streaming floor without any look-back (wrong results)
#endif
  const int lane = threadIdx.x & 31;
  const long long lo = tile - G + 1 > ls ? tile - G + 1 : ls;   // first aggregate folded
  const int n = (int)(tile - lo);                        // aggregates lo .. tile-1
  const int n8 = (n + 7) & ~7;
  const T pad = round_pad<Op, T>(ident);
  for (int w0 = 0; w0 < n8; w0 += 32 * J) {
    StatRaw<T> ra[J];
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const int k = w0 + lane + 32 * j;
      if (k < n) ra[j] = stat_ld<T>(agg, lo + k);
    }
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const int k = w0 + lane + 32 * j;
      if (k < n) {
        for (unsigned polls = 0; !stat_ok<T>(ra[j]); spin_guard(polls)) ra[j] = stat_ld<T>(agg, lo + k);
        lb[k] = stat_val<T>(ra[j]);
      } else if (k < n8) {
        lb[k] = pad;
      }
    }
  }
  __syncwarp();
}
template <class Op, class T>
__device__ __forceinline__ T round_fold(long long tile, int G, long long ls, T own_inc, T ident, T* lb) {
#ifdef GR_SCAN_NOLB
  return own_inc;   // experiment: streaming floor without any look-back (wrong results)
#endif
  const int lane = threadIdx.x & 31;
  const bool first = tile - G < ls;                // no own prefix inside the segment
  const int n = (int)(first ? tile - ls : G - 1);
  const int n8 = (n + 7) & ~7;
  const T pad = round_pad<Op, T>(ident);
  T pre = own_inc;
  if (lane == 0 && n > 0) {
    if (first) { pre = lb[0]; lb[0] = pad; }       // first round: the fold starts at the segment's first tile
    // left fold in tile order; each batch of 8 is read while the previous one
    // is folded, so the chain is one dependent combine per aggregate
    T a[8], b[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) a[q] = lb[q];
#pragma unroll 1
    for (int k = 0; k < n8; k += 8) {
      if (k + 8 < n8) {
#pragma unroll
        for (int q = 0; q < 8; ++q) b[q] = lb[k + 8 + q];
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) pre = Op::template c<T>(pre, a[q]);
#pragma unroll
      for (int q = 0; q < 8; ++q) a[q] = b[q];
    }
  }
  return __shfl_sync(0xffffffffu, pre, 0);
}
// The same look-back with the aggregates between the CTA's previous tile and
// this one combined as a tree across the warp instead of a left fold: each
// lane folds the aggregates k = lane + 32 j (j ascending), then a butterfly
// over the lanes (fixed pattern), then own (+) that — one dependent combine
// per aggregate became ~J + 5, so the look-back is a round trip plus ~100
// cycles.  The association depends only on the tile index and G (the grid,
// one CTA per SM): deterministic on a given GPU, more accurate than the left
// fold, no longer the register-staged kernel's bits.  Returns the tree of
// the aggregates; the caller's prefix is own (+) tree, or the tree alone for
// a segment's first round (tile - G < ls: no own prefix inside the segment).
template <class Op, class T, int J = 5>
__device__ __forceinline__ T round_tree(const unsigned long long* agg, long long tile, int G, long long ls, T ident) {
#ifdef GR_SCAN_NOLB
  return ident;     // experiment: streaming floor without any look-back (wrong results)
#endif
  const int lane = threadIdx.x & 31;
  const bool first = tile - G < ls;
  const long long lo = first ? ls : tile - G + 1;
  const int n = (int)(tile - lo);
  const T pad = round_pad<Op, T>(ident);
  T acc = pad;
  for (int w0 = 0; w0 < n; w0 += 32 * J) {
    StatRaw<T> ra[J];
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const int k = w0 + lane + 32 * j;
      if (k < n) ra[j] = stat_ld<T>(agg, lo + k);
    }
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const int k = w0 + lane + 32 * j;
      if (k < n) {
        for (unsigned polls = 0; !stat_ok<T>(ra[j]); spin_guard(polls)) ra[j] = stat_ld<T>(agg, lo + k);
        acc = Op::template c<T>(acc, stat_val<T>(ra[j]));
      }
    }
  }
#pragma unroll
  for (int m = 1; m < 32; m <<= 1) {
    const T o = shfl_xor<T>(acc, m);
    acc = (lane & m) ? Op::template c<T>(o, acc) : Op::template c<T>(acc, o);
  }
  return acc;
}

template <class Op, class T, int J = 5>
__device__ __forceinline__ T tile_lookback_round(const unsigned long long* agg, long long tile, int G, long long ls,
                                                 T own_inc, T ident, T* lb) {
#ifdef GR_SCAN_NOLB
  return own_inc;   // experiment: streaming floor without any look-back (wrong results)
#endif
#ifdef GR_SCAN_STATS
  const long long c0 = clock64();
#endif
  round_stage<Op, T, J>(agg, tile, G, ls, ident, lb);
#ifdef GR_SCAN_STATS
  const long long c1 = clock64();
#endif
  const T pre = round_fold<Op, T>(tile, G, ls, own_inc, ident, lb);
#ifdef GR_SCAN_STATS
  if ((threadIdx.x & 31) == 0 && blockIdx.x == 0) { gr_scan_stats[4] += c1 - c0; gr_scan_stats[5] += clock64() - c1; gr_scan_stats[6] += 1; }
#endif
  return pre;
}

// acq_rel atomic add (gpu scope): releases the caller's prior writes,
// acquires those released by earlier adds on the same word
__device__ __forceinline__ unsigned atom_add_acq_rel(unsigned int* p, unsigned int v) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
// release-only add (MEMBAR.ALL.GPU + ATOMG): no acquire, so no L1 invalidation
// (an acq_rel or fenced atomic at gpu scope also emits CCTL.IVALL); the rare
// reader that finds the count complete acquires with fence_acq_rel()
__device__ __forceinline__ unsigned atom_add_release(unsigned int* p, unsigned int v) {
  unsigned old;
  asm volatile("atom.release.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// Perfect binary tree over p[0..N) (N a power of two) by ONE warp: each lane
// folds a contiguous chunk as a perfect tree (pairwise stack), the lanes
// combine by the xor butterfly — the same association as block_tree over the
// same range.  N < 32: lanes >= N contribute the identity.
template <class Op, class T, long long N> __device__ __forceinline__ T warp_range_tree(const T* p, T ident) {
  const int lane = threadIdx.x & 31;
  T v;
  if constexpr (N >= 32) {
    constexpr long long CH = N / 32;
    v = chunk_tree<Op, T>(p + lane * CH, CH, CH, ident);
  } else {
    v = lane < N ? __ldcg(p + lane) : ident;
  }
  return warp_tree<Op, T>(v);
}

// Ticket of a group of `expected` blocks: true in exactly the last of them to
// arrive, after every earlier arrival's writes are visible; self-resetting.
// Called by whole blocks (uniformly).
__device__ __forceinline__ bool last_arrival(unsigned int* ticket, unsigned int expected) {
  __shared__ bool am_last_a;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned int prev = atomicAdd(ticket, 1u);
    am_last_a = (prev == expected - 1);
  }
  __syncthreads();
  if (am_last_a) {
    __threadfence();
    if (threadIdx.x == 0) *ticket = 0u;
  }
  return am_last_a;
}

// Grid completion ticket: returns true in exactly one (the last) block, after
// every block's partials are visible.  The ticket self-resets for the next
// launch of the same kernel (stream order serialises launches).
__device__ __forceinline__ bool last_block(unsigned int* ticket) {
  __shared__ bool am_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    unsigned int prev = atomicAdd(ticket, 1u);
    am_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (am_last) {
    __threadfence();
    if (threadIdx.x == 0) *ticket = 0u;
  }
  return am_last;
}

}  // namespace gr
