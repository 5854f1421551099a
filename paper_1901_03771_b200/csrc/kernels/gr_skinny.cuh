// gr_skinny.cuh — skinny GEMM prologue of a row region (C4 layer 2).
//
// The reference sends every np.dot to the library (run_library,
// /root/reference/SPEC.md:391-399; the paper's cuBLAS gemv)
// and fuses only the elementwise consumers of its result.
// For z = A @ B with A [R, K] streamed from HBM and B a small [K, N] operand
// (N <= 16), the product is bound by reading A once — a cuBLAS call writes z
// to HBM and a second kernel reads it back for the row consumers (bias,
// softmax, argmax).  Here the product is the first stage of the consumers'
// row kernel: z never leaves registers.
//
//   * one CTA thread owns RT rows of a BLOCK*RT-row tile (rows L, L+BLOCK,
//     ...: every B operand feeds RT rows); the CTA walks its tiles with a
//     grid stride;
//   * A arrives in [BLOCK rows x 32 columns] boxes by TMA
//     (cp.async.bulk.tensor.2d, 128-byte swizzle) through an S-slot shared-
//     memory ring; thread 0 keeps S boxes in flight across tile boundaries,
//     completion on one mbarrier per slot (expect_tx / complete_tx);
//   * B is read as k-pairs Bp[kp * N + n] = (B[2kp][n], B[2kp+1][n]): one
//     copy per CTA in shared memory (every thread reads the same pair: a
//     broadcast), or 64-bit uniform operands from the constant bank (measured
//     slower: constant-cache latency).  The row's even/odd k terms accumulate
//     in one packed FFMA2 per (k-pair, n); z[n] is the sum of the two halves.  The association differs from OpenBLAS's (as cuBLAS's
//     does): results are checked to a tolerance, not bit-exact.
//   * a thread reads its row's 16-byte chunks through the swizzle (sw128), so
//     the 32 lanes of a warp hit distinct bank groups.
#pragma once

namespace gr {

template <int BLOCK, int KDIM, int N, int S, int RT>
struct Skinny {
  static_assert(KDIM % 32 == 0, "K must be a multiple of the 32-column box");
  static constexpr int ROWS = BLOCK * RT;              // rows per tile (= box rows)
  static constexpr int KB = KDIM / 32;                 // boxes per row tile
  static constexpr unsigned BOX_BYTES = ROWS * 128u;   // 32 f32 columns per row
  static constexpr int SLOT_FLOATS = ROWS * 32;

  float* ring;                 // S slots, 1024-byte aligned (128B-swizzle atoms)
  unsigned long long* full;    // one mbarrier per slot
  const TMap* map;
  long long nrows;
  long long q_issue;           // next box to issue (thread 0)
  long long q_use;             // next box to consume

  __device__ __forceinline__ long long tile_row(long long j) const {
    return ((long long)blockIdx.x + j * (long long)gridDim.x) * ROWS;
  }

  __device__ __forceinline__ void issue_one() {
    const long long j = q_issue / KB;
    const int kb = (int)(q_issue % KB);
    const long long row0 = tile_row(j);
    if (row0 < nrows) {
      const int s = (int)(q_issue % S);
      mbar_arrive_expect_tx(&full[s], BOX_BYTES);
      tma_load_2d(ring + s * SLOT_FLOATS, map, kb * 32, (int)row0, &full[s]);
    }
    ++q_issue;
  }

  __device__ __forceinline__ void init(float* ring_, unsigned long long* full_, const TMap* map_, long long nrows_) {
    ring = ring_;
    full = full_;
    map = map_;
    nrows = nrows_;
    q_issue = 0;
    q_use = 0;
    if (threadIdx.x == 0) {
      for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
      fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int s = 0; s < S; ++s) issue_one();
    }
  }

  // B as k-pairs in shared memory (the shared-memory variant): every thread
  // of the CTA reads the same pair -> broadcast
  static __device__ __forceinline__ void load_pairs(unsigned long long* __restrict__ bs, const float* __restrict__ B) {
    for (int i = threadIdx.x; i < KDIM / 2 * N; i += BLOCK) {
      const int kp = i / N, n = i % N;
      bs[i] = (unsigned long long)__float_as_uint(B[(2 * kp) * N + n]) |
              ((unsigned long long)__float_as_uint(B[(2 * kp + 1) * N + n]) << 32);
    }
  }

  // z[j][n] = sum_k A[row0 + threadIdx.x + j * BLOCK, k] * B[k, n] for this
  // CTA's next tile (RT rows per thread share every B operand)
  __device__ __forceinline__ void tile(float (&z)[RT][N], const unsigned long long* __restrict__ bp) {
    f2 acc[RT][N];
#pragma unroll
    for (int j = 0; j < RT; ++j)
#pragma unroll
      for (int n = 0; n < N; ++n) acc[j][n].v = 0ull;
    const unsigned L = threadIdx.x;
#pragma unroll 1
    for (int kb = 0; kb < KB; ++kb) {
      const int s = (int)(q_use % S);
      mbar_wait(&full[s], (unsigned)((q_use / S) & 1));
      const char* slot = reinterpret_cast<const char*>(ring + s * SLOT_FLOATS);
      const unsigned long long* b = bp + (long long)kb * 16 * N;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        f2 h01[RT], h23[RT];
#pragma unroll
        for (int j = 0; j < RT; ++j) {
          const float4 h = *reinterpret_cast<const float4*>(slot + sw128(L + j * BLOCK, (unsigned)c));
          h01[j] = pk(h.x, h.y);
          h23[j] = pk(h.z, h.w);
        }
#pragma unroll
        for (int n = 0; n < N; ++n) {
          f2 w0, w1;
          w0.v = b[(2 * c) * N + n];
          w1.v = b[(2 * c + 1) * N + n];
#pragma unroll
          for (int j = 0; j < RT; ++j) {
            acc[j][n] = p2::fma(h01[j], w0, acc[j][n]);
            acc[j][n] = p2::fma(h23[j], w1, acc[j][n]);
          }
        }
      }
      ++q_use;
      // every thread has read slot s: thread 0 refills it with box q + S
      __syncthreads();
      if (threadIdx.x == 0) {
        fence_proxy_async();
        issue_one();
      }
    }
#pragma unroll
    for (int j = 0; j < RT; ++j)
#pragma unroll
      for (int n = 0; n < N; ++n) z[j][n] = lo(acc[j][n]) + hi(acc[j][n]);
  }
};

}  // namespace gr
