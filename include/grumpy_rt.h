/*
 * grumpy_rt.h — C-ABI of libgrumpy_rt.so, the drop-in executor boundary of the
 * fused-region path (B200 / sm_100a).
 *
 * The reference defines the executor as the swappable layer: GPU work is
 * "replaced by built-in CPU library kernels behind the same planner interface"
 * and "an optional hook allows swapping in an
 * optimized external implementation behind the same call signature"
 * (SPEC.md:410).  Its executor entry points are
 *     run_map(FusedKernel(Map), leaves, cfg)        -> TensorBuffer
 *     run_map_reduce(FusedKernel(MapReduce), ...)   -> TensorBuffer
 *     run_map_scan(FusedKernel(MapScan), ...)       -> TensorBuffer
 *     run_library(LibraryCall, operand buffers, cfg)-> TensorBuffer
 *     compile(PointProgram) -> executable point fn
 * and the paper's GPU realisation sat on the CUDA driver: PTX loaded and
 * launched through the driver API, automatic H2D/D2H around kernels, cuBLAS for
 * gemv.
 *
 * This header is the B200 replacement for that layer.  Python binds it with
 * ctypes (paper_1901_03771_b200/runtime.py); INTEGRATION.md shows the binding.
 * Conventions:
 *   - every export returns int: 0 = OK, otherwise a GR_E* status below;
 *   - grumpy_rt_last_error() returns a thread-local message for the last
 *     failure on the calling thread (NVRTC failures carry the compile log);
 *   - device pointers cross the boundary as uint64_t; host pointers as void*;
 *   - one process drives one device; all work is ordered on one stream owned
 *     by the runtime (kernels, copies, cuBLAS and NCCL share it).
 */
#ifndef GRUMPY_RT_H_
#define GRUMPY_RT_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  GR_OK = 0,
  GR_ECUDA = 1,      /* CUDA driver error (CUresult in message)           */
  GR_ENVRTC = 2,     /* NVRTC compile error (log in message)              */
  GR_ECUBLAS = 3,    /* cuBLAS status                                     */
  GR_ENCCL = 4,      /* NCCL status                                       */
  GR_EINVAL = 5,     /* bad argument                                      */
  GR_ENOINIT = 6,    /* grumpy_rt_init not called / no device             */
  GR_ENOMEM = 7,     /* device out of memory even after trimming the pool */
  GR_EDLOPEN = 8     /* libcuda.so.1 / libnccl.so.2 could not be loaded   */
};

/* dtype codes shared with the Python side (tensor.DType) */
enum { GR_F32 = 0, GR_F64 = 1, GR_I32 = 2, GR_I64 = 3, GR_BOOL = 4 };
/* reduction ops for NCCL (dag.ReduceOp) */
enum { GR_SUM = 0, GR_PROD = 1, GR_MAX = 2, GR_MIN = 3 };

/* ---- lifecycle / device ------------------------------------------------- */
int grumpy_rt_version(int* version);
/* Load libcuda, retain the primary context of `device`, create the stream. */
int grumpy_rt_init(int device);
int grumpy_rt_device_count(int* count);
/* name: caller buffer of >= 256 bytes */
int grumpy_rt_device_info(int* sm_count, int* cc_major, int* cc_minor,
                          size_t* total_mem, char* name);
const char* grumpy_rt_last_error(void);
/* CUstream of the runtime, for interop (e.g. wrapping in torch) */
int grumpy_rt_stream(uint64_t* stream);

/* ---- caching device memory pool (replaces per-op temporaries,
 *      north_star (5); TensorBuffer storage SPEC.md:37-42) ---------------- */
int grumpy_rt_alloc(size_t bytes, uint64_t* dptr);
int grumpy_rt_free(uint64_t dptr);
int grumpy_rt_pool_stats(size_t* in_use, size_t* cached, size_t* peak, size_t* n_allocs);
int grumpy_rt_pool_trim(void);

/* ---- transfers (the paper's automatic H2D/D2H) -------- */
/* Asynchronous on the runtime stream; src must stay valid until the next
 * grumpy_rt_sync() when it is page-locked. */
int grumpy_rt_h2d(uint64_t dst, const void* src, size_t bytes);
/* Synchronous: returns when dst holds the data. */
int grumpy_rt_d2h(void* dst, uint64_t src, size_t bytes);
int grumpy_rt_d2d(uint64_t dst, uint64_t src, size_t bytes);
int grumpy_rt_memset(uint64_t dst, int byte_value, size_t bytes);
int grumpy_rt_host_alloc(size_t bytes, void** ptr); /* page-locked */
int grumpy_rt_host_free(void* ptr);
int grumpy_rt_host_register(void* ptr, size_t bytes);
int grumpy_rt_host_unregister(void* ptr);

/* ---- compile: PointProgram -> executable --------------
 * NVRTC-compiles `src` (a generated instantiation of the hand-written
 * kernel templates) for sm_100a with `opts`, loads the cubin as a module.
 * A process-wide table and an on-disk cubin cache under `cache_dir` (may be
 * NULL) are keyed by FNV-1a(src, opts).  *compile_ms = NVRTC time, 0 on a
 * cache hit; *cache_hit = 0 (compiled), 1 (memory), 2 (disk), 3 (compiled
 * ahead by grumpy_rt_precompile). */
int grumpy_rt_compile(const char* src, const char* const* opts, int n_opts,
                      const char* cache_dir, uint64_t* module,
                      double* compile_ms, int* cache_hit);
/* JIT/execute pipelining: NVRTC-compile `src` ahead of its
 * first launch — no CUDA context is touched, so worker threads call it while
 * the host thread launches earlier steps; the cubin is kept in memory (and in
 * the disk cache) until grumpy_rt_compile loads it. */
int grumpy_rt_precompile(const char* src, const char* const* opts, int n_opts,
                         const char* cache_dir, double* compile_ms);
/* Compile only (no device needed): writes the sm_100a cubin into `out` when
 * `cap` is large enough; *size is always set.  Used by CPU tests to check
 * every generated kernel builds. */
int grumpy_rt_compile_cubin(const char* src, const char* const* opts, int n_opts,
                            void* out, size_t cap, size_t* size, double* compile_ms);
int grumpy_rt_get_function(uint64_t module, const char* name, uint64_t* fn);
/* Device address and size of a module-scope __constant__/__device__ symbol
 * (constant-bank staging of small row-invariant leaves; filled with
 * grumpy_rt_d2d on the runtime stream before each launch). */
int grumpy_rt_module_global(uint64_t module, const char* name, uint64_t* dptr, size_t* bytes);
/* Encode a 2-D tiled TMA descriptor (CUtensorMap, 128 bytes written to
 * `out128`) for a row-major tensor [dim1][dim0] of `dtype` at `gaddr` whose
 * rows are `stride1` bytes apart; box = [box1][box0] elements; `swizzle` =
 * 0, 32, 64 or 128 (bytes).  Passed to kernels inside their by-value
 * parameter block (__grid_constant__) for cp.async.bulk.tensor loads. */
int grumpy_rt_tensor_map_2d(uint64_t gaddr, int dtype, uint64_t dim0, uint64_t dim1, uint64_t stride1,
                            unsigned box0, unsigned box1, int swizzle, void* out128);
int grumpy_rt_function_info(uint64_t fn, int* num_regs, int* local_bytes,
                            int* static_smem, int* max_threads);
int grumpy_rt_occupancy(uint64_t fn, int block, size_t dyn_smem, int* blocks_per_sm);

/* ---- launch: run_map / run_map_reduce / run_map_scan ---
 * `params` is the kernel's single by-value parameter struct (packed by the
 * code generator's layout), `params_size` its size in bytes.  cluster_x > 1
 * launches with a thread-block cluster of that size. */
int grumpy_rt_launch(uint64_t fn, unsigned gx, unsigned gy, unsigned gz,
                     unsigned bx, unsigned by, unsigned bz, unsigned dyn_smem,
                     unsigned cluster_x, const void* params, size_t params_size);
/* Waits for all work of the runtime's context (every stream). */
int grumpy_rt_sync(void);

/* ---- profiler ranges (NVTX 3) ----------------------------------------------
 * Named, nestable ranges around plan steps for Nsight Systems / Compute
 * (SURVEY.md §5 tracing); no-ops unless a tool injects itself. */
int grumpy_rt_range_push(const char* name);
int grumpy_rt_range_pop(void);

/* ---- streams: copy/compute overlap for streamed materialisation ---------
 * Async work (launch, h2d, d2h_async, d2d, memset, event_record, gemm, NCCL)
 * goes to the "current" stream: the runtime's own stream unless
 * grumpy_rt_set_stream selected another (0 selects the runtime's again). */
int grumpy_rt_stream_create(uint64_t* stream);
int grumpy_rt_stream_destroy(uint64_t stream);
int grumpy_rt_set_stream(uint64_t stream);
/* the current stream waits for `ev` (recorded on any stream) */
int grumpy_rt_stream_wait_event(uint64_t ev);
/* asynchronous D2H on the current stream (dst should be page-locked) */
int grumpy_rt_d2h_async(void* dst, uint64_t src, size_t bytes);
int grumpy_rt_event_sync(uint64_t ev);

/* ---- events (device timing) ------------------------------------------- */
int grumpy_rt_event_create(uint64_t* ev);
int grumpy_rt_event_record(uint64_t ev);
int grumpy_rt_event_elapsed(uint64_t ev_start, uint64_t ev_end, float* ms);
int grumpy_rt_event_destroy(uint64_t ev);

/* ---- run_library: gemm / gemv with transpose flags (
 *      PAPER.md:292-303 cuBLAS).  Row-major semantics:
 *      C[m,n] = op(A)[m,k] * op(B)[k,n];  lda/ldb/ldc are row strides. ---- */
/* FP32 GEMM arithmetic: 0 = FP32 on the CUDA cores (default), 1 = FP32
 * emulated with BF16x9 tensor-core products (cuBLAS 12.9, FP32 accuracy). */
int grumpy_rt_set_gemm_math(int mode);
/* cuBLASLt f32 GEMM with a fused epilogue: row-major C[m,n] = epi(op(A)op(B)
 * + bias[n]), epilogue 0 none / 1 bias / 2 relu(bias) — the library-side
 * alternative to the R1 bias+ReLU region;
 * emulate = 1 uses BF16x9 emulated FP32, 2 only where it pays (m, n >= 128),
 * the rule grumpy_rt_gemm applies in emulation mode. */
int grumpy_rt_gemm_epilogue(int trans_a, int trans_b, int m, int n, int k, uint64_t a, int lda,
                            uint64_t b, int ldb, uint64_t c, int ldc, uint64_t bias, int epilogue,
                            int emulate);
int grumpy_rt_gemm(int trans_a, int trans_b, int m, int n, int k, int dtype,
                   uint64_t a, int lda, uint64_t b, int ldb, uint64_t c, int ldc);
/* y[m] = op(A) x, A row-major [rows, cols] (ld = row stride);
 * trans = 0: m = rows, x has cols entries; trans = 1: m = cols. */
int grumpy_rt_gemv(int trans, int rows, int cols, int dtype, uint64_t a, int lda,
                   uint64_t x, uint64_t y);

/* ---- NCCL (leading-axis sharding; allreduce of reduction partials) ------ */
int grumpy_rt_nccl_load(const char* libnccl_path);
int grumpy_rt_nccl_unique_id(char* id128);
int grumpy_rt_nccl_init(int rank, int nranks, const char* id128);
int grumpy_rt_nccl_allreduce(uint64_t send, uint64_t recv, size_t count, int dtype, int op);
int grumpy_rt_nccl_allgather(uint64_t send, uint64_t recv, size_t count_per_rank, int dtype);
/* ncclGroupStart/End around the collectives of one plan step (one launch) */
int grumpy_rt_nccl_group_start(void);
int grumpy_rt_nccl_group_end(void);
int grumpy_rt_nccl_destroy(void);

#ifdef __cplusplus
}
#endif
#endif /* GRUMPY_RT_H_ */
