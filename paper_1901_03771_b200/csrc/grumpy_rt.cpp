// libgrumpy_rt.so — C-ABI runtime shim for the fused-region path.
//
// Declared in include/grumpy_rt.h (which cites the reference interfaces each
// export replaces).  Design:
//   * CUDA driver API, loaded with dlopen("libcuda.so.1") + cuGetProcAddress so
//     the library itself loads on machines without a driver (CPU CI checks the
//     exports) and fails with GR_ENOINIT only when used;
//   * one device, its primary context and ONE non-blocking stream per process
//     (one process per GPU); kernels, copies, cuBLAS and NCCL all run on it, so
//     stream order is the only synchronisation the pool needs;
//   * NVRTC → cubin → cuModuleLoadData, cached in-process and on disk;
//   * a caching device allocator with size classes;
//   * cuBLAS for run_library (linked), NCCL via dlopen.
#include "../../include/grumpy_rt.h"

#include <cuda.h>
#include <cublasLt.h>
#include <cublas_v2.h>
#include <dlfcn.h>
#include <nvrtc.h>
#include <nvtx3/nvToolsExt.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <sys/stat.h>
#include <unistd.h>
#include <unordered_map>
#include <vector>

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

// ---------------------------------------------------------------------------
// Driver API table (resolved with cuGetProcAddress)
// ---------------------------------------------------------------------------
#define GR_CU_FUNCS(X)               \
  X(cuInit)                          \
  X(cuDeviceGetCount)                \
  X(cuDeviceGet)                     \
  X(cuDeviceGetAttribute)            \
  X(cuDeviceGetName)                 \
  X(cuDeviceTotalMem)                \
  X(cuDevicePrimaryCtxRetain)        \
  X(cuCtxSetCurrent)                 \
  X(cuStreamCreate)                  \
  X(cuStreamSynchronize)             \
  X(cuStreamDestroy)                 \
  X(cuStreamWaitEvent)               \
  X(cuCtxSynchronize)                \
  X(cuMemAlloc)                      \
  X(cuMemFree)                       \
  X(cuMemcpyHtoDAsync)               \
  X(cuMemcpyDtoHAsync)               \
  X(cuMemcpyDtoDAsync)               \
  X(cuMemsetD8Async)                 \
  X(cuMemHostAlloc)                  \
  X(cuMemFreeHost)                   \
  X(cuMemHostRegister)               \
  X(cuMemHostUnregister)             \
  X(cuModuleLoadData)                \
  X(cuModuleGetFunction)             \
  X(cuModuleGetGlobal)               \
  X(cuTensorMapEncodeTiled)          \
  X(cuFuncGetAttribute)              \
  X(cuFuncSetAttribute)              \
  X(cuOccupancyMaxActiveBlocksPerMultiprocessor) \
  X(cuLaunchKernel)                  \
  X(cuLaunchKernelEx)                \
  X(cuEventCreate)                   \
  X(cuEventRecord)                   \
  X(cuEventSynchronize)              \
  X(cuEventElapsedTime)              \
  X(cuEventDestroy)                  \
  X(cuGetErrorString)

#define GR_DECL(name) decltype(&::name) p_##name = nullptr;
struct Driver {
  GR_CU_FUNCS(GR_DECL)
  void* handle = nullptr;
  bool loaded = false;
};
#undef GR_DECL
Driver D;

struct State {
  bool init = false;
  int device = -1;
  CUdevice dev = 0;
  CUcontext ctx = nullptr;
  CUstream stream = nullptr;
  CUstream cur = nullptr;   // stream async work goes to (nullptr: `stream`)
  int sm_count = 0;
  cublasHandle_t cublas = nullptr;
  cublasLtHandle_t lt = nullptr;
  CUdeviceptr lt_ws = 0;          // cuBLASLt workspace
  size_t lt_ws_bytes = 0;
  int gemm_math = 0;              // 0 FP32 (SIMT), 1 FP32 emulated with BF16x9 tensor-core products
  std::mutex mu;
} S;

std::string cu_msg(CUresult r, const char* what) {
  const char* s = nullptr;
  if (D.p_cuGetErrorString) D.p_cuGetErrorString(r, &s);
  char buf[512];
  snprintf(buf, sizeof(buf), "%s failed: CUresult %d (%s)", what, (int)r, s ? s : "?");
  return buf;
}

#define CU_CHECK(call, what)                                 \
  do {                                                       \
    CUresult _r = (call);                                    \
    if (_r != CUDA_SUCCESS) return fail(GR_ECUDA, cu_msg(_r, what)); \
  } while (0)

int load_driver() {
  if (D.loaded) return GR_OK;
  D.handle = dlopen("libcuda.so.1", RTLD_NOW | RTLD_GLOBAL);
  if (!D.handle) return fail(GR_EDLOPEN, std::string("dlopen(libcuda.so.1): ") + dlerror());
  using GetProc = CUresult (*)(const char*, void**, int, cuuint64_t, CUdriverProcAddressQueryResult*);
  auto gp = (GetProc)dlsym(D.handle, "cuGetProcAddress_v2");
  if (!gp) return fail(GR_EDLOPEN, "libcuda.so.1 has no cuGetProcAddress_v2");
#define GR_RESOLVE(name)                                                           \
  {                                                                                \
    void* fp = nullptr;                                                            \
    CUdriverProcAddressQueryResult st;                                             \
    CUresult r = gp(#name, &fp, 12080, CU_GET_PROC_ADDRESS_DEFAULT, &st);          \
    if (r != CUDA_SUCCESS || !fp) return fail(GR_EDLOPEN, "cannot resolve " #name); \
    D.p_##name = (decltype(D.p_##name))fp;                                         \
  }
  GR_CU_FUNCS(GR_RESOLVE)
#undef GR_RESOLVE
  D.loaded = true;
  return GR_OK;
}

static inline CUstream CS() { return S.cur ? S.cur : S.stream; }

int need_init() {
  if (!S.init) return fail(GR_ENOINIT, "grumpy_rt_init has not been called");
  CUresult r = D.p_cuCtxSetCurrent(S.ctx);
  if (r != CUDA_SUCCESS) return fail(GR_ECUDA, cu_msg(r, "cuCtxSetCurrent"));
  return GR_OK;
}

// ---------------------------------------------------------------------------
// Caching allocator.  Sizes are rounded to classes (256 B .. 1 MiB powers of
// two, then 2 MiB multiples) so iterative workloads with fixed shapes hit the
// cache exactly; large blocks may be reused with <= 1/8 slack.  Blocks return
// to the cache on free; ordering is guaranteed by the single stream.
// ---------------------------------------------------------------------------
struct Pool {
  std::multimap<size_t, CUdeviceptr> free_blocks;
  std::unordered_map<CUdeviceptr, size_t> live;
  size_t in_use = 0, cached = 0, peak = 0, n_allocs = 0;
} P;

size_t round_size(size_t b) {
  if (b == 0) b = 1;
  if (b <= (1u << 20)) {
    size_t s = 256;
    while (s < b) s <<= 1;
    return s;
  }
  const size_t two_mib = size_t(2) << 20;
  return (b + two_mib - 1) / two_mib * two_mib;
}

int pool_release_cached() {
  for (auto& kv : P.free_blocks) D.p_cuMemFree(kv.second);
  P.free_blocks.clear();
  P.cached = 0;
  return GR_OK;
}

// ---------------------------------------------------------------------------
// NVRTC module cache
// ---------------------------------------------------------------------------
uint64_t fnv1a(const void* data, size_t n, uint64_t h = 1469598103934665603ull) {
  const unsigned char* p = (const unsigned char*)data;
  for (size_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 1099511628211ull;
  }
  return h;
}
std::unordered_map<uint64_t, CUmodule> g_modules;

bool read_file(const std::string& path, std::vector<char>& out) {
  FILE* f = fopen(path.c_str(), "rb");
  if (!f) return false;
  fseek(f, 0, SEEK_END);
  long n = ftell(f);
  fseek(f, 0, SEEK_SET);
  out.resize(n > 0 ? (size_t)n : 0);
  bool ok = n > 0 && fread(out.data(), 1, (size_t)n, f) == (size_t)n;
  fclose(f);
  return ok;
}

void write_file_atomic(const std::string& path, const std::vector<char>& data) {
  std::string tmp = path + ".tmp." + std::to_string(getpid());
  FILE* f = fopen(tmp.c_str(), "wb");
  if (!f) return;
  bool ok = fwrite(data.data(), 1, data.size(), f) == data.size();
  fclose(f);
  if (ok) rename(tmp.c_str(), path.c_str());
  else unlink(tmp.c_str());
}


// NVRTC source -> cubin (no device needed)
int nvrtc_compile(const char* src, const char* const* opts, int n_opts, std::vector<char>& cubin, double* ms) {
  auto t0 = std::chrono::steady_clock::now();
  nvrtcProgram prog;
  nvrtcResult nr = nvrtcCreateProgram(&prog, src, "grumpy_region.cu", 0, nullptr, nullptr);
  if (nr != NVRTC_SUCCESS) return fail(GR_ENVRTC, std::string("nvrtcCreateProgram: ") + nvrtcGetErrorString(nr));
  nr = nvrtcCompileProgram(prog, n_opts, opts);
  if (nr != NVRTC_SUCCESS) {
    size_t log_size = 0;
    nvrtcGetProgramLogSize(prog, &log_size);
    std::string log(log_size, '\0');
    if (log_size) nvrtcGetProgramLog(prog, &log[0]);
    nvrtcDestroyProgram(&prog);
    return fail(GR_ENVRTC, std::string("NVRTC compile failed: ") + nvrtcGetErrorString(nr) + "\n" + log);
  }
  size_t n = 0;
  nr = nvrtcGetCUBINSize(prog, &n);
  if (nr != NVRTC_SUCCESS || n == 0) {
    nvrtcDestroyProgram(&prog);
    return fail(GR_ENVRTC, "nvrtcGetCUBINSize failed (is --gpu-architecture=sm_100a set?)");
  }
  cubin.resize(n);
  nvrtcGetCUBIN(prog, cubin.data());
  nvrtcDestroyProgram(&prog);
  auto t1 = std::chrono::steady_clock::now();
  if (ms) *ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
  return GR_OK;
}

// ---------------------------------------------------------------------------
// NCCL via dlopen
// ---------------------------------------------------------------------------
struct NcclUid { char internal[128]; };
typedef void* NcclComm;
struct Nccl {
  void* handle = nullptr;
  int (*GetUniqueId)(NcclUid*) = nullptr;
  int (*CommInitRank)(NcclComm*, int, NcclUid, int) = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, NcclComm, CUstream) = nullptr;
  int (*AllGather)(const void*, void*, size_t, int, NcclComm, CUstream) = nullptr;
  int (*CommDestroy)(NcclComm) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
  NcclComm comm = nullptr;
} N;

// ncclDataType_t / ncclRedOp_t values (nccl.h)
int nccl_dtype(int gr) {
  switch (gr) {
    case GR_F32: return 7;   // ncclFloat32
    case GR_F64: return 8;   // ncclFloat64
    case GR_I32: return 2;   // ncclInt32
    case GR_I64: return 4;   // ncclInt64
    case GR_BOOL: return 0;  // ncclInt8
  }
  return -1;
}

int nccl_fail(int r, const char* what) {
  std::string s = std::string(what) + " failed: ncclResult " + std::to_string(r);
  if (N.GetErrorString) s += std::string(" (") + N.GetErrorString(r) + ")";
  return fail(GR_ENCCL, s);
}

size_t dtype_size(int dt) {
  switch (dt) {
    case GR_F32: case GR_I32: return 4;
    case GR_F64: case GR_I64: return 8;
    case GR_BOOL: return 1;
  }
  return 0;
}

}  // namespace

extern "C" {

int grumpy_rt_version(int* version) {
  if (version) *version = 1;
  return GR_OK;
}

const char* grumpy_rt_last_error(void) { return g_err.c_str(); }

int grumpy_rt_device_count(int* count) {
  int r = load_driver();
  if (r) return r;
  CU_CHECK(D.p_cuInit(0), "cuInit");
  int n = 0;
  CU_CHECK(D.p_cuDeviceGetCount(&n), "cuDeviceGetCount");
  *count = n;
  return GR_OK;
}

int grumpy_rt_init(int device) {
  std::lock_guard<std::mutex> lk(S.mu);
  if (S.init) {
    if (device != S.device)
      return fail(GR_EINVAL, "runtime already initialised on device " + std::to_string(S.device));
    return need_init();
  }
  int r = load_driver();
  if (r) return r;
  CU_CHECK(D.p_cuInit(0), "cuInit");
  int n = 0;
  CU_CHECK(D.p_cuDeviceGetCount(&n), "cuDeviceGetCount");
  if (device < 0 || device >= n)
    return fail(GR_ENOINIT, "device " + std::to_string(device) + " not present (" + std::to_string(n) + " devices)");
  CU_CHECK(D.p_cuDeviceGet(&S.dev, device), "cuDeviceGet");
  CU_CHECK(D.p_cuDevicePrimaryCtxRetain(&S.ctx, S.dev), "cuDevicePrimaryCtxRetain");
  CU_CHECK(D.p_cuCtxSetCurrent(S.ctx), "cuCtxSetCurrent");
  CU_CHECK(D.p_cuStreamCreate(&S.stream, CU_STREAM_NON_BLOCKING), "cuStreamCreate");
  CU_CHECK(D.p_cuDeviceGetAttribute(&S.sm_count, CU_DEVICE_ATTRIBUTE_MULTIPROCESSOR_COUNT, S.dev),
           "cuDeviceGetAttribute");
  S.device = device;
  S.init = true;
  return GR_OK;
}

int grumpy_rt_device_info(int* sm_count, int* cc_major, int* cc_minor, size_t* total_mem, char* name) {
  int r = need_init();
  if (r) return r;
  if (sm_count) *sm_count = S.sm_count;
  if (cc_major) CU_CHECK(D.p_cuDeviceGetAttribute(cc_major, CU_DEVICE_ATTRIBUTE_COMPUTE_CAPABILITY_MAJOR, S.dev), "attr");
  if (cc_minor) CU_CHECK(D.p_cuDeviceGetAttribute(cc_minor, CU_DEVICE_ATTRIBUTE_COMPUTE_CAPABILITY_MINOR, S.dev), "attr");
  if (total_mem) CU_CHECK(D.p_cuDeviceTotalMem(total_mem, S.dev), "cuDeviceTotalMem");
  if (name) CU_CHECK(D.p_cuDeviceGetName(name, 255, S.dev), "cuDeviceGetName");
  return GR_OK;
}

int grumpy_rt_stream(uint64_t* stream) {
  int r = need_init();
  if (r) return r;
  *stream = (uint64_t)(uintptr_t)S.stream;
  return GR_OK;
}

// ---- pool -------------------------------------------------------------------
int grumpy_rt_alloc(size_t bytes, uint64_t* dptr) {
  int r = need_init();
  if (r) return r;
  std::lock_guard<std::mutex> lk(S.mu);
  size_t sz = round_size(bytes);
  auto it = P.free_blocks.lower_bound(sz);
  if (it != P.free_blocks.end() && (it->first == sz || (sz > (1u << 20) && it->first <= sz + sz / 8))) {
    CUdeviceptr p = it->second;
    size_t bsz = it->first;
    P.free_blocks.erase(it);
    P.cached -= bsz;
    P.live[p] = bsz;
    P.in_use += bsz;
    if (P.in_use > P.peak) P.peak = P.in_use;
    *dptr = (uint64_t)p;
    return GR_OK;
  }
  CUdeviceptr p = 0;
  CUresult cr = D.p_cuMemAlloc(&p, sz);
  if (cr == CUDA_ERROR_OUT_OF_MEMORY) {
    D.p_cuCtxSynchronize();
    pool_release_cached();
    cr = D.p_cuMemAlloc(&p, sz);
  }
  if (cr == CUDA_ERROR_OUT_OF_MEMORY)
    return fail(GR_ENOMEM, "device out of memory allocating " + std::to_string(sz) + " bytes (in use " +
                               std::to_string(P.in_use) + ")");
  if (cr != CUDA_SUCCESS) return fail(GR_ECUDA, cu_msg(cr, "cuMemAlloc"));
  P.live[p] = sz;
  P.in_use += sz;
  P.n_allocs += 1;
  if (P.in_use > P.peak) P.peak = P.in_use;
  *dptr = (uint64_t)p;
  return GR_OK;
}

int grumpy_rt_free(uint64_t dptr) {
  if (!S.init) return GR_OK;  // interpreter shutdown after teardown
  std::lock_guard<std::mutex> lk(S.mu);
  auto it = P.live.find((CUdeviceptr)dptr);
  if (it == P.live.end()) return fail(GR_EINVAL, "free of unknown pointer");
  size_t sz = it->second;
  P.live.erase(it);
  P.in_use -= sz;
  P.free_blocks.emplace(sz, (CUdeviceptr)dptr);
  P.cached += sz;
  return GR_OK;
}

int grumpy_rt_pool_stats(size_t* in_use, size_t* cached, size_t* peak, size_t* n_allocs) {
  std::lock_guard<std::mutex> lk(S.mu);
  if (in_use) *in_use = P.in_use;
  if (cached) *cached = P.cached;
  if (peak) *peak = P.peak;
  if (n_allocs) *n_allocs = P.n_allocs;
  return GR_OK;
}

int grumpy_rt_pool_trim(void) {
  int r = need_init();
  if (r) return r;
  CU_CHECK(D.p_cuCtxSynchronize(), "cuCtxSynchronize");
  std::lock_guard<std::mutex> lk(S.mu);
  return pool_release_cached();
}

// ---- transfers ----------------------------------------------------------------
int grumpy_rt_h2d(uint64_t dst, const void* src, size_t bytes) {
  int r = need_init();
  if (r) return r;
  if (!bytes) return GR_OK;
  CU_CHECK(D.p_cuMemcpyHtoDAsync((CUdeviceptr)dst, src, bytes, CS()), "cuMemcpyHtoDAsync");
  return GR_OK;
}

int grumpy_rt_d2h(void* dst, uint64_t src, size_t bytes) {
  int r = need_init();
  if (r) return r;
  if (bytes) CU_CHECK(D.p_cuMemcpyDtoHAsync(dst, (CUdeviceptr)src, bytes, CS()), "cuMemcpyDtoHAsync");
  CU_CHECK(D.p_cuStreamSynchronize(CS()), "cuStreamSynchronize");
  return GR_OK;
}

int grumpy_rt_d2d(uint64_t dst, uint64_t src, size_t bytes) {
  int r = need_init();
  if (r) return r;
  if (!bytes) return GR_OK;
  CU_CHECK(D.p_cuMemcpyDtoDAsync((CUdeviceptr)dst, (CUdeviceptr)src, bytes, CS()), "cuMemcpyDtoDAsync");
  return GR_OK;
}

int grumpy_rt_memset(uint64_t dst, int byte_value, size_t bytes) {
  int r = need_init();
  if (r) return r;
  if (!bytes) return GR_OK;
  CU_CHECK(D.p_cuMemsetD8Async((CUdeviceptr)dst, (unsigned char)byte_value, bytes, CS()), "cuMemsetD8Async");
  return GR_OK;
}

int grumpy_rt_host_alloc(size_t bytes, void** ptr) {
  int r = need_init();
  if (r) return r;
  CU_CHECK(D.p_cuMemHostAlloc(ptr, bytes ? bytes : 1, CU_MEMHOSTALLOC_PORTABLE), "cuMemHostAlloc");
  return GR_OK;
}

int grumpy_rt_host_free(void* ptr) {
  int r = need_init();
  if (r) return r;
  CU_CHECK(D.p_cuMemFreeHost(ptr), "cuMemFreeHost");
  return GR_OK;
}

int grumpy_rt_host_register(void* ptr, size_t bytes) {
  int r = need_init();
  if (r) return r;
  CU_CHECK(D.p_cuMemHostRegister(ptr, bytes, CU_MEMHOSTREGISTER_PORTABLE), "cuMemHostRegister");
  return GR_OK;
}

int grumpy_rt_host_unregister(void* ptr) {
  int r = need_init();
  if (r) return r;
  CU_CHECK(D.p_cuMemHostUnregister(ptr), "cuMemHostUnregister");
  return GR_OK;
}

// ---- compile ------------------------------------------------------------------
static uint64_t source_key(const char* src, const char* const* opts, int n_opts) {
  uint64_t h = fnv1a(src, strlen(src));
  for (int i = 0; i < n_opts; ++i) {
    h = fnv1a(opts[i], strlen(opts[i]), h);
    h = fnv1a("\x1f", 1, h);
  }
  int nv_major = 0, nv_minor = 0;
  nvrtcVersion(&nv_major, &nv_minor);
  h = fnv1a(&nv_major, sizeof(nv_major), h);
  h = fnv1a(&nv_minor, sizeof(nv_minor), h);
  return h;
}

// cubins compiled ahead of their first launch (grumpy_rt_precompile), by key
static std::unordered_map<uint64_t, std::vector<char>> g_cubins;
static std::mutex g_cubins_mu;

int grumpy_rt_precompile(const char* src, const char* const* opts, int n_opts, const char* cache_dir,
                         double* compile_ms) {
  // NVRTC only — no CUDA context needed, safe to call from worker threads
  if (compile_ms) *compile_ms = 0.0;
  const uint64_t h = source_key(src, opts, n_opts);
  {
    std::lock_guard<std::mutex> lk(S.mu);
    if (g_modules.count(h)) return GR_OK;
  }
  {
    std::lock_guard<std::mutex> lk(g_cubins_mu);
    if (g_cubins.count(h)) return GR_OK;
  }
  char key[32];
  snprintf(key, sizeof(key), "%016llx", (unsigned long long)h);
  std::string path;
  std::vector<char> cubin;
  if (cache_dir && cache_dir[0]) {
    path = std::string(cache_dir) + "/" + key + ".cubin";
    if (read_file(path, cubin)) return GR_OK;     // the loader reads it from disk
  }
  int rc = nvrtc_compile(src, opts, n_opts, cubin, compile_ms);
  if (rc) return rc;
  if (!path.empty()) {
    mkdir(cache_dir, 0755);
    write_file_atomic(path, cubin);
  }
  std::lock_guard<std::mutex> lk(g_cubins_mu);
  g_cubins[h] = std::move(cubin);
  return GR_OK;
}

int grumpy_rt_compile(const char* src, const char* const* opts, int n_opts, const char* cache_dir,
                      uint64_t* module, double* compile_ms, int* cache_hit) {
  int r = need_init();
  if (r) return r;
  if (compile_ms) *compile_ms = 0.0;
  if (cache_hit) *cache_hit = 0;
  const uint64_t h = source_key(src, opts, n_opts);
  {
    std::lock_guard<std::mutex> lk(S.mu);
    auto it = g_modules.find(h);
    if (it != g_modules.end()) {
      *module = (uint64_t)(uintptr_t)it->second;
      if (cache_hit) *cache_hit = 1;
      return GR_OK;
    }
  }
  char key[32];
  snprintf(key, sizeof(key), "%016llx", (unsigned long long)h);
  std::string path;
  std::vector<char> cubin;
  bool have = false;
  {
    std::lock_guard<std::mutex> lk(g_cubins_mu);
    auto it = g_cubins.find(h);
    if (it != g_cubins.end()) {
      cubin = std::move(it->second);
      g_cubins.erase(it);
      have = true;
      if (cache_hit) *cache_hit = 3;
    }
  }
  if (!have && cache_dir && cache_dir[0]) {
    path = std::string(cache_dir) + "/" + key + ".cubin";
    have = read_file(path, cubin);
    if (have && cache_hit) *cache_hit = 2;
  }
  if (!have) {
    int rc = nvrtc_compile(src, opts, n_opts, cubin, compile_ms);
    if (rc) return rc;
    if (!path.empty()) {
      mkdir(cache_dir, 0755);
      write_file_atomic(path, cubin);
    }
  }
  CUmodule mod;
  CU_CHECK(D.p_cuModuleLoadData(&mod, cubin.data()), "cuModuleLoadData");
  {
    std::lock_guard<std::mutex> lk(S.mu);
    g_modules[h] = mod;
  }
  *module = (uint64_t)(uintptr_t)mod;
  return GR_OK;
}

int grumpy_rt_compile_cubin(const char* src, const char* const* opts, int n_opts, void* out, size_t cap,
                            size_t* size, double* compile_ms) {
  std::vector<char> cubin;
  int rc = nvrtc_compile(src, opts, n_opts, cubin, compile_ms);
  if (rc) return rc;
  *size = cubin.size();
  if (out && cap >= cubin.size()) memcpy(out, cubin.data(), cubin.size());
  return GR_OK;
}

int grumpy_rt_get_function(uint64_t module, const char* name, uint64_t* fn) {
  int r = need_init();
  if (r) return r;
  CUfunction f;
  CU_CHECK(D.p_cuModuleGetFunction(&f, (CUmodule)(uintptr_t)module, name), "cuModuleGetFunction");
  *fn = (uint64_t)(uintptr_t)f;
  return GR_OK;
}

int grumpy_rt_module_global(uint64_t module, const char* name, uint64_t* dptr, size_t* bytes) {
  int r = need_init();
  if (r) return r;
  CUdeviceptr p = 0;
  size_t n = 0;
  CU_CHECK(D.p_cuModuleGetGlobal(&p, &n, (CUmodule)(uintptr_t)module, name), "cuModuleGetGlobal");
  *dptr = (uint64_t)p;
  if (bytes) *bytes = n;
  return GR_OK;
}

int grumpy_rt_tensor_map_2d(uint64_t gaddr, int dtype, uint64_t dim0, uint64_t dim1, uint64_t stride1,
                            unsigned box0, unsigned box1, int swizzle, void* out128) {
  int r = load_driver();
  if (r) return r;
  CUtensorMapDataType dt;
  switch (dtype) {
    case GR_F32: dt = CU_TENSOR_MAP_DATA_TYPE_FLOAT32; break;
    case GR_F64: dt = CU_TENSOR_MAP_DATA_TYPE_FLOAT64; break;
    case GR_I32: dt = CU_TENSOR_MAP_DATA_TYPE_INT32; break;
    case GR_I64: dt = CU_TENSOR_MAP_DATA_TYPE_INT64; break;
    case GR_BOOL: dt = CU_TENSOR_MAP_DATA_TYPE_UINT8; break;
    default: return fail(GR_EINVAL, "tensor map: bad dtype");
  }
  CUtensorMapSwizzle sw;
  switch (swizzle) {
    case 0: sw = CU_TENSOR_MAP_SWIZZLE_NONE; break;
    case 32: sw = CU_TENSOR_MAP_SWIZZLE_32B; break;
    case 64: sw = CU_TENSOR_MAP_SWIZZLE_64B; break;
    case 128: sw = CU_TENSOR_MAP_SWIZZLE_128B; break;
    default: return fail(GR_EINVAL, "tensor map: swizzle must be 0, 32, 64 or 128");
  }
  const cuuint64_t dims[2] = {dim0, dim1};
  const cuuint64_t strides[1] = {stride1};
  const cuuint32_t box[2] = {box0, box1};
  const cuuint32_t estr[2] = {1, 1};
  CUtensorMap m;
  CU_CHECK(D.p_cuTensorMapEncodeTiled(&m, dt, 2, (void*)(uintptr_t)gaddr, dims, strides, box, estr,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE),
           "cuTensorMapEncodeTiled");
  memcpy(out128, &m, sizeof(m));
  return GR_OK;
}

int grumpy_rt_function_info(uint64_t fn, int* num_regs, int* local_bytes, int* static_smem, int* max_threads) {
  int r = need_init();
  if (r) return r;
  CUfunction f = (CUfunction)(uintptr_t)fn;
  if (num_regs) CU_CHECK(D.p_cuFuncGetAttribute(num_regs, CU_FUNC_ATTRIBUTE_NUM_REGS, f), "attr");
  if (local_bytes) CU_CHECK(D.p_cuFuncGetAttribute(local_bytes, CU_FUNC_ATTRIBUTE_LOCAL_SIZE_BYTES, f), "attr");
  if (static_smem) CU_CHECK(D.p_cuFuncGetAttribute(static_smem, CU_FUNC_ATTRIBUTE_SHARED_SIZE_BYTES, f), "attr");
  if (max_threads) CU_CHECK(D.p_cuFuncGetAttribute(max_threads, CU_FUNC_ATTRIBUTE_MAX_THREADS_PER_BLOCK, f), "attr");
  return GR_OK;
}

// Kernels that stage through dynamic shared memory (bulk-copy rings) get the
// whole unified L1/shared array as shared memory; the others keep the default
// carve-out (maximum L1 for their LDG streams).
static int smem_attrs(CUfunction f, size_t dyn_smem) {
  // opt in whenever dynamic + static shared memory may pass the 48 KB default
  if (dyn_smem > 32 * 1024)
    CU_CHECK(D.p_cuFuncSetAttribute(f, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, (int)dyn_smem), "attr");
  if (dyn_smem > 0)
    CU_CHECK(D.p_cuFuncSetAttribute(f, CU_FUNC_ATTRIBUTE_PREFERRED_SHARED_MEMORY_CARVEOUT, 100), "attr");
  return GR_OK;
}

int grumpy_rt_occupancy(uint64_t fn, int block, size_t dyn_smem, int* blocks_per_sm) {
  int r = need_init();
  if (r) return r;
  CUfunction f = (CUfunction)(uintptr_t)fn;
  r = smem_attrs(f, dyn_smem);
  if (r) return r;
  CU_CHECK(D.p_cuOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, f, block, dyn_smem), "occupancy");
  return GR_OK;
}

// ---- launch -----------------------------------------------------------------
int grumpy_rt_launch(uint64_t fn, unsigned gx, unsigned gy, unsigned gz, unsigned bx, unsigned by, unsigned bz,
                     unsigned dyn_smem, unsigned cluster_x, const void* params, size_t params_size) {
  int r = need_init();
  if (r) return r;
  CUfunction f = (CUfunction)(uintptr_t)fn;
  r = smem_attrs(f, dyn_smem);
  if (r) return r;
  size_t sz = params_size;
  void* extra[] = {CU_LAUNCH_PARAM_BUFFER_POINTER, const_cast<void*>(params), CU_LAUNCH_PARAM_BUFFER_SIZE, &sz,
                   CU_LAUNCH_PARAM_END};
  if (cluster_x > 1) {
    CUlaunchConfig cfg;
    memset(&cfg, 0, sizeof(cfg));
    cfg.gridDimX = gx; cfg.gridDimY = gy; cfg.gridDimZ = gz;
    cfg.blockDimX = bx; cfg.blockDimY = by; cfg.blockDimZ = bz;
    cfg.sharedMemBytes = dyn_smem;
    cfg.hStream = CS();
    CUlaunchAttribute attr;
    memset(&attr, 0, sizeof(attr));
    attr.id = CU_LAUNCH_ATTRIBUTE_CLUSTER_DIMENSION;
    attr.value.clusterDim.x = cluster_x;
    attr.value.clusterDim.y = 1;
    attr.value.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    CU_CHECK(D.p_cuLaunchKernelEx(&cfg, f, nullptr, extra), "cuLaunchKernelEx");
    return GR_OK;
  }
  CU_CHECK(D.p_cuLaunchKernel(f, gx, gy, gz, bx, by, bz, dyn_smem, CS(), nullptr, extra), "cuLaunchKernel");
  return GR_OK;
}

int grumpy_rt_sync(void) {
  int r = need_init();
  if (r) return r;
  CU_CHECK(D.p_cuCtxSynchronize(), "cuCtxSynchronize");
  return GR_OK;
}

// ---- profiler ranges ----------------------------------------------------------
int grumpy_rt_range_push(const char* name) {
  nvtxRangePushA(name ? name : "");
  return GR_OK;
}

int grumpy_rt_range_pop(void) {
  nvtxRangePop();
  return GR_OK;
}

// ---- streams (copy/compute overlap of streamed materialisation) --------------
int grumpy_rt_stream_create(uint64_t* stream) {
  int r = need_init();
  if (r) return r;
  CUstream st;
  CU_CHECK(D.p_cuStreamCreate(&st, CU_STREAM_NON_BLOCKING), "cuStreamCreate");
  *stream = (uint64_t)(uintptr_t)st;
  return GR_OK;
}

int grumpy_rt_stream_destroy(uint64_t stream) {
  if (!S.init || !stream) return GR_OK;
  if (S.cur == (CUstream)(uintptr_t)stream) S.cur = nullptr;
  CU_CHECK(D.p_cuStreamDestroy((CUstream)(uintptr_t)stream), "cuStreamDestroy");
  return GR_OK;
}

int grumpy_rt_set_stream(uint64_t stream) {
  int r = need_init();
  if (r) return r;
  S.cur = (CUstream)(uintptr_t)stream;
  if (S.cublas) cublasSetStream(S.cublas, CS());
  return GR_OK;
}

int grumpy_rt_stream_wait_event(uint64_t ev) {
  int r = need_init();
  if (r) return r;
  CU_CHECK(D.p_cuStreamWaitEvent(CS(), (CUevent)(uintptr_t)ev, 0), "cuStreamWaitEvent");
  return GR_OK;
}

int grumpy_rt_d2h_async(void* dst, uint64_t src, size_t bytes) {
  int r = need_init();
  if (r) return r;
  if (bytes) CU_CHECK(D.p_cuMemcpyDtoHAsync(dst, (CUdeviceptr)src, bytes, CS()), "cuMemcpyDtoHAsync");
  return GR_OK;
}

int grumpy_rt_event_sync(uint64_t ev) {
  int r = need_init();
  if (r) return r;
  CU_CHECK(D.p_cuEventSynchronize((CUevent)(uintptr_t)ev), "cuEventSynchronize");
  return GR_OK;
}

// ---- events -------------------------------------------------------------------
int grumpy_rt_event_create(uint64_t* ev) {
  int r = need_init();
  if (r) return r;
  CUevent e;
  CU_CHECK(D.p_cuEventCreate(&e, CU_EVENT_DEFAULT), "cuEventCreate");
  *ev = (uint64_t)(uintptr_t)e;
  return GR_OK;
}

int grumpy_rt_event_record(uint64_t ev) {
  int r = need_init();
  if (r) return r;
  CU_CHECK(D.p_cuEventRecord((CUevent)(uintptr_t)ev, CS()), "cuEventRecord");
  return GR_OK;
}

int grumpy_rt_event_elapsed(uint64_t ev_start, uint64_t ev_end, float* ms) {
  int r = need_init();
  if (r) return r;
  CU_CHECK(D.p_cuEventSynchronize((CUevent)(uintptr_t)ev_end), "cuEventSynchronize");
  CU_CHECK(D.p_cuEventElapsedTime(ms, (CUevent)(uintptr_t)ev_start, (CUevent)(uintptr_t)ev_end),
           "cuEventElapsedTime");
  return GR_OK;
}

int grumpy_rt_event_destroy(uint64_t ev) {
  if (!S.init) return GR_OK;
  CU_CHECK(D.p_cuEventDestroy((CUevent)(uintptr_t)ev), "cuEventDestroy");
  return GR_OK;
}

// ---- cuBLAS -------------------------------------------------------------------
static void apply_gemm_math();
static int ensure_cublas() {
  if (S.cublas) return GR_OK;
  cublasStatus_t st = cublasCreate(&S.cublas);
  if (st != CUBLAS_STATUS_SUCCESS) return fail(GR_ECUBLAS, "cublasCreate: status " + std::to_string((int)st));
  cublasSetStream(S.cublas, CS());
  // FP32 stays FP32 (no TF32): NumPy/OpenBLAS parity;
  // optionally FP32 emulated by BF16x9 products on the tensor cores
  // (grumpy_rt_set_gemm_math), which keeps FP32 accuracy.
  apply_gemm_math();
  return GR_OK;
}

// BF16x9 emulation needs cuBLAS >= 12.9.  The process may hold an older
// libcublas.so.12 (e.g. PyTorch's wheel, loaded first), so the 12.9-only
// entry point is looked up at run time instead of being linked.
typedef cublasStatus_t (*SetEmulationFn)(cublasHandle_t, cublasEmulationStrategy_t);
static SetEmulationFn emulation_fn() {
  static SetEmulationFn fn = (SetEmulationFn)dlsym(RTLD_DEFAULT, "cublasSetEmulationStrategy");
  return fn;
}
static bool emulation_available() {
  return emulation_fn() != nullptr && cublasLtGetVersion() >= 120900;
}
static void apply_gemm_math() {
  if (!S.cublas) return;
  cublasSetMathMode(S.cublas, S.gemm_math ? CUBLAS_FP32_EMULATED_BF16X9_MATH : CUBLAS_DEFAULT_MATH);
  if (emulation_fn())
    emulation_fn()(S.cublas, S.gemm_math ? (getenv("GRUMPY_EMULATION_EAGER") ? CUBLAS_EMULATION_STRATEGY_EAGER : CUBLAS_EMULATION_STRATEGY_PERFORMANT) : CUBLAS_EMULATION_STRATEGY_DEFAULT);
}

static bool gemm_emulation_pays(int m, int n) { return m >= 128 && n >= 128; }

int grumpy_rt_set_gemm_math(int mode) {
  if (mode != 0 && mode != 1) return fail(GR_EINVAL, "gemm math mode must be 0 (fp32) or 1 (bf16x9 emulation)");
  if (mode == 1 && !emulation_available())
    return fail(GR_EINVAL, "BF16x9 FP32 emulation needs cuBLAS >= 12.9 (an older libcublas.so.12 is loaded)");
  S.gemm_math = mode;
  apply_gemm_math();
  return GR_OK;
}

// cuBLASLt f32 GEMM with a fused epilogue (none / +bias / relu(+bias)):
// row-major C[m,n] = epi(op(A) op(B) + bias[n]); bias runs along C's columns.
int grumpy_rt_gemm_epilogue(int trans_a, int trans_b, int m, int n, int k, uint64_t a, int lda, uint64_t b,
                            int ldb, uint64_t c, int ldc, uint64_t bias, int epilogue, int emulate) {
  int r = need_init();
  if (r) return r;
  if (!S.lt) {
    if (cublasLtCreate(&S.lt) != CUBLAS_STATUS_SUCCESS) return fail(GR_ECUBLAS, "cublasLtCreate failed");
    S.lt_ws_bytes = 32u << 20;
    CUresult cr = D.p_cuMemAlloc(&S.lt_ws, S.lt_ws_bytes);
    if (cr != CUDA_SUCCESS) return fail(GR_ECUDA, cu_msg(cr, "cuMemAlloc (cublasLt workspace)"));
  }
  if (epilogue < 0 || epilogue > 2) return fail(GR_EINVAL, "epilogue must be 0 (none), 1 (bias), 2 (relu+bias)");
  // column-major view: C^T[n,m] = op(B)^T[n,k] op(A)^T[k,m]; the bias is per row of C^T
  cublasOperation_t opa = trans_a ? CUBLAS_OP_T : CUBLAS_OP_N;
  cublasOperation_t opb = trans_b ? CUBLAS_OP_T : CUBLAS_OP_N;
  cublasLtMatmulDesc_t desc = nullptr;
  cublasLtMatrixLayout_t la = nullptr, lb = nullptr, lc = nullptr;
  cublasLtMatmulPreference_t pref = nullptr;
  cublasStatus_t st;
  int out = GR_OK;
  if (emulate && !emulation_available())
    return fail(GR_EINVAL, "BF16x9 FP32 emulation needs cuBLAS >= 12.9 (an older libcublas.so.12 is loaded)");
  if (emulate == 2) emulate = gemm_emulation_pays(m, n);   // 2: emulate where it pays
  const cublasComputeType_t ct = emulate ? CUBLAS_COMPUTE_32F_EMULATED_16BFX9 : CUBLAS_COMPUTE_32F;
  do {
    if ((st = cublasLtMatmulDescCreate(&desc, ct, CUDA_R_32F)) != CUBLAS_STATUS_SUCCESS) break;
    cublasLtMatmulDescSetAttribute(desc, CUBLASLT_MATMUL_DESC_TRANSA, &opb, sizeof(opb));
    cublasLtMatmulDescSetAttribute(desc, CUBLASLT_MATMUL_DESC_TRANSB, &opa, sizeof(opa));
    cublasLtEpilogue_t epi = epilogue == 2 ? CUBLASLT_EPILOGUE_RELU_BIAS
                           : epilogue == 1 ? CUBLASLT_EPILOGUE_BIAS : CUBLASLT_EPILOGUE_DEFAULT;
    cublasLtMatmulDescSetAttribute(desc, CUBLASLT_MATMUL_DESC_EPILOGUE, &epi, sizeof(epi));
    if (epilogue) {
      const void* bp = (const void*)(uintptr_t)bias;
      cublasLtMatmulDescSetAttribute(desc, CUBLASLT_MATMUL_DESC_BIAS_POINTER, &bp, sizeof(bp));
      cudaDataType_t bt = CUDA_R_32F;
      cublasLtMatmulDescSetAttribute(desc, CUBLASLT_MATMUL_DESC_BIAS_DATA_TYPE, &bt, sizeof(bt));
    }
    // first operand of the column-major product: B^T (stored as row-major B)
    const int b_rows = trans_b ? k : n, b_cols = trans_b ? n : k;
    const int a_rows = trans_a ? m : k, a_cols = trans_a ? k : m;
    if ((st = cublasLtMatrixLayoutCreate(&la, CUDA_R_32F, b_rows, b_cols, ldb)) != CUBLAS_STATUS_SUCCESS) break;
    if ((st = cublasLtMatrixLayoutCreate(&lb, CUDA_R_32F, a_rows, a_cols, lda)) != CUBLAS_STATUS_SUCCESS) break;
    if ((st = cublasLtMatrixLayoutCreate(&lc, CUDA_R_32F, n, m, ldc)) != CUBLAS_STATUS_SUCCESS) break;
    if ((st = cublasLtMatmulPreferenceCreate(&pref)) != CUBLAS_STATUS_SUCCESS) break;
    cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &S.lt_ws_bytes,
                                         sizeof(S.lt_ws_bytes));
    cublasLtMatmulHeuristicResult_t heur;
    int found = 0;
    st = cublasLtMatmulAlgoGetHeuristic(S.lt, desc, la, lb, lc, lc, pref, 1, &heur, &found);
    if (st != CUBLAS_STATUS_SUCCESS) break;
    if (!found) { out = fail(GR_ECUBLAS, "cublasLt: no algorithm for this gemm/epilogue"); break; }
    const float one = 1.f, zero = 0.f;
    st = cublasLtMatmul(S.lt, desc, &one, (const void*)(uintptr_t)b, la, (const void*)(uintptr_t)a, lb, &zero,
                        (const void*)(uintptr_t)c, lc, (void*)(uintptr_t)c, lc, &heur.algo,
                        (void*)(uintptr_t)S.lt_ws, S.lt_ws_bytes, CS());
  } while (0);
  if (pref) cublasLtMatmulPreferenceDestroy(pref);
  if (lc) cublasLtMatrixLayoutDestroy(lc);
  if (lb) cublasLtMatrixLayoutDestroy(lb);
  if (la) cublasLtMatrixLayoutDestroy(la);
  if (desc) cublasLtMatmulDescDestroy(desc);
  if (out != GR_OK) return out;
  if (st != CUBLAS_STATUS_SUCCESS) return fail(GR_ECUBLAS, "cublasLt matmul: status " + std::to_string((int)st));
  return GR_OK;
}

int grumpy_rt_gemm(int trans_a, int trans_b, int m, int n, int k, int dtype, uint64_t a, int lda, uint64_t b,
                   int ldb, uint64_t c, int ldc) {
  int r = need_init();
  if (r) return r;
  r = ensure_cublas();
  if (r) return r;
  // Row-major C = op(A) op(B)  <=>  column-major C^T = op(B)^T op(A)^T.
  cublasOperation_t opa = trans_a ? CUBLAS_OP_T : CUBLAS_OP_N;
  cublasOperation_t opb = trans_b ? CUBLAS_OP_T : CUBLAS_OP_N;
  cublasStatus_t st;
  if (dtype == GR_F32) {
    const float one = 1.f, zero = 0.f;
    // BF16x9 emulation pays only for GEMMs large in both output dimensions
    // (tools/skinny_gemm_probe.py: 65536x1024 @ 1024xN — N=16/64 emulated
    // 245/248 us vs 111/165 us FP32; N=256 319 vs 566 us; N=1024 0.68 vs
    // 1.67 ms); cuBLAS's own PERFORMANT strategy still emulates the skinny ones
    const bool emu = S.gemm_math && gemm_emulation_pays(m, n);
    cublasSetMathMode(S.cublas, emu ? CUBLAS_FP32_EMULATED_BF16X9_MATH : CUBLAS_DEFAULT_MATH);
    st = cublasSgemm(S.cublas, opb, opa, n, m, k, &one, (const float*)b, ldb, (const float*)a, lda, &zero,
                     (float*)c, ldc);
  } else if (dtype == GR_F64) {
    const double one = 1.0, zero = 0.0;
    st = cublasDgemm(S.cublas, opb, opa, n, m, k, &one, (const double*)b, ldb, (const double*)a, lda, &zero,
                     (double*)c, ldc);
  } else {
    return fail(GR_EINVAL, "gemm dtype must be f32 or f64");
  }
  if (st != CUBLAS_STATUS_SUCCESS) return fail(GR_ECUBLAS, "cublas gemm: status " + std::to_string((int)st));
  return GR_OK;
}

int grumpy_rt_gemv(int trans, int rows, int cols, int dtype, uint64_t a, int lda, uint64_t x, uint64_t y) {
  int r = need_init();
  if (r) return r;
  r = ensure_cublas();
  if (r) return r;
  // Column-major view of row-major A[rows, cols] is A^T[cols, rows].
  // trans = 0: y = A x  = (A^T)^T x -> OP_T;  trans = 1: y = A^T x -> OP_N.
  cublasOperation_t op = trans ? CUBLAS_OP_N : CUBLAS_OP_T;
  cublasStatus_t st;
  if (dtype == GR_F32) {
    const float one = 1.f, zero = 0.f;
    st = cublasSgemv(S.cublas, op, cols, rows, &one, (const float*)a, lda, (const float*)x, 1, &zero, (float*)y, 1);
  } else if (dtype == GR_F64) {
    const double one = 1.0, zero = 0.0;
    st = cublasDgemv(S.cublas, op, cols, rows, &one, (const double*)a, lda, (const double*)x, 1, &zero,
                     (double*)y, 1);
  } else {
    return fail(GR_EINVAL, "gemv dtype must be f32 or f64");
  }
  if (st != CUBLAS_STATUS_SUCCESS) return fail(GR_ECUBLAS, "cublas gemv: status " + std::to_string((int)st));
  return GR_OK;
}

// ---- NCCL ---------------------------------------------------------------------
int grumpy_rt_nccl_load(const char* path) {
  if (N.handle) return GR_OK;
  N.handle = dlopen(path && path[0] ? path : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!N.handle) return fail(GR_EDLOPEN, std::string("dlopen(libnccl): ") + dlerror());
#define GR_NSYM(field, sym)                                                  \
  N.field = (decltype(N.field))dlsym(N.handle, sym);                         \
  if (!N.field) return fail(GR_EDLOPEN, std::string("libnccl lacks ") + sym);
  GR_NSYM(GetUniqueId, "ncclGetUniqueId")
  GR_NSYM(CommInitRank, "ncclCommInitRank")
  GR_NSYM(AllReduce, "ncclAllReduce")
  GR_NSYM(AllGather, "ncclAllGather")
  GR_NSYM(CommDestroy, "ncclCommDestroy")
  GR_NSYM(GroupStart, "ncclGroupStart")
  GR_NSYM(GroupEnd, "ncclGroupEnd")
  GR_NSYM(GetErrorString, "ncclGetErrorString")
#undef GR_NSYM
  return GR_OK;
}

int grumpy_rt_nccl_unique_id(char* id128) {
  if (!N.handle) return fail(GR_ENOINIT, "grumpy_rt_nccl_load first");
  NcclUid uid;
  int rr = N.GetUniqueId(&uid);
  if (rr) return nccl_fail(rr, "ncclGetUniqueId");
  memcpy(id128, uid.internal, 128);
  return GR_OK;
}

int grumpy_rt_nccl_init(int rank, int nranks, const char* id128) {
  int r = need_init();
  if (r) return r;
  if (!N.handle) return fail(GR_ENOINIT, "grumpy_rt_nccl_load first");
  NcclUid uid;
  memcpy(uid.internal, id128, 128);
  int rr = N.CommInitRank(&N.comm, nranks, uid, rank);
  if (rr) return nccl_fail(rr, "ncclCommInitRank");
  return GR_OK;
}

int grumpy_rt_nccl_allreduce(uint64_t send, uint64_t recv, size_t count, int dtype, int op) {
  int r = need_init();
  if (r) return r;
  if (!N.comm) return fail(GR_ENOINIT, "NCCL communicator not initialised");
  int nd = nccl_dtype(dtype);
  if (nd < 0 || op < 0 || op > 3) return fail(GR_EINVAL, "bad dtype/op");
  // grumpy op codes match ncclSum=0, ncclProd=1, ncclMax=2, ncclMin=3
  int rr = N.AllReduce((const void*)send, (void*)recv, count, nd, op, N.comm, CS());
  if (rr) return nccl_fail(rr, "ncclAllReduce");
  return GR_OK;
}

int grumpy_rt_nccl_allgather(uint64_t send, uint64_t recv, size_t count_per_rank, int dtype) {
  int r = need_init();
  if (r) return r;
  if (!N.comm) return fail(GR_ENOINIT, "NCCL communicator not initialised");
  int nd = nccl_dtype(dtype);
  if (nd < 0) return fail(GR_EINVAL, "bad dtype");
  (void)dtype_size;
  int rr = N.AllGather((const void*)send, (void*)recv, count_per_rank, nd, N.comm, CS());
  if (rr) return nccl_fail(rr, "ncclAllGather");
  return GR_OK;
}

// Several collectives of one plan step issued as ONE NCCL launch (the
// k-means step allreduces four f64 partial sums and the counts)
int grumpy_rt_nccl_group_start(void) {
  if (!N.handle) return fail(GR_ENOINIT, "grumpy_rt_nccl_load first");
  int rr = N.GroupStart();
  if (rr) return nccl_fail(rr, "ncclGroupStart");
  return GR_OK;
}

int grumpy_rt_nccl_group_end(void) {
  if (!N.handle) return fail(GR_ENOINIT, "grumpy_rt_nccl_load first");
  int rr = N.GroupEnd();
  if (rr) return nccl_fail(rr, "ncclGroupEnd");
  return GR_OK;
}

int grumpy_rt_nccl_destroy(void) {
  if (N.comm && N.CommDestroy) N.CommDestroy(N.comm);
  N.comm = nullptr;
  return GR_OK;
}

}  // extern "C"
