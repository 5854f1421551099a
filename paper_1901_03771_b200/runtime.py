"""ctypes binding of the C-ABI shim ``libgrumpy_rt.so`` (include/grumpy_rt.h).

This is the Python side of the drop-in executor boundary:
device buffers from the caching pool, transfers, NVRTC compile + module cache,
kernel launch, events, cuBLAS and NCCL.  There is no CPU fallback: if the
library or a device is missing, ``get()`` raises ``NativeLibraryMissing``.
"""

from __future__ import annotations

import ctypes
import hashlib
import os
import struct
import threading
import weakref
from typing import Optional, Sequence

import numpy as np

from .errors import NativeLibraryMissing, RuntimeFailure
from .tensor import DType

# bytes of per-thread local memory (spill) a register-capped rebuild of a map
# kernel may use and still be kept for its extra resident CTAs
TUNE_MAX_LOCAL = int(os.environ.get("GRUMPY_TUNE_MAX_LOCAL", "8"))

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libgrumpy_rt.so")
KERNEL_DIR = os.path.join(HERE, "csrc", "kernels")

GR_DTYPE = {DType.f32: 0, DType.f64: 1, DType.i32: 2, DType.i64: 3, DType.bool8: 4}

# Every export of include/grumpy_rt.h with its ctypes signature.
_u64 = ctypes.c_uint64
_sz = ctypes.c_size_t
_i = ctypes.c_int
_p = ctypes.c_void_p
_ip = ctypes.POINTER(ctypes.c_int)
_u64p = ctypes.POINTER(ctypes.c_uint64)
_szp = ctypes.POINTER(ctypes.c_size_t)
_dp = ctypes.POINTER(ctypes.c_double)
_fp = ctypes.POINTER(ctypes.c_float)
_cp = ctypes.c_char_p
_cpp = ctypes.POINTER(ctypes.c_char_p)

SIGNATURES = {
    "grumpy_rt_version": [_ip],
    "grumpy_rt_init": [_i],
    "grumpy_rt_device_count": [_ip],
    "grumpy_rt_device_info": [_ip, _ip, _ip, _szp, _cp],
    "grumpy_rt_last_error": None,
    "grumpy_rt_stream": [_u64p],
    "grumpy_rt_alloc": [_sz, _u64p],
    "grumpy_rt_free": [_u64],
    "grumpy_rt_pool_stats": [_szp, _szp, _szp, _szp],
    "grumpy_rt_pool_trim": [],
    "grumpy_rt_h2d": [_u64, _p, _sz],
    "grumpy_rt_d2h": [_p, _u64, _sz],
    "grumpy_rt_d2d": [_u64, _u64, _sz],
    "grumpy_rt_memset": [_u64, _i, _sz],
    "grumpy_rt_host_alloc": [_sz, ctypes.POINTER(_p)],
    "grumpy_rt_host_free": [_p],
    "grumpy_rt_host_register": [_p, _sz],
    "grumpy_rt_host_unregister": [_p],
    "grumpy_rt_compile": [_cp, _cpp, _i, _cp, _u64p, _dp, _ip],
    "grumpy_rt_compile_cubin": [_cp, _cpp, _i, _p, _sz, _szp, _dp],
    "grumpy_rt_precompile": [_cp, _cpp, _i, _cp, _dp],
    "grumpy_rt_get_function": [_u64, _cp, _u64p],
    "grumpy_rt_module_global": [_u64, _cp, _u64p, ctypes.POINTER(ctypes.c_size_t)],
    "grumpy_rt_tensor_map_2d": [_u64, _i, _u64, _u64, _u64, ctypes.c_uint, ctypes.c_uint, _i, _p],
    "grumpy_rt_function_info": [_u64, _ip, _ip, _ip, _ip],
    "grumpy_rt_occupancy": [_u64, _i, _sz, _ip],
    "grumpy_rt_launch": [_u64, ctypes.c_uint, ctypes.c_uint, ctypes.c_uint, ctypes.c_uint,
                         ctypes.c_uint, ctypes.c_uint, ctypes.c_uint, ctypes.c_uint, _p, _sz],
    "grumpy_rt_sync": [],
    "grumpy_rt_range_push": [_cp],
    "grumpy_rt_range_pop": [],
    "grumpy_rt_stream_create": [_u64p],
    "grumpy_rt_stream_destroy": [_u64],
    "grumpy_rt_set_stream": [_u64],
    "grumpy_rt_stream_wait_event": [_u64],
    "grumpy_rt_d2h_async": [_p, _u64, _sz],
    "grumpy_rt_event_sync": [_u64],
    "grumpy_rt_event_create": [_u64p],
    "grumpy_rt_event_record": [_u64],
    "grumpy_rt_event_elapsed": [_u64, _u64, _fp],
    "grumpy_rt_event_destroy": [_u64],
    "grumpy_rt_gemm": [_i, _i, _i, _i, _i, _i, _u64, _i, _u64, _i, _u64, _i],
    "grumpy_rt_gemv": [_i, _i, _i, _i, _u64, _i, _u64, _u64],
    "grumpy_rt_set_gemm_math": [_i],
    "grumpy_rt_gemm_epilogue": [_i, _i, _i, _i, _i, _u64, _i, _u64, _i, _u64, _i, _u64, _i, _i],
    "grumpy_rt_nccl_load": [_cp],
    "grumpy_rt_nccl_unique_id": [_cp],
    "grumpy_rt_nccl_init": [_i, _i, _cp],
    "grumpy_rt_nccl_allreduce": [_u64, _u64, _sz, _i, _i],
    "grumpy_rt_nccl_allgather": [_u64, _u64, _sz, _i],
    "grumpy_rt_nccl_group_start": [],
    "grumpy_rt_nccl_group_end": [],
    "grumpy_rt_nccl_destroy": [],
}

NVRTC_OPTS = [
    "--gpu-architecture=sm_100a",
    "--std=c++17",
    "--fmad=false",          # NumPy never contracts a*b+c: bit-exact +,-,*
    "--ftz=false",           # keep denormals like x86 NumPy
    "--prec-div=true",
    "--prec-sqrt=true",
    "-lineinfo",
    "-DNDEBUG",
]

_lib = None
_lib_lock = threading.Lock()


def load_library(path: str = LIB_PATH):
    """Load and type the shim (no device needed)."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise NativeLibraryMissing(
                f"{path} is not built; run `python -m paper_1901_03771_b200.build_native` "
                "or __graft_entry__.build()")
        lib = ctypes.CDLL(path)
        for name, argtypes in SIGNATURES.items():
            f = getattr(lib, name)
            if argtypes is None:
                f.restype = ctypes.c_char_p
                f.argtypes = []
            else:
                f.restype = ctypes.c_int
                f.argtypes = argtypes
        _lib = lib
        return lib


def _check(rc):
    if rc != 0:
        msg = _lib.grumpy_rt_last_error().decode(errors="replace")
        raise RuntimeFailure(rc, msg)


def nvrtc_options():
    return [o.encode() for o in NVRTC_OPTS] + [f"-I{KERNEL_DIR}".encode()]


def compile_cubin(source: str) -> bytes:
    """NVRTC → sm_100a cubin without a device (CPU-side build checks)."""
    lib = load_library()
    opts = nvrtc_options()
    arr = (ctypes.c_char_p * len(opts))(*opts)
    size = ctypes.c_size_t(0)
    ms = ctypes.c_double(0)
    _check(lib.grumpy_rt_compile_cubin(source.encode(), arr, len(opts), None, 0, ctypes.byref(size), ctypes.byref(ms)))
    buf = ctypes.create_string_buffer(size.value)
    _check(lib.grumpy_rt_compile_cubin(source.encode(), arr, len(opts), buf, size.value, ctypes.byref(size), ctypes.byref(ms)))
    return buf.raw


class DeviceBuffer:
    """A pool allocation; returned to the pool when garbage-collected."""

    __slots__ = ("ptr", "nbytes", "_rt", "__weakref__")

    def __init__(self, rt: "Runtime", nbytes: int):
        self._rt = rt
        self.nbytes = int(nbytes)
        p = ctypes.c_uint64(0)
        _check(rt.lib.grumpy_rt_alloc(max(self.nbytes, 1), ctypes.byref(p)))
        self.ptr = p.value
        rt.stats_allocs += 1

    def __del__(self):
        try:
            if self.ptr and _lib is not None:
                _lib.grumpy_rt_free(self.ptr)
        except Exception:  # interpreter shutdown
            pass
        self.ptr = 0

    def copy_from_host(self, arr: np.ndarray):
        assert arr.flags.c_contiguous and arr.nbytes <= self.nbytes
        _check(self._rt.lib.grumpy_rt_h2d(self.ptr, arr.ctypes.data, arr.nbytes))

    def copy_to_host(self, out: np.ndarray):
        if out.nbytes:
            _check(self._rt.lib.grumpy_rt_d2h(out.ctypes.data, self.ptr, out.nbytes))

    def to_numpy(self, dtype: DType, shape) -> np.ndarray:
        out = np.empty(shape, dtype=dtype.np)
        if out.nbytes:
            _check(self._rt.lib.grumpy_rt_d2h(out.ctypes.data, self.ptr, out.nbytes))
        return out


class Kernel:
    """A loaded kernel: function handle plus launch geometry policy."""

    __slots__ = ("fn", "name", "block", "blocks_per_sm", "num_regs", "compile_ms", "cache_hit", "source", "module")

    def __init__(self, fn, name, block, blocks_per_sm, num_regs, compile_ms, cache_hit, source, module=0):
        self.module = module
        self.fn = fn
        self.name = name
        self.block = block
        self.blocks_per_sm = blocks_per_sm
        self.num_regs = num_regs
        self.compile_ms = compile_ms
        self.cache_hit = cache_hit
        self.source = source


class Runtime:
    """Per-process device runtime (one process drives one GPU)."""

    def __init__(self, device: int):
        self.lib = load_library()
        rc = self.lib.grumpy_rt_init(device)
        if rc != 0:
            msg = self.lib.grumpy_rt_last_error().decode(errors="replace")
            raise NativeLibraryMissing(f"CUDA device {device} unusable: {msg}")
        self.device = device
        sm = ctypes.c_int(0)
        ma = ctypes.c_int(0)
        mi = ctypes.c_int(0)
        tm = ctypes.c_size_t(0)
        name = ctypes.create_string_buffer(256)
        _check(self.lib.grumpy_rt_device_info(ctypes.byref(sm), ctypes.byref(ma), ctypes.byref(mi),
                                              ctypes.byref(tm), name))
        self.sm_count = sm.value
        self.cc = (ma.value, mi.value)
        self.total_mem = tm.value
        self.name = name.value.decode()
        # the on-disk cubin cache is keyed by source + options; the kernel
        # headers the sources include are versioned by the directory name
        self.cache_dir = os.path.join(
            os.environ.get("GRUMPY_CACHE_DIR", os.path.join(os.path.expanduser("~"), ".cache", "grumpy")),
            _headers_digest())
        try:
            os.makedirs(self.cache_dir, exist_ok=True)
        except OSError:
            pass
        self._kernels = {}
        self._pending = {}            # source -> Future of a precompile job
        self.gemm_math = "fp32"
        want = os.environ.get("GRUMPY_GEMM_MATH", "bf16x9")
        try:
            self.set_gemm_math(want)
        except RuntimeFailure:
            # an older cuBLAS was loaded first (e.g. PyTorch's wheel): FP32 SIMT
            self.gemm_math = "fp32"
        self._pool = None
        self.stats_allocs = 0
        self.launches = 0
        self.compile_ms_total = 0.0

    # -- memory
    def alloc(self, nbytes: int) -> DeviceBuffer:
        return DeviceBuffer(self, nbytes)

    def upload(self, arr: np.ndarray) -> DeviceBuffer:
        arr = np.ascontiguousarray(arr)
        buf = DeviceBuffer(self, arr.nbytes)
        buf.copy_from_host(arr)
        return buf

    def memset(self, buf: DeviceBuffer, value: int = 0):
        _check(self.lib.grumpy_rt_memset(buf.ptr, value, buf.nbytes))

    def d2d(self, dst: DeviceBuffer, src: DeviceBuffer, nbytes: int):
        _check(self.lib.grumpy_rt_d2d(dst.ptr, src.ptr, nbytes))

    def sync(self):
        _check(self.lib.grumpy_rt_sync())

    def range_push(self, name: str):
        """NVTX range around host-side work (Nsight Systems / Compute)."""
        _check(self.lib.grumpy_rt_range_push(name.encode()))

    def range_pop(self):
        _check(self.lib.grumpy_rt_range_pop())

    def function(self, k: "Kernel", name: str) -> "Kernel":
        """Another kernel of ``k``'s module (e.g. a leaf repack kernel)."""
        fn = ctypes.c_uint64(0)
        _check(self.lib.grumpy_rt_get_function(k.module, name.encode(), ctypes.byref(fn)))
        return Kernel(fn.value, name, 256, 1, 0, 0.0, 1, "", k.module)

    def module_global(self, k: "Kernel", name: str):
        """(device address, bytes) of a module-scope symbol of ``k``'s module."""
        p = ctypes.c_uint64(0)
        n = ctypes.c_size_t(0)
        _check(self.lib.grumpy_rt_module_global(k.module, name.encode(), ctypes.byref(p), ctypes.byref(n)))
        return p.value, n.value

    def tensor_map_2d(self, gaddr: int, dtype: DType, dim0: int, dim1: int, stride1: int,
                      box0: int, box1: int, swizzle: int = 128) -> bytes:
        """128-byte CUtensorMap for a row-major [dim1][dim0] tensor (TMA)."""
        buf = ctypes.create_string_buffer(128)
        _check(self.lib.grumpy_rt_tensor_map_2d(gaddr, GR_DTYPE[dtype], dim0, dim1, stride1, box0, box1,
                                                swizzle, buf))
        return buf.raw

    def d2d_raw(self, dst: int, src: int, nbytes: int):
        _check(self.lib.grumpy_rt_d2d(dst, src, nbytes))

    def pool_stats(self):
        v = [ctypes.c_size_t(0) for _ in range(4)]
        _check(self.lib.grumpy_rt_pool_stats(*[ctypes.byref(x) for x in v]))
        return {"in_use": v[0].value, "cached": v[1].value, "peak": v[2].value, "cuMemAlloc_calls": v[3].value}

    def pool_trim(self):
        _check(self.lib.grumpy_rt_pool_trim())

    def host_alloc(self, nbytes: int):
        p = ctypes.c_void_p(0)
        _check(self.lib.grumpy_rt_host_alloc(nbytes, ctypes.byref(p)))
        return p.value

    def host_free(self, ptr):
        _check(self.lib.grumpy_rt_host_free(ptr))

    def pinned_empty(self, shape, dtype) -> np.ndarray:
        """A NumPy array backed by page-locked host memory (freed with the array)."""
        dt = np.dtype(dtype)
        n = int(np.prod(shape)) * dt.itemsize
        ptr = self.host_alloc(max(n, 1))
        raw = (ctypes.c_char * max(n, 1)).from_address(ptr)
        arr = np.frombuffer(raw, dtype=dt, count=int(np.prod(shape))).reshape(shape)
        rt = self
        weakref.finalize(raw, lambda: rt.host_free(ptr) if _lib is not None else None)
        return arr

    # -- compile / launch
    def kernel(self, source: str, name: str, block: int, smem: int = 0, tune: bool = False) -> Kernel:
        """Compile + load.  ``tune``: when the kernel sits a few registers above
        an occupancy cliff, recompile with ``__launch_bounds__(block, occ+1)``
        and keep that build if ptxas fits it without spilling."""
        k = self._kernels.get((source, name, tune))
        if k is not None:
            return k
        k = self._kernel(source, name, block, smem)
        if tune and smem == 0:
            want = k.blocks_per_sm + 1
            cap = (65536 // (want * block)) // 8 * 8
            tag = f"__launch_bounds__({block})"
            if want * block <= 2048 and 0 < k.num_regs - cap <= 8 and tag in source:
                k2 = self._kernel(source.replace(tag, f"__launch_bounds__({block}, {want})"), name, block, smem)
                local = ctypes.c_int(0)
                _check(self.lib.grumpy_rt_function_info(k2.fn, None, ctypes.byref(local), None, None))
                if local.value <= TUNE_MAX_LOCAL and k2.blocks_per_sm > k.blocks_per_sm:
                    k = k2
        self._kernels[(source, name, tune)] = k
        return k

    def precompile(self, sources: Sequence[str]) -> None:
        """Start NVRTC compiles of ``sources`` on worker threads (ctypes drops
        the GIL in the call); ``_kernel`` waits for its source's job, then
        loads the cubin it left.  Used when a plan has several uncompiled
        steps: their compiles overlap each other and the earlier launches."""
        import concurrent.futures as cf
        if self._pool is None:
            self._pool = cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1),
                                               thread_name_prefix="grumpy-nvrtc")
        for src in sources:
            if src in self._pending or any(k[0] == src for k in self._kernels):
                continue
            self._pending[src] = self._pool.submit(self._precompile_one, src)

    def _precompile_one(self, source: str) -> float:
        opts = nvrtc_options()
        arr = (ctypes.c_char_p * len(opts))(*opts)
        ms = ctypes.c_double(0)
        _check(self.lib.grumpy_rt_precompile(source.encode(), arr, len(opts), self.cache_dir.encode(),
                                             ctypes.byref(ms)))
        return ms.value

    def _kernel(self, source: str, name: str, block: int, smem: int = 0) -> Kernel:
        pre_ms = 0.0
        fut = self._pending.pop(source, None)
        if fut is not None:
            pre_ms = fut.result()     # raises the compile error here, on the launching thread
        opts = nvrtc_options()
        arr = (ctypes.c_char_p * len(opts))(*opts)
        mod = ctypes.c_uint64(0)
        ms = ctypes.c_double(0)
        hit = ctypes.c_int(0)
        _check(self.lib.grumpy_rt_compile(source.encode(), arr, len(opts), self.cache_dir.encode(),
                                          ctypes.byref(mod), ctypes.byref(ms), ctypes.byref(hit)))
        fn = ctypes.c_uint64(0)
        _check(self.lib.grumpy_rt_get_function(mod.value, name.encode(), ctypes.byref(fn)))
        occ = ctypes.c_int(0)
        _check(self.lib.grumpy_rt_occupancy(fn.value, block, smem, ctypes.byref(occ)))
        regs = ctypes.c_int(0)
        _check(self.lib.grumpy_rt_function_info(fn.value, ctypes.byref(regs), None, None, None))
        cms, h = ms.value, hit.value
        if h == 3:                    # compiled ahead on a worker thread: still a compile
            cms, h = pre_ms, 0
        self.compile_ms_total += cms
        return Kernel(fn.value, name, block, max(occ.value, 1), regs.value, cms, h, source, mod.value)

    def launch(self, k: Kernel, grid, block, params: bytes, smem: int = 0, cluster: int = 1):
        gx, gy, gz = (grid, 1, 1) if isinstance(grid, int) else grid
        bx, by, bz = (block, 1, 1) if isinstance(block, int) else block
        _check(self.lib.grumpy_rt_launch(k.fn, gx, gy, gz, bx, by, bz, smem, cluster, params, len(params)))
        self.launches += 1

    # -- streams (streamed materialisation: copies overlap kernels)
    def stream_create(self) -> int:
        st = ctypes.c_uint64(0)
        _check(self.lib.grumpy_rt_stream_create(ctypes.byref(st)))
        return st.value

    def stream_destroy(self, st: int):
        _check(self.lib.grumpy_rt_stream_destroy(st))

    def set_stream(self, st: int = 0):
        """Route async work to stream ``st`` (0: the runtime's own stream)."""
        _check(self.lib.grumpy_rt_set_stream(st))

    def wait_event(self, ev):
        """The current stream waits for ``ev``."""
        _check(self.lib.grumpy_rt_stream_wait_event(ev))

    def h2d_async(self, dst_ptr: int, arr: np.ndarray):
        _check(self.lib.grumpy_rt_h2d(dst_ptr, arr.ctypes.data, arr.nbytes))

    def d2h_async(self, out: np.ndarray, src_ptr: int):
        _check(self.lib.grumpy_rt_d2h_async(out.ctypes.data, src_ptr, out.nbytes))

    def event_sync(self, ev):
        _check(self.lib.grumpy_rt_event_sync(ev))

    # -- events
    def event(self):
        e = ctypes.c_uint64(0)
        _check(self.lib.grumpy_rt_event_create(ctypes.byref(e)))
        return e.value

    def record(self, ev):
        _check(self.lib.grumpy_rt_event_record(ev))

    def elapsed_ms(self, e0, e1) -> float:
        ms = ctypes.c_float(0)
        _check(self.lib.grumpy_rt_event_elapsed(e0, e1, ctypes.byref(ms)))
        return ms.value

    # -- library (cuBLAS)
    def gemm(self, trans_a, trans_b, m, n, k, dtype: DType, a, lda, b, ldb, c, ldc):
        _check(self.lib.grumpy_rt_gemm(int(trans_a), int(trans_b), m, n, k, GR_DTYPE[dtype],
                                       a, lda, b, ldb, c, ldc))

    def set_gemm_math(self, mode: str) -> None:
        """"fp32" (CUDA cores) or "bf16x9" (FP32 emulated on the tensor cores)."""
        _check(self.lib.grumpy_rt_set_gemm_math({"fp32": 0, "bf16x9": 1}[mode]))
        self.gemm_math = mode

    def gemm_epilogue(self, trans_a, trans_b, m, n, k, a, lda, b, ldb, c, ldc, bias=0, epilogue="none",
                      emulate=False):
        """cuBLASLt f32 GEMM, epilogue "none" | "bias" | "relu_bias" (bias along columns);
        emulate: 0 FP32, 1 BF16x9-emulated FP32, 2 emulated where it pays (both output dims >= 128)."""
        _check(self.lib.grumpy_rt_gemm_epilogue(int(trans_a), int(trans_b), m, n, k, a, lda, b, ldb, c, ldc,
                                                bias, {"none": 0, "bias": 1, "relu_bias": 2}[epilogue],
                                                int(emulate)))

    def gemv(self, trans, rows, cols, dtype: DType, a, lda, x, y):
        _check(self.lib.grumpy_rt_gemv(int(trans), rows, cols, GR_DTYPE[dtype], a, lda, x, y))

    # -- NCCL
    def nccl_load(self):
        path = ""
        try:
            import nvidia.nccl  # noqa: F401  (pip wheel bundled with torch)
            cand = os.path.join(os.path.dirname(nvidia.nccl.__file__ or nvidia.nccl.__path__[0]), "lib", "libnccl.so.2")
            if not os.path.exists(cand):
                cand = os.path.join(list(nvidia.nccl.__path__)[0], "lib", "libnccl.so.2")
            path = cand if os.path.exists(cand) else ""
        except Exception:
            path = ""
        _check(self.lib.grumpy_rt_nccl_load(path.encode()))

    def nccl_unique_id(self) -> bytes:
        buf = ctypes.create_string_buffer(128)
        _check(self.lib.grumpy_rt_nccl_unique_id(buf))
        return buf.raw

    def nccl_init(self, rank, nranks, uid: bytes):
        _check(self.lib.grumpy_rt_nccl_init(rank, nranks, uid))

    def nccl_allreduce(self, send: int, recv: int, count: int, dtype: DType, op: int):
        _check(self.lib.grumpy_rt_nccl_allreduce(send, recv, count, GR_DTYPE[dtype], op))

    def nccl_allgather(self, send: int, recv: int, count: int, dtype: DType):
        _check(self.lib.grumpy_rt_nccl_allgather(send, recv, count, GR_DTYPE[dtype]))

    def nccl_group_start(self):
        _check(self.lib.grumpy_rt_nccl_group_start())

    def nccl_group_end(self):
        _check(self.lib.grumpy_rt_nccl_group_end())


_rt: Optional[Runtime] = None


def device_count() -> int:
    """CUDA devices visible to this process (0 when there is no driver)."""
    n = ctypes.c_int(0)
    try:
        rc = load_library().grumpy_rt_device_count(ctypes.byref(n))
    except Exception:  # noqa: BLE001 — no shim: no devices usable
        return 0
    return n.value if rc == 0 else 0


def default_device() -> int:
    for var in ("GRUMPY_DEVICE", "LOCAL_RANK"):
        if os.environ.get(var):
            return int(os.environ[var])
    return 0


def get() -> Runtime:
    """The process runtime (created on first use)."""
    global _rt
    if _rt is None:
        _rt = Runtime(default_device())
    return _rt


def _headers_digest() -> str:
    h = hashlib.sha1()
    kdir = os.path.join(os.path.dirname(os.path.abspath(__file__)), "csrc", "kernels")
    for fn in sorted(os.listdir(kdir)):
        if fn.endswith((".cuh", ".h")):
            h.update(fn.encode())
            with open(os.path.join(kdir, fn), "rb") as f:
                h.update(f.read())
    return "h" + h.hexdigest()[:16]


def pack_params(ptrs: Sequence[int]) -> bytes:
    return struct.pack(f"<{len(ptrs)}Q", *ptrs)
