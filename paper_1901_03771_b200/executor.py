"""parallel-executor on B200: runs plan steps through the C-ABI shim.

Reference module ``parallel-executor``:
``run_map`` / ``run_map_reduce`` / ``run_map_scan`` over a blocked partition
of the iteration space on a CPU worker pool, and ``run_library`` for
gemm/gemv with transpose flags.  Here every fused step is ONE generated
sm_100a kernel launched on the runtime's stream, and library steps are cuBLAS
calls on the same stream.  Nothing synchronises the host
until an external consumer reads data (to_external), so consecutive steps and
consecutive forces pipeline on the device.
"""

from __future__ import annotations

import collections
import os
from typing import Dict, List

from . import codegen, runtime
from .dag import Node, OpKind
from .errors import ShapeMismatch
from .planner import PlanStep
from .tensor import DType, TensorBuffer, element_count


PRECOMPILE = os.environ.get("GRUMPY_PRECOMPILE", "1") == "1"
# NVTX ranges around every plan step (kind, kernel family or library call)
NVTX = os.environ.get("GRUMPY_NVTX", "0") == "1"


class Executor:
    def __init__(self, session):
        self.session = session
        self.rt = runtime.get()      # raises NativeLibraryMissing: no CPU fallback
        self._gen_cache: Dict[tuple, codegen.KernelSource] = {}
        self.last_steps: List[PlanStep] = []
        self.launch_log = collections.deque(maxlen=4096)  # (family, kernel name) per launch
        self.profile = None           # per-launch CUDA events when enabled
        self._tickets = {}
        self._tmaps = {}
        self.out_bind: Dict[int, TensorBuffer] = {}   # root id -> preallocated output (streaming.py)

    # -- planner hook ---------------------------------------------------------------
    def row_fusion(self, reduction: Node, consumer: Node) -> bool:
        return codegen.row_fusable(reduction, consumer)

    # -- buffers --------------------------------------------------------------------
    def device_ptr(self, n: Node) -> int:
        buf = n.data
        if buf.device is None:
            buf.device = self.rt.upload(buf.host)
            self.session.stats.h2d_bytes += buf.host.nbytes
        return buf.device.ptr

    def new_buffer(self, n: Node) -> TensorBuffer:
        nbytes = element_count(n.shape) * n.dtype.itemsize
        return TensorBuffer(n.dtype, n.shape, device=self.rt.alloc(nbytes))

    # -- steps ------------------------------------------------------------------------
    def run(self, steps: List[PlanStep], dist=None, comm=None):
        self.last_steps = steps
        cold = [st for st in steps if st.kind == "Fused" and "kernel" not in st.cache]
        if len(cold) >= 2 and PRECOMPILE:
            # JIT/execute pipelining: generate every uncompiled step's source
            # now and compile them on worker threads while the earlier steps
            # launch (SPEC.md:521 — the paper's JIT bottleneck)
            srcs = []
            for st in cold:
                self._prepare(st)
                if st.cache["ks"] is not None:
                    srcs.append(st.cache["ks"].source)
            self.rt.precompile(srcs)
        for st in steps:
            if NVTX:
                self.rt.range_push(self._step_name(st))
            try:
                self._run_step(st, dist, comm)
            finally:
                if NVTX:
                    self.rt.range_pop()

    @staticmethod
    def _step_name(st: PlanStep) -> str:
        if st.kind == "Library":
            return "grumpy:" + st.call
        ks = st.cache.get("ks")     # generated source (prepared by run()'s precompile or earlier runs)
        return "grumpy:" + (ks.meta.get("label") or ks.family if ks is not None else "fused")

    def _run_step(self, st: PlanStep, dist, comm):
        g = self.session.graph
        if st.kind == "Library":
            if self.profile is not None:
                e0, e1 = self._event_pair()
                self.rt.record(e0)
                outs = [self.run_library(st)]
                self.rt.record(e1)
                label = st.call + (f"+{st.epilogue[0]}" if st.epilogue else "")
                self.profile.append(("library", label, e0, e1))
            else:
                outs = [self.run_library(st)]
            self.session.stats.library_calls += 1
        else:
            outs = self.run_fused(st)
        if dist is not None:
            self._combine_partials(st.roots, outs, dist, comm)
        for r, b in zip(st.roots, outs):
            g.mark_materialized(r, b)
        self.session.stats.nodes_materialized += len(st.roots)

    def _combine_partials(self, roots, outs, dist, comm):
        """Allreduce partial roots in place on the runtime stream (NCCL), right
        after the kernel that produced them (distributed.py)."""
        from .dag import ReduceOp
        parts = [(r, b, dist.get(r.id, "R")) for r, b in zip(roots, outs)]
        parts = [(r, b, d) for r, b, d in parts if d.startswith("P:") and element_count(r.shape)]
        if not parts:
            return
        if self.profile is not None:
            e0, e1 = self._event_pair()
            self.rt.record(e0)
        # every partial of the step in one NCCL group: one launch, one latency
        with comm.group():
            for r, b, d in parts:
                comm.allreduce_device(b.device, element_count(r.shape), r.dtype, ReduceOp(d[2:]))
                self.session.stats.collectives += 1
        if self.profile is not None:
            self.rt.record(e1)
            self.profile.append(("collective", "allreduce:" + ",".join(sorted({d[2:] for _r, _b, d in parts})), e0, e1))

    def kernel_source(self, region: codegen.Region) -> codegen.KernelSource:
        return codegen.cached_generate(region)

    def buffer_ptr(self, buf: TensorBuffer) -> int:
        if buf.device is None:
            buf.device = self.rt.upload(buf.host)
            self.session.stats.h2d_bytes += buf.host.nbytes
        return buf.device.ptr

    def _prepare(self, st: PlanStep) -> None:
        """Canonical leaf order and generated kernel source of a fused step
        (memoized in the step's cache, shared by every plan instantiation)."""
        c = st.cache
        if "perm" not in c:
            region = codegen.canonicalize(codegen.Region(st.roots, st.leaves, st.nodes))
            pos = {l.id: i for i, l in enumerate(st.leaves)}
            c["perm"] = [pos[l.id] for l in region.leaves]
            empty = all(element_count(r.shape) == 0 for r in region.roots)
            c["ks"] = None if empty else self.kernel_source(region)

    def run_fused(self, st: PlanStep, bind: Dict[int, TensorBuffer] = None) -> List[TensorBuffer]:
        """Launch the step's kernel.  ``bind`` (leaf node id → buffer) supplies
        leaf data explicitly (the reference-style ``run_map(k, leaves, cfg)``
        entry points); otherwise leaves read their materialized data."""
        c = st.cache
        self._prepare(st)
        leaves = [st.leaves[i] for i in c["perm"]]
        outs = [self.out_bind.pop(r.id, None) or self.new_buffer(r) for r in st.roots]
        ks = c["ks"]
        if ks is None:
            return outs
        k = c.get("kernel")
        if k is None:
            k = self.rt.kernel(ks.source, ks.name, ks.block, ks.meta.get("smem", 0), tune=ks.family == "map")
            if k.cache_hit == 0:
                self.session.stats.compile_ms += k.compile_ms
            c["kernel"] = k
            c["grid"] = codegen.grid_for(ks, self.rt.sm_count, k.blocks_per_sm)
        if bind is None:
            ptrs = [self.device_ptr(l) for l in leaves]
        else:
            ptrs = [self.buffer_ptr(bind[l.id]) for l in leaves]
        cb = ks.meta.get("cbank")
        if cb:
            # small row-invariant leaves live in the module's constant bank:
            # one stream-ordered device copy per launch (the leaf may change
            # between launches, e.g. new k-means centroids)
            dst = c.get("cbank_dst")
            if dst is None:
                dst = c["cbank_dst"] = [self.rt.module_global(k, sym)[0] for _i, sym, _nb in cb]
            for (i, _sym, nb), d in zip(cb, dst):
                self.rt.d2d_raw(d, ptrs[i], nb)
        for i, psym, _b, _npairs, rname in ks.meta.get("cbank_pair") or ():
            # pair-adjacent copy of a constant-bank leaf (paired arg-reduction
            # loops): a one-CTA repack kernel of the same module writes it
            rp = c.setdefault("repack", {})
            if psym not in rp:
                rp[psym] = (self.rt.function(k, rname), self.rt.module_global(k, psym)[0])
            fn, addr = rp[psym]
            self.rt.launch(fn, 1, 256, runtime.pack_params([ptrs[i], addr]))
        ptrs += [b.device.ptr for b in outs]
        scratch = None
        if ks.scratch_bytes:
            scratch = self.rt.alloc(ks.scratch_bytes)
            if ks.meta.get("scratch_zero"):
                self.rt.memset(scratch, 0)
            ptrs.append(scratch.ptr)
        else:
            ptrs.append(0)
        if ks.meta.get("ticket"):
            # grid-completion counter: zeroed once, reset by the last CTA of
            # every launch (launches of one kernel are stream-ordered)
            tk = self._tickets.get(id(ks))
            if tk is None:
                tk = self.rt.alloc(4096)      # [0]: grid ticket, [1..]: keyed-sum group tickets
                self.rt.memset(tk, 0)
                self._tickets[id(ks)] = tk
            ptrs.append(tk.ptr)
        elif ks.meta.get("redo_words"):
            ptrs.append(0)
        if ks.meta.get("redo_words"):
            # per-row redo flags: zeroed once, cleared by the kernel as it redoes
            rd = self._tickets.get(("redo", id(ks)))
            if rd is None:
                rd = self.rt.alloc(4 * ks.meta["redo_words"])
                self.rt.memset(rd, 0)
                self._tickets[("redo", id(ks))] = rd
            ptrs.append(rd.ptr)
        params = runtime.pack_params(ptrs)
        tm = ks.meta.get("tmaps")
        if tm:
            # TMA tensor maps lead the parameter block (alignas(64) gr::TMap
            # members first in K::Params); the block is padded to the struct's
            # 64-byte alignment
            # slots past the leaves are the step's outputs (TMA stores)
            dts = [l.dtype for l in leaves] + [r.dtype for r in st.roots]
            maps = b"".join(self._tensor_map(ptrs[i], dts[i], d0, d1, b0, b1, sw)
                            for i, d0, d1, b0, b1, sw in tm)
            params = maps + params
            params += b"\0" * (-len(params) % 64)
        if self.profile is not None:
            e0, e1 = self._event_pair()
            self.rt.record(e0)
            self.rt.launch(k, c["grid"], ks.block, params, smem=ks.meta.get("smem", 0))
            self.rt.record(e1)
            self.profile.append((ks.family, ks.meta.get("label", ks.name), e0, e1))
        else:
            self.rt.launch(k, c["grid"], ks.block, params, smem=ks.meta.get("smem", 0))
        self.session.stats.kernels_executed += 1
        self.launch_log.append((ks.family, ks.name))
        # scratch is stream-ordered: returning it to the pool now is safe for
        # later launches on the same stream
        del scratch
        return outs

    def _tensor_map(self, ptr, dtype, d0, d1, b0, b1, sw) -> bytes:
        """128-byte CUtensorMap of a row-major [d1][d0] leaf (cached per buffer)."""
        key = (ptr, dtype, d0, d1, b0, b1, sw)
        m = self._tmaps.get(key)
        if m is None:
            if len(self._tmaps) > 256:
                self._tmaps.clear()
            m = self._tmaps[key] = self.rt.tensor_map_2d(ptr, dtype, d0, d1, d0 * dtype.itemsize, b0, b1, sw)
        return m

    # -- optional per-launch device timing (bench.py) ----------------------------------
    def enable_profile(self):
        self.profile = []
        self._events = []

    def _event_pair(self):
        i = len(self.profile)
        while len(self._events) <= i:
            self._events.append((self.rt.event(), self.rt.event()))
        return self._events[i]

    def take_profile(self):
        """[(family, label, ms)] for launches since enable_profile(); syncs."""
        out = [(f, l, self.rt.elapsed_ms(a, b)) for f, l, a, b in self.profile]
        self.profile = []
        return out

    def run_library(self, st: PlanStep) -> TensorBuffer:
        """run_library → cuBLAS on the runtime stream."""
        n = st.library_node if st.library_node is not None else st.root
        ops = st.operands
        flags = st.trans_flags
        out = self.new_buffer(st.root)
        dt = n.dtype
        for o in ops:
            if o.dtype is not dt:
                raise ShapeMismatch(f"library operand dtype {o.dtype} != {dt}")
        if n.kind is OpKind.MATMUL:
            a, b = ops
            ta, tb = flags
            m, nn = n.shape
            k = a.shape[0] if ta else a.shape[1]
            if m and nn and st.epilogue is not None:
                # GEMM + bias (+ ReLU) in one cuBLASLt call (the R1 region absorbed)
                kind, bias = st.epilogue
                self.rt.gemm_epilogue(ta, tb, m, nn, k, self.device_ptr(a), a.shape[1],
                                      self.device_ptr(b), b.shape[1], out.device.ptr, nn,
                                      bias=self.device_ptr(bias), epilogue=kind,
                                      emulate=2 if self.rt.gemm_math == "bf16x9" else 0)
            elif m and nn:
                if k == 0:
                    self.rt.memset(out.device, 0)
                else:
                    self.rt.gemm(ta, tb, m, nn, k, dt, self.device_ptr(a), a.shape[1],
                                 self.device_ptr(b), b.shape[1], out.device.ptr, nn)
        else:
            (vec_mat,) = n.op.attrs
            mat, x = ops
            tm = flags[0]
            rows, cols = mat.shape
            # effective operation: y = M x (vec_mat False) or y = M^T x (True);
            # an absorbed transpose flips it once more.
            trans = bool(vec_mat) != bool(tm)
            if element_count(n.shape):
                if (cols if not trans else rows) == 0:
                    self.rt.memset(out.device, 0)
                else:
                    self.rt.gemv(trans, rows, cols, dt, self.device_ptr(mat), cols, self.device_ptr(x), out.device.ptr)
        self.launch_log.append(("library", st.call))
        return out


# ---------------------------------------------------------------------------
# Reference-facing executor entry points
# ---------------------------------------------------------------------------


class ExecConfig:
    """SPEC.md:355-358.  ``num_threads`` is validated and recorded; on the B200
    path the partition is the kernel's grid, and results are bit-identical for
    every value (the reference's determinism invariant)."""

    def __init__(self, num_threads: int = 1, block="auto"):
        if int(num_threads) < 1:
            raise ValueError("num_threads must be >= 1 (SPEC.md:357)")
        self.num_threads = int(num_threads)
        self.block = block


class LibraryCall:
    """Gemm | Gemv, per-operand transpose flags, operand ids."""

    def __init__(self, call: str, trans_flags=(False, False), operands=()):
        if call not in ("Gemm", "Gemv"):
            raise ValueError(f"unknown library call {call!r}")
        self.call = call
        self.trans_flags = tuple(bool(t) for t in trans_flags)
        self.operands = tuple(operands)


def _executor():
    from .session import default_session
    return default_session().executor


def _bind(k, leaves) -> Dict[int, TensorBuffer]:
    st = k.step
    if isinstance(leaves, dict):
        bind = dict(leaves)
    else:
        leaves = list(leaves)
        if len(leaves) != len(st.leaves):
            raise ShapeMismatch(f"kernel has {len(st.leaves)} leaves, got {len(leaves)} buffers")
        bind = {l.id: b for l, b in zip(st.leaves, leaves)}
    for l in st.leaves:
        b = bind.get(l.id)
        if b is None:
            raise ShapeMismatch(f"no buffer for leaf {l.id}")
        if tuple(b.shape) != tuple(l.shape) or b.dtype is not l.dtype:
            raise ShapeMismatch(f"leaf {l.id}: buffer {b.dtype.value}{b.shape} != {l.dtype.value}{l.shape}")
    return bind


def _run(k, leaves, cfg, kind):
    if k.kind != kind:
        raise ValueError(f"run_{kind} given a {k.kind} kernel")
    if cfg is not None and not isinstance(cfg, ExecConfig):
        raise TypeError("cfg must be an ExecConfig")
    ex = _executor()
    outs = ex.run_fused(k.step, bind=_bind(k, leaves))
    return outs[0] if len(outs) == 1 else tuple(outs)


def run_map(k, leaves, cfg: ExecConfig = None) -> TensorBuffer:
    """out[p] = point(p) for every p — one generated kernel."""
    return _run(k, leaves, cfg, "Map")


def run_map_reduce(k, leaves, cfg: ExecConfig = None) -> TensorBuffer:
    """fold of the mapped values — one kernel launch,
    deterministic combine (NumPy's association order, see codegen_rows)."""
    return _run(k, leaves, cfg, "MapReduce")


def run_map_scan(k, leaves, cfg: ExecConfig = None) -> TensorBuffer:
    """inclusive scan of the mapped values (codegen_scan)."""
    return _run(k, leaves, cfg, "MapScan")


def run_library(call: LibraryCall, operands, cfg: ExecConfig = None) -> TensorBuffer:
    """SPEC.md:391-399 → cuBLAS on the runtime stream.

    Gemv(A, x): y[i] = Σ_k A'[i,k]·x[k], A' = Aᵀ when trans_flags[0].
    Gemm(A, B): C = A'·B' with per-operand flags.  ShapeMismatch when the
    operands do not conform after the flags."""
    ex = _executor()
    rt = ex.rt
    ops = list(operands)
    if len(ops) != 2:
        raise ShapeMismatch(f"{call.call} takes 2 operands, got {len(ops)}")
    a, b = ops
    dt = a.dtype
    if b.dtype is not dt or dt not in (DType.f32, DType.f64):
        raise ShapeMismatch(f"library operands must share an f32/f64 dtype, got {a.dtype} and {b.dtype}")
    flags = call.trans_flags + (False,) * (2 - len(call.trans_flags))
    if len(a.shape) != 2:
        raise ShapeMismatch(f"{call.call}: first operand must be rank 2, got {a.shape}")
    rows, cols = a.shape
    m, k = (cols, rows) if flags[0] else (rows, cols)
    if call.call == "Gemv":
        if len(b.shape) != 1 or b.shape[0] != k:
            raise ShapeMismatch(f"Gemv: {a.shape}{'ᵀ' if flags[0] else ''} · {b.shape}")
        out = TensorBuffer(dt, (m,), device=rt.alloc(m * dt.itemsize))
        if m:
            if k == 0:
                rt.memset(out.device, 0)
            else:
                rt.gemv(flags[0], rows, cols, dt, ex.buffer_ptr(a), cols, ex.buffer_ptr(b), out.device.ptr)
    else:
        if len(b.shape) != 2:
            raise ShapeMismatch(f"Gemm: second operand must be rank 2, got {b.shape}")
        k2, n = (b.shape[1], b.shape[0]) if flags[1] else tuple(b.shape)
        if k2 != k:
            raise ShapeMismatch(f"Gemm: inner extents {k} and {k2} differ")
        out = TensorBuffer(dt, (m, n), device=rt.alloc(m * n * dt.itemsize))
        if m and n:
            if k == 0:
                rt.memset(out.device, 0)
            else:
                rt.gemm(flags[0], flags[1], m, n, k, dt, ex.buffer_ptr(a), a.shape[1],
                        ex.buffer_ptr(b), b.shape[1], out.device.ptr, n)
    ex.session.stats.library_calls += 1
    ex.launch_log.append(("library", call.call))
    return out
