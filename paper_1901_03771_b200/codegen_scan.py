"""Map-scan family: cumsum / cumprod / maximum.accumulate with a fused map prologue.

Reference: run_map_scan: inclusive scan of
the mapped values along one axis, a three-phase blocked scan on CPU threads
(SPEC.md:385); PAPER.md:545-551 (map-scan primitive).  NumPy's accumulate is a
sequential left fold along the axis (out[k] = out[k-1] ⊕ x[k]).

* scans along an axis with many independent lines: one thread per line, the
  line folded sequentially — exactly NumPy's association (bit-identical);
* long 1-D scans (axis=None or a single long line): a single-pass scan with
  decoupled look-back — each CTA scans a 2048-element tile (thread-sequential
  runs, warp-shuffle + shared-memory combine of run totals), publishes its
  aggregate and inclusive prefix, and folds its predecessors' published values
  (``gr::scan_lookback``); deterministic, float results within tolerance of
  the sequential fold (reassociation), integers exact.
"""

from __future__ import annotations

from typing import List

from .codegen import HEADER, Aff, KernelSource, Region, Var, _params_struct, c_literal
from .codegen_rows import _COMBINE, _IDENT, _OPS, LoopEmitter, NotFusable, render, _flat_coords
from .dag import OpKind, ReduceOp
from .errors import UnsupportedNodeInFusedStep
from .tensor import DType, element_count, row_major_strides

TILE_THREADS = 256
ITEMS = 8


def generate(region: Region, kname="gr_region") -> KernelSource:
    scans = [r for r in region.roots if r.kind is OpKind.SCAN]
    if len(scans) != 1 or len(region.roots) != 1:
        raise NotFusable(scans[0] if scans else region.roots[0], "a scan runs as its own single-root step")
    s = scans[0]
    rop, axis, odt = s.op.attrs
    x = s.preds[0]
    for n in region.nodes:
        if n is not s and n.kind in (OpKind.SCAN, OpKind.REDUCE, OpKind.ARGREDUCE, OpKind.KEYED_SUM):
            raise NotFusable(n, "reductions before a scan run as their own step")
    if axis is None or len(x.shape) == 1:
        n = element_count(x.shape)
        if n > 8192:
            return _gen_lookback(region, s, x, rop, kname)
        return _gen_lines(region, s, x, rop, None, kname)
    return _gen_lines(region, s, x, rop, axis, kname)


def _gen_lines(region, s, x, rop, axis, kname, block=128) -> KernelSource:
    T = s.dtype
    ct = T.ctype
    em = LoopEmitter(region)
    if axis is None:
        kept_shape = ()
        n = element_count(x.shape)
    else:
        kept_shape = tuple(d for i, d in enumerate(x.shape) if i != axis)
        n = x.shape[axis]
    L = max(element_count(kept_shape), 1)
    rvar = Var("r", 1)
    kept = []
    rest = Aff.of(rvar)
    for d in range(len(kept_shape) - 1, -1, -1):
        if d == 0:
            kept.append(rest)
        else:
            kept.append(Aff.of(em.derived_var(1, f"{rest.c()} % {kept_shape[d]}")))
            rest = Aff.of(em.derived_var(1, f"{rest.c()} / {kept_shape[d]}"))
    kept.reverse()
    acc = em.var_decl(1, ct, c_literal(_IDENT[rop](T), T))
    k, sc, saved = em.open(1, "for", trip=n)
    if axis is None:
        coords = _flat_coords(em, x.shape, Aff.of(k), k)
        off = Aff.of(k)
    else:
        coords = list(kept[:axis]) + [Aff.of(k)] + list(kept[axis:])
        st = row_major_strides(s.shape)
        off = Aff.of(0)
        for c, sd in zip(coords, st):
            off = off + c.scale(sd)
    v = em.cast(em.value(x, coords), x.dtype, T)
    comb = _COMBINE[rop]
    em.stmt(k.level, f"{acc} = ({k.name} == 0) ? {v[0]} : {comb}<{ct}>({acc}, {v[0]});")
    em.stmt(k.level, f"p.out0[{off.c()}] = {acc};")
    em.close(sc, saved)
    lines = ["static __device__ __forceinline__ void line(const Params& p, const long long r) {"]
    lines += ["  " + c for c in em.consts]
    lines += render(em.row, 1)
    lines.append("}")
    src = [HEADER, '#include "gr_reduce.cuh"\n', "struct K {", _params_struct(region),
           f"  static constexpr long long NLINES = {L}LL;", "  " + "\n  ".join(lines), "};",
           f'extern "C" __global__ void __launch_bounds__({block}) {kname}(const K::Params p) {{',
           "  const long long stride = (long long)gridDim.x * blockDim.x;",
           "  for (long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x; r < K::NLINES; r += stride)",
           "    K::line(p, r);", "}"]
    return KernelSource("scan", "\n".join(src) + "\n", kname, list(range(len(region.leaves))), [0],
                        block=block, groups=L, vec=1, unroll=1, meta={"lines": L, "length": n, "exact": True})


def _gen_lookback(region, s, x, rop, kname) -> KernelSource:
    T = s.dtype
    ct = T.ctype
    N = element_count(x.shape)
    tile = TILE_THREADS * ITEMS
    ntiles = -(-N // tile)
    em = LoopEmitter(region, vec_loads=False)
    j, sc, saved = em.open(1, "for", trip=ITEMS, unroll=True)
    lin_name = em.emit(j.level, "long long", f"base + {j.name}")
    lin = Var(lin_name, j.level)
    cl = em.emit(j.level, "long long", f"{lin_name} < {N}LL ? {lin_name} : {N - 1}LL")
    coords = _flat_coords(em, x.shape, Aff.of(Var(cl, j.level)), j)
    v = em.cast(em.value(x, coords), x.dtype, T)
    comb = _COMBINE[rop]
    em.stmt(j.level, f"vals[{j.name}] = {v[0]};")
    em.close(sc, saved)
    ident = c_literal(_IDENT[rop](T), T)
    lines = [f"static __device__ __forceinline__ void load(const Params& p, const long long base, {ct} (&vals)[{ITEMS}]) {{"]
    lines += ["  " + c for c in em.consts]
    lines += render(em.row, 1)
    lines.append("}")
    params = _params_struct(region)
    op = _OPS[rop]
    kern = f'''extern "C" __global__ void __launch_bounds__({TILE_THREADS}) {kname}(const K::Params p) {{
  __shared__ long long tile_id;
  __shared__ {ct} wsum[{TILE_THREADS // 32}];
  __shared__ {ct} tile_prefix;
  unsigned long long* flags = reinterpret_cast<unsigned long long*>(p.scratch);
  gr::ScanState<{ct}> st{{flags + 1, reinterpret_cast<{ct}*>(flags + 1 + {ntiles}), reinterpret_cast<{ct}*>(flags + 1 + 2 * {ntiles})}};
  for (;;) {{
    if (threadIdx.x == 0) tile_id = (long long)atomicAdd(&flags[0], 1ull);
    __syncthreads();
    const long long t = tile_id;
    __syncthreads();
    if (t >= {ntiles}LL) break;
    const long long base = t * {tile}LL + (long long)threadIdx.x * {ITEMS};
    {ct} vals[{ITEMS}];
    K::load(p, base, vals);
    // thread-sequential inclusive run
#pragma unroll
    for (int i = 1; i < {ITEMS}; ++i) vals[i] = {comb}<{ct}>(vals[i - 1], vals[i]);
    const int valid = (int)(({N}LL - base) < {ITEMS} ? ({N}LL - base) : {ITEMS});
    {ct} run = valid > 0 ? vals[valid - 1] : {ident};
    // warp inclusive scan of run totals (lane order)
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    {ct} inc = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {{
      {ct} y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc = {comb}<{ct}>(y, inc);
    }}
    if (lane == 31) wsum[w] = inc;
    __syncthreads();
    if (threadIdx.x == 0) {{
      {ct} acc = wsum[0];
      for (int i = 1; i < {TILE_THREADS // 32}; ++i) {{ acc = {comb}<{ct}>(acc, wsum[i]); wsum[i] = acc; }}
      tile_prefix = gr::scan_lookback<{op}, {ct}>(st, t, acc);
    }}
    __syncthreads();
    // exclusive prefix of this thread = tile prefix (+) warps before (+) lanes before
    {ct} excl_lane = __shfl_up_sync(0xffffffffu, inc, 1);
    bool has = false;
    {ct} pre = {ident};
    if (t > 0) {{ pre = tile_prefix; has = true; }}
    if (w > 0) {{ pre = has ? {comb}<{ct}>(pre, wsum[w - 1]) : wsum[w - 1]; has = true; }}
    if (lane > 0) {{ pre = has ? {comb}<{ct}>(pre, excl_lane) : excl_lane; has = true; }}
#pragma unroll
    for (int i = 0; i < {ITEMS}; ++i) {{
      if (i < valid) p.out0[base + i] = has ? {comb}<{ct}>(pre, vals[i]) : vals[i];
    }}
    __syncthreads();
  }}
}}'''
    src = [HEADER, '#include "gr_reduce.cuh"\n', "struct K {", params, "  " + "\n  ".join(lines), "};", kern]
    scratch = 8 * (1 + ntiles) + 2 * ntiles * max(T.itemsize, 8) + 256
    return KernelSource("scan", "\n".join(src) + "\n", kname, list(range(len(region.leaves))), [0],
                        block=TILE_THREADS, groups=ntiles * TILE_THREADS, vec=1, unroll=1, scratch_bytes=scratch,
                        meta={"tiles": ntiles, "scratch_zero": True, "exact": not T.is_float,
                              "label": "scan-lookback"})
