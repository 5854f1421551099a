"""Map-scan family: cumsum / cumprod / maximum.accumulate with a fused map prologue.

Reference: run_map_scan: inclusive scan of
the mapped values along one axis, a three-phase blocked scan on CPU threads
(SPEC.md:385); PAPER.md:545-551 (map-scan primitive).  NumPy's accumulate is a
sequential left fold along the axis (out[k] = out[k-1] ⊕ x[k]).

* scans along an axis with many independent lines keep that order exactly
  (bit-identical to NumPy): a thread per line when lines are strided
  (``_gen_lines``), a warp per 16 lines through a padded shared tile when
  they are contiguous (``_gen_rows_t``);
* long scans (1-D, flat n-D, or few long lines as segments) run as one
  single-pass kernel: tiles dealt round-robin over a persistent grid, each
  tile's aggregate published in a 64-bit status word (value and flag, no
  fences), and a look-back by rounds — the prefix of tile t is the CTA's own
  inclusive prefix of tile t - G combined with a warp tree of the G - 1
  aggregates in between (``gr::round_tree``), so no look-back waits for
  another.  ``_gen_lookback_tma`` feeds the tiles by TMA through a shared
  ring (the default); ``_gen_lookback`` stages them through registers for the
  layouts TMA cannot take.  Deterministic; float results within the
  reassociation bound of NumPy's sequential fold, integers and max exact.
"""

from __future__ import annotations

import os
from typing import List

from .codegen import HEADER, Aff, KernelSource, Region, Var, _params_struct, bcast_coords, c_literal
from .codegen_rows import _COMBINE, _IDENT, _OPS, LoopEmitter, NotFusable, render, _flat_coords
from .dag import OpKind, ReduceOp
from .errors import UnsupportedNodeInFusedStep
from .tensor import DType, element_count, row_major_strides

ITEMS = 16

# Long 1-D scans whose inputs are contiguous arrays of the scan's length: TMA
# tile ring (see _gen_lookback_tma)
SCAN_TMA = os.environ.get("GRUMPY_SCAN_TMA", "1") == "1"
SCAN_TMA_MIN = 1 << 20
SCAN_TMA_SMEM = 200 * 1024
SCAN_TMA_STAGES = int(os.environ.get("GRUMPY_SCAN_STAGES", "6"))
SCAN_TMA_LAG = int(os.environ.get("GRUMPY_SCAN_LAG", "2"))   # 3 with the left fold (GRUMPY_SCAN_TREE=0)
SCAN_TMA_LBW = int(os.environ.get("GRUMPY_SCAN_LBW", "1"))   # 2 with the left fold
SCAN_TMA_ITEMS = int(os.environ.get("GRUMPY_SCAN_ITEMS", "16"))
# look-back by rounds (gr::tile_lookback_round): the prefix starts from the
# CTA's own inclusive prefix of one round earlier instead of the nearest one
# another CTA published
SCAN_TMA_ROUND = os.environ.get("GRUMPY_SCAN_ROUND", "1") == "1"
# the aggregates of a round combined as a warp tree (not a left fold)
SCAN_TMA_TREE = os.environ.get("GRUMPY_SCAN_TREE", "1") == "1"
# the register-staged kernel with the same look-back (static round-robin
# tiles over its persistent grid); off: dynamic claims + nearest-prefix walk
SCAN_REG_ROUNDS = os.environ.get("GRUMPY_SCAN_REG_ROUNDS", "1") == "1"


def generate(region: Region, kname="gr_region") -> KernelSource:
    scans = [r for r in region.roots if r.kind is OpKind.SCAN]
    if len(scans) != 1 or len(region.roots) != 1:
        raise NotFusable(scans[0] if scans else region.roots[0], "a scan runs as its own single-root step")
    s = scans[0]
    rop, axis, odt = s.op.attrs
    x = s.preds[0]
    seed = s.preds[1] if len(s.preds) > 1 else None
    for n in region.nodes:
        if n is not s and n.kind in (OpKind.SCAN, OpKind.REDUCE, OpKind.ARGREDUCE, OpKind.KEYED_SUM):
            raise NotFusable(n, "reductions before a scan run as their own step")
    if axis is None or len(x.shape) == 1:
        n = element_count(x.shape)
        if SCAN_TMA and n >= SCAN_TMA_MIN:
            try:
                # an n-D operand is scanned in its flat row-major order
                ks = _gen_lookback_tma(region, s, x, rop, kname, flat=len(x.shape) > 1)
                if ks is not None:
                    return ks
            except NotFusable:
                pass
        if n > 8192:
            return _gen_lookback(region, s, x, rop, kname)
        return _gen_lines(region, s, x, rop, None, kname)
    if axis == len(x.shape) - 1 and seed is None and x.shape[-1] > 1:
        lines = element_count(x.shape[:-1])
        if lines < ROWS_T_MIN_LINES and element_count(x.shape) >= SCAN_TMA_MIN and x.shape[-1] >= 8192:
            # too few lines for a warp per 16 of them to fill the GPU: one
            # look-back scan per line (tolerance instead of NumPy's order) —
            # the TMA kernel when lines are whole tiles, else register-staged
            if SCAN_TMA:
                try:
                    ks = _gen_lookback_tma(region, s, x, rop, kname)
                    if ks is not None:
                        return ks
                except NotFusable:
                    pass
            return _gen_lookback(region, s, x, rop, kname, segments=True)
        if ROWS_T and lines >= 32:
            return _gen_rows_t(region, s, x, rop, kname)
    return _gen_lines(region, s, x, rop, axis, kname)


# scans along the contiguous (last) axis: a warp per 16 lines, staged through
# shared memory so loads and stores are coalesced (see _gen_rows_t)
ROWS_T = os.environ.get("GRUMPY_SCAN_ROWS_T", "1") == "1"
ROWS_T_CW = int(os.environ.get("GRUMPY_SCAN_ROWS_CW", "64"))       # columns per chunk
# below this many lines a scan along the last axis whose lines are whole
# look-back tiles runs as one look-back scan per line (_gen_lookback_tma)
# (the warp-per-16-lines kernel keeps one 64-column chunk per line in flight:
# it needs ~28 warps per SM to stream at full rate — 16384x16384 took 0.95 ms
# there against 0.34 segmented, 65536x4096 0.41 ms; tools/rows_mid_probe.py)
ROWS_T_MIN_LINES = int(os.environ.get("GRUMPY_SCAN_ROWS_MIN_LINES", str(148 * 16 * 28)))
ROWS_T_RPW = int(os.environ.get("GRUMPY_SCAN_ROWS_RPW", "16"))     # lines per warp (16 lanes fold; measured 0.415 vs 0.427 ms for 32)
ROWS_T_WPB = int(os.environ.get("GRUMPY_SCAN_ROWS_WPB", "1"))      # warps per CTA (1: even spread of the 32-line groups over the SMs)


def _gen_rows_t(region, s, x, rop, kname) -> KernelSource:
    """Scan along the contiguous last axis, one warp per RPW (16) lines.

    A thread per line (``_gen_lines``) reads 32 different lines per warp
    instruction there — 32 cache lines per request in both directions.  Here a
    warp takes RPW lines a chunk of CW columns at a time: the map prologue is
    evaluated with lanes along the columns (coalesced loads, one 128-byte line
    per instruction) into a padded shared tile, each lane folds its own line's
    chunk sequentially in place (stride CW+1: conflict-free), and the chunk
    leaves with lanes along the columns again (coalesced stores).  The fold is
    NumPy's sequential left fold per line, so results are bit-identical to
    the thread-per-line kernel."""
    T = s.dtype
    ct = T.ctype
    shape = tuple(x.shape)
    n = shape[-1]
    kept_shape = shape[:-1]
    L = element_count(kept_shape)
    CW, WPB, RPW = ROWS_T_CW, ROWS_T_WPB, ROWS_T_RPW
    em = LoopEmitter(region)
    rvar, kvar = Var("r", 1), Var("k", 1)
    kept = []
    rest = Aff.of(rvar)
    for d in range(len(kept_shape) - 1, -1, -1):
        if d == 0:
            kept.append(rest)
        else:
            kept.append(Aff.of(em.derived_var(1, f"{rest.c()} % {kept_shape[d]}")))
            rest = Aff.of(em.derived_var(1, f"{rest.c()} / {kept_shape[d]}"))
    kept.reverse()
    v = em.cast(em.value(x, kept + [Aff.of(kvar)]), x.dtype, T)
    fn = [f"static __device__ __forceinline__ {ct} val(const Params& p, const long long r, const long long k) {{"]
    fn += ["  " + c for c in em.consts]
    fn += render(em.row, 1)
    fn += [f"  return {v[0]};", "}"]
    comb = _COMBINE[rop]
    H = CW // 32
    # the shared tile stays within the 48 KB of static shared memory
    WPB = max(1, min(WPB, (48 * 1024) // (RPW * (CW + 1) * T.itemsize)))
    kern = f"""extern "C" __global__ void __launch_bounds__({32 * WPB}) {kname}(const K::Params p) {{
  __shared__ {ct} tile[{WPB}][{RPW}][{CW + 1}];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  {ct} (*tl)[{CW + 1}] = tile[w];
  constexpr long long NG = (K::NLINES + {RPW - 1}) / {RPW};
  {ct} v[{RPW}][{H}];
  // map prologue of one chunk, lanes along the columns: coalesced loads
  auto load = [&](const long long r0, const long long c0) {{
#pragma unroll
    for (int j = 0; j < {RPW}; ++j) {{
#pragma unroll
      for (int h = 0; h < {H}; ++h) {{
        const long long r = r0 + j, k = c0 + 32 * h + lane;
        if (r < K::NLINES && k < K::N) v[j][h] = K::val(p, r, k);
      }}
    }}
  }};
  for (long long g = (long long)blockIdx.x * {WPB} + w; g < NG; g += (long long)gridDim.x * {WPB}) {{
    const long long r0 = g * {RPW};
    {ct} acc = {c_literal(_IDENT[rop](T), T)};
    load(r0, 0);
    for (long long c0 = 0; c0 < K::N; c0 += {CW}) {{
#pragma unroll
      for (int j = 0; j < {RPW}; ++j) {{
#pragma unroll
        for (int h = 0; h < {H}; ++h) tl[j][32 * h + lane] = v[j][h];
      }}
      __syncwarp();
      // the next chunk's loads are in flight while this one is folded and stored
      if (c0 + {CW} < K::N) load(r0, c0 + {CW});
      // each lane folds its own line's chunk in place (NumPy's order)
      if (lane >= {RPW}) {{
      }} else if (c0 > 0 && c0 + {CW} <= K::N) {{
#pragma unroll
        for (int k = 0; k < {CW}; ++k) {{ acc = {comb}<{ct}>(acc, tl[lane][k]); tl[lane][k] = acc; }}
      }} else {{
        const int cn = K::N - c0 < {CW} ? (int)(K::N - c0) : {CW};
        int k0 = 0;
        if (c0 == 0) {{ acc = tl[lane][0]; k0 = 1; }}
        for (int k = k0; k < cn; ++k) {{ acc = {comb}<{ct}>(acc, tl[lane][k]); tl[lane][k] = acc; }}
      }}
      __syncwarp();
#pragma unroll
      for (int j = 0; j < {RPW}; ++j) {{
#pragma unroll
        for (int h = 0; h < {H}; ++h) {{
          const long long r = r0 + j, k = c0 + 32 * h + lane;
          if (r < K::NLINES && k < K::N) p.out0[r * K::N + k] = tl[j][32 * h + lane];
        }}
      }}
      __syncwarp();
    }}
  }}
}}"""
    src = [HEADER, '#include "gr_reduce.cuh"\n', "struct K {", _params_struct(region),
           f"  static constexpr long long NLINES = {L}LL;", f"  static constexpr long long N = {n}LL;",
           "  " + "\n  ".join(fn), "};", kern]
    ng = -(-L // RPW)
    return KernelSource("scan", "\n".join(src) + "\n", kname, list(range(len(region.leaves))), [0],
                        block=32 * WPB, groups=ng * 32, vec=1, unroll=1,
                        meta={"lines": L, "length": n, "exact": True, "label": "scan-rows"})


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
    seed = s.preds[1] if len(s.preds) > 1 else None
    if seed is not None:
        # seeded fold (a streamed chunk's carry): the line starts from its seed
        sv = em.cast(em.value(seed, bcast_coords(kept, kept_shape, seed.shape) if kept_shape else [Aff.of(0)] * len(seed.shape)),
                     seed.dtype, T)
        acc = em.var_decl(1, ct, sv[0])
    else:
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
    if seed is not None:
        em.stmt(k.level, f"{acc} = {comb}<{ct}>({acc}, {v[0]});")
    else:
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


def _gen_lookback(region, s, x, rop, kname, segments=False) -> KernelSource:
    """One pass over a long 1-D scan: 4096-element tiles, coalesced (vector)
    loads of the map prologue into a padded shared tile, a thread-sequential
    run per thread, warp and CTA combines, and the deterministic look-back of
    gr::tile_lookback; results leave through the shared tile as coalesced
    vector stores.

    A matrix scanned along its last axis runs as one such scan per line
    (segments): every line starts at a tile boundary (ceil(n / tile) tiles per
    line, the last one partial) and the look-back stops at the line's first
    tile."""
    T = s.dtype
    ct = T.ctype
    N = element_count(x.shape)
    # 8192-element tiles (fewer tiles in flight: shorter look-back walks);
    # 4096 for 8-byte types so the shared tile stays within 48 KB
    TILE_THREADS = int(os.environ.get("GRUMPY_SCAN_TPB", "512")) if T.itemsize <= 4 else 256
    tile = TILE_THREADS * ITEMS
    n_seg = x.shape[-1] if segments else N               # segment (line) length
    TPL = -(-n_seg // tile)                              # tiles per segment
    ntiles = TPL * (N // n_seg)
    SW = 1 if T.itemsize <= 4 else 2      # 64-bit status words per published value
    vec = max(1, min(4, 16 // max(T.itemsize, x.dtype.itemsize)))
    # every tile starts on a vector boundary (tile bases are multiples of the
    # tile in one long scan; a line's tiles start at multiples of its length)
    aligned = not segments or n_seg % vec == 0
    chunks = ITEMS // vec
    ident = c_literal(_IDENT[rop](T), T)
    comb = _COMBINE[rop]
    seed = s.preds[1] if len(s.preds) > 1 else None
    seeded = "true" if seed is not None else "false"
    seed_fn = _seed_fn(region, seed, T)
    seedv = "K::seed_value(p)" if seed is not None else c_literal(_IDENT[rop](T), T)
    op = _OPS[rop]

    def load_fn(name, full):
        # element e of the tile = j*(TPB*vec) + vec*tid + v (striped, coalesced)
        em = LoopEmitter(region, vec_loads=full)
        tb = Var("tb", 1, align=tile)
        tt = Var("tt", 1)
        j, sj, a = em.open(1, "for", trip=chunks, unroll=True)
        v, sv, b = em.open(j.level, "for", trip=vec, unroll=True)
        e = Aff.of(j).scale(TILE_THREADS * vec) + Aff.of(tt).scale(vec) + Aff.of(v)
        if full:
            lin = Aff.of(tb) + e
        else:
            raw = em.emit(v.level, "long long", f"tb + {e.c()}")
            lin = Aff.of(Var(em.emit(v.level, "long long", f"{raw} < lim ? {raw} : lim - 1"), v.level))
        coords = _flat_coords(em, x.shape, lin, v)
        val = em.cast(em.value(x, coords), x.dtype, T)
        keep = "" if full else f"(tb + {e.c()} < lim) ? "
        tail = "" if full else f" : {ident}"
        em.stmt(v.level, f"buf[gr::spad({e.c()})] = {keep}{val[0]}{tail};")
        em.close(sv, b)
        em.close(sj, a)
        out = [f"static __device__ __forceinline__ void {name}(const Params& p, const long long tb, const long long lim, {ct}* buf) {{",
               "  const long long tt = threadIdx.x; (void)lim;"]
        out += ["  " + c for c in em.consts]
        out += render(em.row, 1)
        out.append("}")
        return out

    lines = load_fn("load_full", True) + load_fn("load_tail", False)
    params = _params_struct(region)
    TP = tile + tile // 32          # padded shared tile
    NTH = TILE_THREADS + 32         # + the look-back warp
    # residency: two shared tiles per CTA; cap registers so the shared memory,
    # not the register file, sets the CTAs per SM
    minb = max(1, min(int(os.environ.get("GRUMPY_SCAN_MINB", "8")), (227 * 1024) // (2 * TP * T.itemsize + 1024)))
    REG_ROUNDS_C = "true" if SCAN_REG_ROUNDS else "false"
    if SCAN_REG_ROUNDS:
        # static round-robin tiles over the persistent grid (every CTA
        # resident) and the look-back by rounds with a warp tree, as in the
        # TMA kernel (gr::round_tree)
        ls_expr = f"(t / {TPL}LL) * {TPL}LL"
        lookback = f'''      {ct} pre;
      if (t % {TPL}LL == 0) {{ pre = {seedv}; own = tagg[i & 1]; }}
      else {{
        const {ct} tree = gr::round_tree<{op}, {ct}>(aggs, t, (int)gridDim.x, {ls_expr}, {ident});
        pre = t - (long long)gridDim.x < {ls_expr} ? tree : {comb}<{ct}>(own, tree);
        own = {comb}<{ct}>(pre, tagg[i & 1]);
      }}'''
        first_tile = f"  t = blockIdx.x < {ntiles}LL ? (long long)blockIdx.x : -1;"
        next_tile = f"    const long long tn = t + gridDim.x < {ntiles}LL ? t + gridDim.x : -1;"
    else:
        # dynamic tile claims and the nearest-published-prefix walk
        # (gr::tile_lookback); a seed (streamed carry) joins tile 0: its
        # inclusive prefix is seed (+) aggregate, its exclusive prefix the seed
        lookback = f'''      const {ct} pre0 = gr::tile_lookback<{op}, {ct}>(aggs, incs, t, {seeded} && t == 0 ? {comb}<{ct}>({seedv}, tagg[i & 1]) : tagg[i & 1], {ident}, (t / {TPL}LL) * {TPL}LL);
      const {ct} pre = {seeded} && t == 0 ? {seedv} : pre0;'''
        first_tile = f'''  {{
    if (threadIdx.x == 0) next_id = (long long)atomicAdd(counter, 1ull);
    asm volatile("bar.sync 1, {TILE_THREADS};" ::: "memory");
    t = next_id < {ntiles}LL ? next_id : -1;
    asm volatile("bar.sync 1, {TILE_THREADS};" ::: "memory");
  }}'''
        next_tile = f'''    if (threadIdx.x == 0) next_id = (long long)atomicAdd(counter, 1ull);
    asm volatile("bar.sync 1, {TILE_THREADS};" ::: "memory");
    const long long tn = next_id < {ntiles}LL ? next_id : -1;
    asm volatile("bar.sync 1, {TILE_THREADS};" ::: "memory");'''
    kern = f'''extern "C" __global__ void __launch_bounds__({NTH}, {minb}) {kname}(const K::Params p) {{
  // warps 0..{TILE_THREADS // 32 - 1}: data (load, tile-local scan, store) over two shared tiles;
  // warp {TILE_THREADS // 32}: look-back — tile i's prefix is resolved while the data warps
  // load and scan tile i+1 (named barriers: 1 data warps, 2 "staged", 3 "prefix ready")
  extern __shared__ __align__(16) unsigned char smem_raw[];
  {ct}* bufs = reinterpret_cast<{ct}*>(smem_raw);
  __shared__ {ct} wsum[2][{TILE_THREADS // 32}];
  __shared__ {ct} tagg[2];
  __shared__ {ct} tpre[2];
  __shared__ long long tids[2];
  __shared__ long long next_id;
  unsigned long long* counter = reinterpret_cast<unsigned long long*>(p.scratch);
  unsigned long long* aggs = counter + 1;                       // tile aggregates (status words)
  unsigned long long* incs = aggs + {ntiles * SW}LL;            // tile inclusive prefixes
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (w == {TILE_THREADS // 32}) {{
    {ct} own = {ident};   // rounds: this CTA's inclusive prefix of its previous tile
    (void)own;
    for (int i = 0;; ++i) {{
#ifdef GR_SCAN_STATS
      const long long cw = clock64();
#endif
      asm volatile("bar.sync 2, {NTH};" ::: "memory");
#ifdef GR_SCAN_STATS
      if (lane == 0) atomicAdd(&gr::gr_scan_stats[3], (unsigned long long)(clock64() - cw));
#endif
      const long long t = tids[i & 1];
      if (t < 0) break;
{lookback}
      if (lane == 0) tpre[i & 1] = pre;
      asm volatile("bar.arrive 3, {NTH};" ::: "memory");
    }}
    return;
  }}
  // ---- data warps
  long long t;
{first_tile}
  int b = 0;
  if (t >= 0) K::stage(p, t, bufs, wsum[0], &tagg[0], &tids[0], aggs, lane, w);
  else if (threadIdx.x == 0) tids[0] = -1;
  asm volatile("bar.arrive 2, {NTH};" ::: "memory");
  while (t >= 0) {{
{next_tile}
    if (tn >= 0) K::stage(p, tn, bufs + (b ^ 1) * {TP}LL, wsum[b ^ 1], &tagg[b ^ 1], &tids[b ^ 1], aggs, lane, w);
    asm volatile("bar.sync 3, {NTH};" ::: "memory");
    // tile t: prefix (+) tile-local inclusive scan, coalesced stores
    {{
      const {ct}* buf = bufs + b * {TP}LL;
      const {ct} pre = tpre[b];
      const long long ln = t / {TPL}LL, tc = t % {TPL}LL;
      const long long tb = ln * {n_seg}LL + tc * {tile}LL;
      const long long lim = ln * {n_seg}LL + ({n_seg}LL < (tc + 1) * {tile}LL ? {n_seg}LL : (tc + 1) * {tile}LL);
#pragma unroll
      for (int j = 0; j < {chunks}; ++j) {{
        const long long e = (long long)j * {TILE_THREADS * vec} + {vec} * threadIdx.x;
        {ct} o[{vec}];
#pragma unroll
        for (int v = 0; v < {vec}; ++v) {{ const {ct} x = buf[gr::spad(e + v)]; o[v] = (tc > 0 || {seeded}) ? {comb}<{ct}>(pre, x) : x; }}
        if ({"true" if aligned else "false"} && tb + e + {vec} <= lim) {{
          gr::stv<{ct}, {vec}>(p.out0 + tb + e, o);
        }} else {{
          for (int v = 0; v < {vec}; ++v) if (tb + e + v < lim) p.out0[tb + e + v] = o[v];
        }}
      }}
    }}
    if (tn < 0 && threadIdx.x == 0) tids[b ^ 1] = -1;
    asm volatile("bar.sync 1, {TILE_THREADS};" ::: "memory");   // buffer b free, tids visible
    asm volatile("bar.arrive 2, {NTH};" ::: "memory");
    t = tn;
    b ^= 1;
  }}
}}'''
    stage = [f"static __device__ __forceinline__ void stage(const Params& p, const long long t, {ct}* buf, {ct}* ws, {ct}* agg_s, long long* tid_s, unsigned long long* aggs, const int lane, const int w) {{",
             f"  const long long ln = t / {TPL}LL, tc = t % {TPL}LL;",
             f"  const long long tb = ln * {n_seg}LL + tc * {tile}LL;",
             f"  const long long lim = ln * {n_seg}LL + ({n_seg}LL < (tc + 1) * {tile}LL ? {n_seg}LL : (tc + 1) * {tile}LL);",
             f"  if ({'true' if aligned else 'false'} && tb + {tile}LL <= lim) load_full(p, tb, lim, buf); else load_tail(p, tb, lim, buf);",
             f'  asm volatile("bar.sync 1, {TILE_THREADS};" ::: "memory");',
             f"  {ct} vals[{ITEMS}];",
             "#pragma unroll",
             f"  for (int i = 0; i < {ITEMS}; ++i) vals[i] = buf[gr::spad({ITEMS} * threadIdx.x + i)];",
             "#pragma unroll",
             f"  for (int i = 1; i < {ITEMS}; ++i) vals[i] = {comb}<{ct}>(vals[i - 1], vals[i]);",
             f"  {ct} inc = vals[{ITEMS - 1}];",
             "#pragma unroll",
             "  for (int o = 1; o < 32; o <<= 1) {",
             f"    const {ct} y = __shfl_up_sync(0xffffffffu, inc, o);",
             f"    if (lane >= o) inc = {comb}<{ct}>(y, inc);",
             "  }",
             "  if (lane == 31) ws[w] = inc;",
             f'  asm volatile("bar.sync 1, {TILE_THREADS};" ::: "memory");',
             "  if (threadIdx.x == 0) {",
             f"    {ct} acc = ws[0];",
             f"    for (int i = 1; i < {TILE_THREADS // 32}; ++i) {{ acc = {comb}<{ct}>(acc, ws[i]); ws[i] = acc; }}",
             f"    if ({seeded} && {REG_ROUNDS_C} && t == 0) acc = {comb}<{ct}>({seedv}, acc);   // rounds: tile 0's aggregate carries the seed",
             "    *agg_s = acc;",
             "    *tid_s = t;",
             f"    gr::stat_put<{ct}>(aggs, t, acc);",
             "  }",
             f'  asm volatile("bar.sync 1, {TILE_THREADS};" ::: "memory");',
             f"  const {ct} lane_ex = __shfl_up_sync(0xffffffffu, inc, 1);",
             "  bool has = false;",
             f"  {ct} loc = {ident};",
             "  if (w > 0) { loc = ws[w - 1]; has = true; }",
             f"  if (lane > 0) {{ loc = has ? {comb}<{ct}>(loc, lane_ex) : lane_ex; has = true; }}",
             "#pragma unroll",
             f"  for (int i = 0; i < {ITEMS}; ++i) buf[gr::spad({ITEMS} * threadIdx.x + i)] = has ? {comb}<{ct}>(loc, vals[i]) : vals[i];",
             f'  asm volatile("bar.sync 1, {TILE_THREADS};" ::: "memory");',
             "}"]
    lines = lines + stage + seed_fn
    src = [HEADER, '#include "gr_reduce.cuh"\n', "struct K {", params, "  " + "\n  ".join(lines), "};", kern]
    scratch = 8 + 8 * SW * 2 * ntiles + 256
    return KernelSource("scan", "\n".join(src) + "\n", kname, list(range(len(region.leaves))), [0],
                        block=NTH, groups=ntiles * NTH, vec=1, unroll=1, scratch_bytes=scratch,
                        meta={"tiles": ntiles, "scratch_zero": True, "exact": not T.is_float,
                              "label": "scan-lookback", "smem": 2 * TP * T.itemsize})


class _StagedEmitter(LoopEmitter):
    """Loop emitter whose staged leaves are read from a swizzled shared-memory
    tile (16-byte chunks, gr::lds_sw) instead of global memory."""

    def __init__(self, region, staged, tvars, flat=None):
        super().__init__(region, vec_loads=True)
        self.staged = staged      # leaf id -> name of the tile's base pointer
        self.tvars = tvars        # [(var, coef)]: the tile's first element = sum(coef * var)
        # flat scans of an n-D operand: (the operand's row-major offset of the
        # element, its offset within the tile without the vector lane, the
        # vector-lane loop variable); a staged leaf read at exactly that
        # offset is the tile's element
        self.flat = flat

    def bounds_exempt(self, leaf):
        # staged leaves come from the TMA tile (out-of-range lanes of the
        # last tile read zero fill, never global memory)
        return leaf.id in self.staged

    def load_leaf(self, leaf, off):
        sym = self.staged.get(leaf.id)
        if sym is None:
            if off.level >= 2:
                raise NotFusable(leaf, "unstaged leaf read per element")
            return super().load_leaf(leaf, off)
        if self.flat is not None:
            expect, rel, vv, trip = self.flat
            if off.key() != expect.key():
                raise NotFusable(leaf, "staged leaf read off the tile")
            return self._staged_vec(leaf, sym, rel, vv, trip)
        lvl = off.level
        sc = self.stack[lvl] if lvl >= 2 else None
        if sc is None or sc.kind != "for" or not sc.unroll or sc.var is None or off.coef(sc.var) != 1:
            raise NotFusable(leaf, "staged leaf not read along the item loop")
        rest = off.without(sc.var)
        if any(rest.coef(tv) != c for tv, c in self.tvars) or sc.trip * leaf.dtype.itemsize != 16:
            raise NotFusable(leaf, "staged leaf read off the tile")
        rel = rest
        for tv, _ in self.tvars:
            rel = rel.without(tv)
        return self._staged_vec(leaf, sym, rel, sc.var, sc.trip)

    def _staged_vec(self, leaf, sym, rel, vv, trip):
        """The staged leaf's vector at tile offset ``rel`` (one 16-byte chunk,
        loaded once per chunk), indexed by the vector-lane loop ``vv``."""
        lvl = vv.level
        key = ("svec", leaf.id, rel.key())
        hit = self.memo.get(key)
        if hit is not None and (hit[1] == 0 or (hit[1] < len(self.stack) and self.stack[hit[1]] is hit[2])):
            return f"{hit[0]}[{vv.name}]", lvl
        T = leaf.dtype.ctype
        name = self.fresh("L")
        plvl = max(rel.level, 1)
        self.stmt(plvl, f"{T} {name}[{trip}];")
        self.stmt(plvl, f"gr::lds_sw<{T}, {trip}>({name}, {sym}, (unsigned){rel.c()});")
        self.memo[key] = (name, plvl, self.stack[plvl] if plvl > 0 else None)
        return f"{name}[{vv.name}]", lvl


def _gen_lookback_tma(region, s, x, rop, kname, flat=False):
    """Single-pass look-back scan fed by TMA (sm_100a).

    A producer warp streams each input leaf's 32 KB tile into a ring of
    shared-memory stages with cp.async.bulk.tensor (128-byte swizzle,
    mbarrier completion) as far ahead as the ring allows, so the loads of
    the next tiles are always in flight; 16 data warps read their 16
    consecutive elements per thread straight from the swizzled tile
    (conflict-free 16-byte chunks), evaluate the map prologue in registers and
    scan (thread run, warp, CTA), and look-back warps resolve the tile prefix
    while the data warps scan the next tiles.  The finished tile is written
    back into its stage and leaves with one TMA tensor store.

    Tiles go round-robin over a persistent grid of G CTAs (one per SM, all
    resident), so the look-back is by rounds: the prefix of tile t is the
    CTA's own inclusive prefix of tile t - G combined with the G - 1
    aggregates in between — one L2 round trip, and it never waits for
    another CTA's look-back (the nearest-published-prefix walk of
    gr::tile_lookback made a chain of them: 0.51 ms at 2^28).  The default
    combines those aggregates as a warp tree (gr::round_tree: ~100 cycles
    after the loads, so two tiles of lag hide the look-back; 0.341 ms, more
    accurate than a left fold, deterministic for a given grid).  With
    GRUMPY_SCAN_TREE=0 they are left-folded by one lane (gr::round_stage /
    round_fold, the register-staged kernel's association, bit-identical to
    it; 1.8k cycles per fold, two look-back warps alternate tiles and hand
    the CTA's prefix over in shared memory: 0.40 ms)."""
    T = s.dtype
    ct = T.ctype
    N = element_count(x.shape)
    isz = T.itemsize
    if isz not in (4, 8):
        return None
    staged = [l for l in region.leaves if tuple(l.shape) == tuple(x.shape)]
    if not staged or any(l.dtype.itemsize != isz for l in staged):
        return None
    W = 128 // isz                       # elements per 128-byte line
    # TMA moves whole 128-byte lines: the last N % W elements of a 1-D scan
    # (the tail) are read and written by the threads that own them
    NM = N - N % W
    TPB = 512 if isz == 4 else 256
    ITEMS = SCAN_TMA_ITEMS                # elements per data thread (16: 32 KB tiles, 32: 64 KB)
    tile = TPB * ITEMS
    segmented = len(x.shape) > 1 and not flat
    if N % W and (segmented or NM < 2 * tile):
        return None
    # segments: a scan along the last axis of a matrix is one scan per line;
    # lines made of whole tiles keep every tile inside one line
    seg = x.shape[-1] if segmented else N
    if seg % tile and segmented:
        return None
    TPL = seg // tile if segmented else -(-N // tile)     # tiles per segment
    tile_b = tile * isz                  # 32 KB
    rows = tile // W                     # 128-byte lines per tile
    box = min(rows, 256)                 # TMA box: at most 256 lines (32 KB)
    nbox = rows // box
    ntiles = -(-N // tile)
    NL = len(staged)
    S_ = min(SCAN_TMA_STAGES, SCAN_TMA_SMEM // (NL * tile_b))
    if S_ < 3:
        return None
    vec = 16 // isz
    NW = TPB // 32
    ident = c_literal(_IDENT[rop](T), T)
    comb = _COMBINE[rop]
    seed = s.preds[1] if len(s.preds) > 1 else None
    seeded = "true" if seed is not None else "false"
    seed_fn = _seed_fn(region, seed, T)
    seedv = "K::seed_value(p)" if seed is not None else c_literal(_IDENT[rop](T), T)
    op = _OPS[rop]

    # ---- per-thread items: the map prologue on 16 consecutive elements
    tb = Var("tb", 1, align=tile)
    tt = Var("tt", 1)
    if len(x.shape) == 1:
        em = _StagedEmitter(region, {l.id: f"sg{k}" for k, l in enumerate(staged)}, [(tb, 1)])
        tile_coords = lambda e_: [Aff.of(tb) + e_]        # noqa: E731
    elif flat:
        em = _StagedEmitter(region, {l.id: f"sg{k}" for k, l in enumerate(staged)}, [])
        tile_coords = None
    else:
        # the tile's line and first column; the line's kept coordinates
        tln, tkb = Var("tln", 1), Var("tkb", 1, align=tile)
        em = _StagedEmitter(region, {l.id: f"sg{k}" for k, l in enumerate(staged)}, [])
        kept_shape = x.shape[:-1]
        kept, rest_, stride = [], tln, seg
        for d in range(len(kept_shape) - 1, -1, -1):
            # the tile's base is sum(coordinate_d * stride_d) over the line's coordinates
            cv = rest_ if d == 0 else em.derived_var(1, f"{rest_.name} % {kept_shape[d]}")
            kept.append(Aff.of(cv))
            em.tvars.append((cv, stride))
            stride *= kept_shape[d]
            if d:
                rest_ = em.derived_var(1, f"{rest_.name} / {kept_shape[d]}")
        kept.reverse()
        em.tvars.append((tkb, 1))
        tile_coords = lambda e_: kept + [Aff.of(tkb) + e_]    # noqa: E731
    j, sj, a = em.open(1, "for", trip=ITEMS // vec, unroll=True)
    v, sv, b = em.open(j.level, "for", trip=vec, unroll=True)
    e = Aff.of(tt).scale(ITEMS) + Aff.of(j).scale(vec) + Aff.of(v)
    if tile_coords is None:
        # flat order of an n-D operand: its coordinates from the flat index;
        # identity-mapped contiguous leaves are read at exactly the operand's
        # row-major offset, i.e. the tile's element
        coords = _flat_coords(em, x.shape, Aff.of(tb) + e, v)
        expect = Aff.of(0)
        for c, sd in zip(coords, row_major_strides(x.shape)):
            expect = expect + c.scale(sd)
        em.flat = (expect, Aff.of(tt).scale(ITEMS) + Aff.of(j).scale(vec), v, vec)
        tile_coords = lambda e_: coords     # noqa: E731
    val = em.cast(em.value(x, tile_coords(e)), x.dtype, T)
    em.stmt(v.level, f"vals[{vec} * {j.name} + {v.name}] = {val[0]};")
    em.close(sv, b)
    em.close(sj, a)
    args = "".join(f", const unsigned char* sg{k}" for k in range(NL))
    items = [f"static __device__ __forceinline__ void items(const Params& p, const long long tb{args}, {ct} (&vals)[{ITEMS}]) {{",
             "  const long long tt = threadIdx.x; (void)tb;"]
    if segmented:
        items.append(f"  const long long tln = tb / {seg}LL, tkb = tb % {seg}LL;")
    items += ["  " + c for c in em.consts]
    items += render(em.row, 1)
    items.append("}")
    body = "\n".join(items)
    for i, l in enumerate(region.leaves):
        if l in staged and f"p.in{i}" in body:
            raise NotFusable(l, "staged leaf also read from global memory")
    tail_fn, tail_load, tail_store = [], "", ""
    if NM < N:
        # the tail's mapped values straight from global memory
        te = LoopEmitter(region)
        ix = Var("ix", 1)
        tv = te.cast(te.value(x, _flat_coords(te, x.shape, Aff.of(ix), ix)), x.dtype, T)
        tail_fn = [f"static __device__ __forceinline__ {ct} tail_value(const Params& p, const long long ix) {{"]
        tail_fn += ["  " + c for c in te.consts] + render(te.row, 1) + [f"  return {tv[0]};", "}"]
        tail_load = f'''    if (t == {ntiles - 1}LL) {{
#pragma unroll
      for (int k2 = 0; k2 < {ITEMS}; ++k2) {{
        const long long ix = t * {tile}LL + {ITEMS} * threadIdx.x + k2;
        if (ix >= {NM}LL && ix < {N}LL) vals[k2] = K::tail_value(p, ix);
      }}
    }}'''
        tail_store = f'''      if (tj == {ntiles - 1}LL) {{
#pragma unroll
        for (int k2 = 0; k2 < {vec}; ++k2) {{
          const long long ix = tj * {tile}LL + {ITEMS} * threadIdx.x + {vec} * q + k2;
          if (ix >= {NM}LL && ix < {N}LL) p.out0[ix] = o[k2];
        }}
      }}'''

    params = _params_struct(region)
    maps = "".join(f"    gr::TMap tmap{k};\n" for k in range(NL + 1))
    params = params.replace("  struct Params {\n", "  struct Params {\n" + maps, 1)
    LAG = min(SCAN_TMA_LAG, S_ - 2)       # tiles waiting for their prefix
    NLW = SCAN_TMA_LBW                    # look-back warps
    rounds = SCAN_TMA_ROUND
    if segmented and not rounds:
        return None                      # segments need the look-back by rounds
    ls_expr = f"(t / {TPL}LL) * {TPL}LL"
    if rounds and SCAN_TMA_TREE:
        # the aggregates since the CTA's previous tile combined as a warp tree
        # (gr::round_tree) before the CTA's inclusive prefix is needed
        take_own = ("" if NLW == 1 else
                    f"""        if (i > 0) {{
          gr::mbar_wait(&own_bar, (i - 1) & 1);
          own = own_v;
        }}
""")
        give_own = "" if NLW == 1 else "\n      __syncwarp();   // every lane has read own_v\n      if (lane == 0) { own_v = own; gr::mbar_arrive(&own_bar); }"
        lb_call = f"""      {ct} pre;
      if (t % {TPL}LL == 0) {{
{take_own}        pre = {seedv}; own = mb_agg[m];
      }} else {{
        const {ct} tree = gr::round_tree<{op}, {ct}>(aggs, t, (int)gridDim.x, {ls_expr}, {ident});
{take_own}        pre = t - (long long)gridDim.x < {ls_expr} ? tree : {comb}<{ct}>(own, tree);
        own = {comb}<{ct}>(pre, mb_agg[m]);
      }}{give_own}"""
    elif rounds and NLW == 1:
        # the data warps publish tile 0's aggregate with the seed folded in
        lb_call = f"""      {ct} pre;
      if (t % {TPL}LL == 0) {{ pre = {seedv}; own = mb_agg[m]; }}
      else {{
        pre = gr::tile_lookback_round<{op}, {ct}>(aggs, t, (int)gridDim.x, (t / {TPL}LL) * {TPL}LL, own, {ident}, lbw[k].v);
        own = {comb}<{ct}>(pre, mb_agg[m]);
      }}"""
    elif rounds:
        # several look-back warps take the iterations in turn: each stages its
        # tile's aggregates while the previous warp folds, then takes over the
        # CTA's inclusive prefix (own_v, sequence-numbered) for its own fold
        lb_call = f"""      {ct} pre;
      // a segment's first tile has no prefix, but it still takes its turn in
      // the CTA's sequence of inclusive prefixes (own_bar counts iterations)
      const bool s0 = t % {TPL}LL == 0;
      if (!s0) gr::round_stage<{op}, {ct}>(aggs, t, (int)gridDim.x, (t / {TPL}LL) * {TPL}LL, {ident}, lbw[k].v);
      if (i > 0) {{
        gr::mbar_wait(&own_bar, (i - 1) & 1);
        own = own_v;
      }}
      if (s0) {{ pre = {seedv}; own = mb_agg[m]; }}
      else {{
        pre = gr::round_fold<{op}, {ct}>(t, (int)gridDim.x, (t / {TPL}LL) * {TPL}LL, own, {ident}, lbw[k].v);
        own = {comb}<{ct}>(pre, mb_agg[m]);
      }}
      __syncwarp();   // every lane has read own_v
      if (lane == 0) {{ own_v = own; gr::mbar_arrive(&own_bar); }}"""
    else:
        lb_call = (f"      const {ct} pre0 = gr::tile_lookback_buf<{op}, {ct}>(aggs, incs, t, {seeded} && t == 0 ? "
                   f"{comb}<{ct}>({seedv}, mb_agg[m]) : mb_agg[m], {ident}, lbw[k].v);\n"
                   f"      const {ct} pre = {seeded} && t == 0 ? {seedv} : pre0;")
    agg0 = f"{seeded} && t == 0 ? {comb}<{ct}>({seedv}, acc) : acc" if rounds else "acc"
    M = LAG + NLW                         # mailbox slots
    NTH = TPB + 32 * NLW + 32
    sgs = ", ".join(f"ring + ((long long)s * {NL} + {k}) * {tile_b}" for k in range(NL))
    loads = "\n".join(f"        gr::tma_load_2d(ring + ((long long)s * {NL} + {k}) * {tile_b} + {b * box * 128}, &p.tmap{k}, 0, (int)(t * {rows} + {b * box}), &full[s]);"
                      for k in range(NL) for b in range(nbox))
    kern = f"""extern "C" __global__ void __launch_bounds__({NTH}, 1) {kname}(const __grid_constant__ K::Params p) {{
  // warps 0..{NW - 1}: data (scan); warps {NW}..{NW + NLW - 1}: look-back (iteration i
  // goes to warp NW + i % {NLW}); warp {NW + NLW}: TMA producer.  A tile's
  // locally scanned values wait in its stage for {LAG} iterations while its
  // prefix resolves; mailboxes in shared memory hand tiles to the look-back
  // warps and prefixes back (sequence-numbered, volatile + block fences).
  extern __shared__ unsigned char smem_raw[];
  unsigned char* ring = smem_raw + ((1024u - (gr::smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ unsigned long long full[{S_}], empty[{S_}];
  __shared__ long long stid[{S_}];
  __shared__ {ct} wsum[2][{NW}];
  __shared__ long long mb_tid[{M}];
  __shared__ {ct} mb_agg[{M}], mb_pre[{M}];
  // mailbox slot m carries iterations m, m + {M}, ...: its k-th use is phase
  // k of mb_pub[m] (tile published) and mb_done[m] (prefix ready)
  __shared__ unsigned long long mb_pub[{M}], mb_done[{M}];
  __shared__ gr::LookbackBuf<{ct}> lbw[{NLW}];
  // several look-back warps: the CTA's inclusive prefix handed from
  // iteration i to i + 1 (phase i of own_bar)
  __shared__ {ct} own_v;
  __shared__ unsigned long long own_bar;
  unsigned long long* aggs = reinterpret_cast<unsigned long long*>(p.scratch) + 1;
  unsigned long long* incs = aggs + {ntiles * (1 if isz <= 4 else 2)}LL;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) {{
    for (int i = 0; i < {S_}; ++i) {{ gr::mbar_init(&full[i], 1); gr::mbar_init(&empty[i], 1); }}
    for (int i = 0; i < {M}; ++i) {{ gr::mbar_init(&mb_pub[i], 1); gr::mbar_init(&mb_done[i], 1); }}
    gr::mbar_init(&own_bar, 1);
    gr::fence_mbar_init();
  }}
  __syncthreads();
  if (w == {NW + NLW}) {{
    if (lane == 0) {{
      for (int i = 0;; ++i) {{
        const int s = i % {S_};
        if (i >= {S_}) gr::mbar_wait(&empty[s], ((i / {S_}) - 1) & 1);
        // static round-robin tiles: the grid is persistent (one CTA per SM, all
        // resident), so tiles are processed in rounds of gridDim.x and a tile's
        // look-back reaches back about one round, however deep the ring
        const long long t = (long long)blockIdx.x + (long long)i * gridDim.x;
        if (t >= {ntiles}LL) {{ stid[s] = -1; gr::mbar_arrive(&full[s]); break; }}
        stid[s] = t;
        gr::mbar_arrive_expect_tx(&full[s], {NL * tile_b}u);
{loads}
      }}
    }}
    return;
  }}
  if (w >= {NW}) {{
    const int k = w - {NW};
    {ct} own = {ident};   // round look-back: this CTA's inclusive prefix of its previous tile
    (void)own;
    for (int i = k;; i += {NLW}) {{
      const int m = i % {M};
#ifdef GR_SCAN_STATS
      const long long cw = clock64();
#endif
      gr::mbar_wait(&mb_pub[m], (i / {M}) & 1);
#ifdef GR_SCAN_STATS
      if (lane == 0 && blockIdx.x == 0) {{ if (i == 0) {{ gr::gr_scan_stats[4] = gr::gr_scan_stats[5] = gr::gr_scan_stats[6] = gr::gr_scan_stats[7] = 0; gr::gr_scan_stats[3] = clock64(); }}
                                          else gr::gr_scan_stats[7] += clock64() - cw; }}
#endif
      const long long t = mb_tid[m];
      if (t < 0) {{
#ifdef GR_SCAN_STATS
        if (blockIdx.x == 0 && lane == 0) {{
          const unsigned long long* q = gr::gr_scan_stats;
          printf("GR_SCAN_STATS CTA 0: look-backs=%llu load+wait=%llu fold=%llu mailbox-idle=%llu cycles per look-back, %llu cycles in all\\n",
                 q[6], q[4] / (q[6] + 1), q[5] / (q[6] + 1), q[7] / (q[6] + 1), (unsigned long long)clock64() - q[3]);
        }}
#endif
        break;
      }}
{lb_call}
      if (lane == 0) {{ mb_pre[m] = pre; gr::mbar_arrive(&mb_done[m]); }}
      __syncwarp();
    }}
    return;
  }}
  // ---- data warps
  long long ptid[{LAG + 1}];
  int srel = -1;
  auto finalize = [&](const int j, const long long tj) {{
    // tile of iteration j: prefix (+) its tile-local scan (waiting in its
    // stage), back into the stage, one TMA store
    const int m = j % {M};
    if (threadIdx.x == 0) gr::mbar_wait(&mb_done[m], (j / {M}) & 1);
    asm volatile("bar.sync 1, {TPB};" ::: "memory");
    const {ct} pre = mb_pre[m];
    unsigned char* ob = ring + (long long)(j % {S_}) * {NL * tile_b};
#pragma unroll
    for (int q = 0; q < {ITEMS // vec}; ++q) {{
      {ct} o[{vec}];
      gr::lds_sw<{ct}, {vec}>(o, ob, {ITEMS} * threadIdx.x + {vec} * q);
      if (tj % {TPL}LL != 0 || {seeded}) {{
#pragma unroll
        for (int k2 = 0; k2 < {vec}; ++k2) o[k2] = {comb}<{ct}>(pre, o[k2]);
        gr::sts_sw<{ct}, {vec}>(ob, {ITEMS} * threadIdx.x + {vec} * q, o);
      }}
{tail_store}
    }}
    gr::fence_proxy_async();
    asm volatile("bar.sync 1, {TPB};" ::: "memory");
    if (threadIdx.x == 0) {{
      for (int b = 0; b < {nbox}; ++b) gr::tma_store_2d(&p.tmap{NL}, 0, (int)(tj * {rows} + b * {box}), ob + b * {box * 128});
      gr::bulk_commit();
      gr::bulk_wait_read<1>();
      if (srel >= 0) gr::mbar_arrive(&empty[srel]);
    }}
    srel = j % {S_};
  }};
  for (int i = 0;; ++i) {{
    const int s = i % {S_};
    gr::mbar_wait(&full[s], (i / {S_}) & 1);
    const long long t = stid[s];
    if (t < 0) {{
      if (threadIdx.x == 0) {{
        for (int e = 0; e < {NLW}; ++e) {{ mb_tid[(i + e) % {M}] = -1; gr::mbar_arrive(&mb_pub[(i + e) % {M}]); }}
      }}
      for (int j = (i > {LAG} ? i - {LAG} : 0); j < i; ++j) finalize(j, ptid[j % {LAG + 1}]);
      break;
    }}
    {ct} vals[{ITEMS}];
    unsigned char* sb = ring + (long long)s * {NL * tile_b};
    K::items(p, t * {tile}LL, {sgs}, vals);
{tail_load}
#pragma unroll
    for (int k2 = 1; k2 < {ITEMS}; ++k2) vals[k2] = {comb}<{ct}>(vals[k2 - 1], vals[k2]);
    {ct} inc = vals[{ITEMS - 1}];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {{
      const {ct} y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc = {comb}<{ct}>(y, inc);
    }}
    {ct}* ws = wsum[i & 1];
    if (lane == 31) ws[w] = inc;
    asm volatile("bar.sync 1, {TPB};" ::: "memory");
    if (threadIdx.x == 0) {{
      {ct} acc = ws[0];
      for (int k2 = 1; k2 < {NW}; ++k2) {{ acc = {comb}<{ct}>(acc, ws[k2]); ws[k2] = acc; }}
      const {ct} agg = {agg0};
      gr::stat_put<{ct}>(aggs, t, agg);
      const int m = i % {M};
      mb_tid[m] = t;
      mb_agg[m] = agg;
      gr::mbar_arrive(&mb_pub[m]);          // release: the waiting look-back warp sees tid and agg
    }}
    asm volatile("bar.sync 1, {TPB};" ::: "memory");
    const {ct} lane_ex = __shfl_up_sync(0xffffffffu, inc, 1);
    bool has = false;
    {ct} loc = {ident};
    if (w > 0) {{ loc = ws[w - 1]; has = true; }}
    if (lane > 0) {{ loc = has ? {comb}<{ct}>(loc, lane_ex) : lane_ex; has = true; }}
    // tile-local inclusive scan back into the stage (this thread's own chunks)
#pragma unroll
    for (int q = 0; q < {ITEMS // vec}; ++q) {{
      {ct} o[{vec}];
#pragma unroll
      for (int k2 = 0; k2 < {vec}; ++k2) o[k2] = has ? {comb}<{ct}>(loc, vals[{vec} * q + k2]) : vals[{vec} * q + k2];
      gr::sts_sw<{ct}, {vec}>(sb, {ITEMS} * threadIdx.x + {vec} * q, o);
    }}
    ptid[i % {LAG + 1}] = t;
    if (i >= {LAG}) finalize(i - {LAG}, ptid[(i - {LAG}) % {LAG + 1}]);
  }}
  if (threadIdx.x == 0) gr::bulk_wait<0>();
}}"""
    pre = "".join(f"#define {d.replace('=', ' ', 1)}\n" for d in os.environ.get("GRUMPY_SCAN_DEFINES", "").split(",") if d)  # experiments
    src = [pre + HEADER, '#include "gr_reduce.cuh"\n#include "gr_tma.cuh"\n', "struct K {", params,
           "  " + body.replace("\n", "\n  "), "  " + "\n  ".join(seed_fn + tail_fn), "};", kern]
    scratch = 8 + 8 * (1 if isz <= 4 else 2) * 2 * ntiles + 256
    slots = [region.leaves.index(l) for l in staged]
    tmaps = [(i, W, NM // W, W, box, 128) for i in slots] + [(len(region.leaves), W, NM // W, W, box, 128)]
    return KernelSource("scan", "\n".join(src) + "\n", kname, list(range(len(region.leaves))), [0],
                        block=NTH, groups=ntiles * NTH, vec=1, unroll=1, scratch_bytes=scratch,
                        meta={"tiles": ntiles, "scratch_zero": True, "exact": not T.is_float,
                              "label": "scan-tma", "smem": S_ * NL * tile_b + 1024, "tmaps": tmaps,
                              "stages": S_})


def _seed_fn(region, seed, T):
    """K::seed_value(p): the value seeding a long scan (a streamed chunk's
    carry — a view of the previous chunk's result), through the region's
    index maps."""
    if seed is None:
        return []
    se = LoopEmitter(region)
    v = se.cast(se.value(seed, [Aff.of(0)] * len(seed.shape)), seed.dtype, T)
    out = [f"static __device__ __forceinline__ {T.ctype} seed_value(const Params& p) {{"]
    out += ["  " + c for c in se.consts]
    out += render(se.row, 1)
    out += [f"  return {v[0]};", "}"]
    return out
