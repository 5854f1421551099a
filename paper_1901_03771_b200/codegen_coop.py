"""Cooperative row family (K3): a thread group per long row, row in registers.

Used for regions whose reductions all reduce the full (single) column axis
of long rows — row-normalise (x - mean)/std and its total, softmax over wide
rows, row-wise argmax.  The thread-per-row family (codegen_rows.py) would
serialise a 4096-element row in one thread with uncoalesced loads; here:

* a row of C = 128·2^k elements is spread over TPR = (C/128)·P threads; thread
  (leaf l, part h) owns elements 128·l + 8·m + h·VEC + v (m < 16, v < VEC),
  i.e. VEC of NumPy's eight leaf accumulators, so every leaf access is one
  16-byte load and each warp instruction covers whole 32-byte sectors;
* every leaf the region reads along the row is loaded ONCE into registers
  (``S[16][VEC]``) and reused by every phase (sum for the mean, sum of
  squares, the normalised store, the total) — HBM sees x exactly once;
* row sums are combined as NumPy's pairwise_sum does: the 8 accumulators of a
  leaf as ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), leaves in a perfect binary tree
  (``gr::row_sum``) — bit-identical to numpy.add.reduce along the row;
* totals fold one partial per row with the last-CTA tree of gr_reduce.cuh.
"""

from __future__ import annotations

import os

from typing import Optional

from .codegen import HEADER, Aff, KernelSource, NotPairable, Region, Var, _params_struct, bcast_coords, c_literal
from .codegen_rows import (
    _COMBINE, _IDENT, _OPS, LoopEmitter, NotFusable, render, thread_space,
)
from .dag import Node, OpKind, ReduceOp
from .tensor import DType, element_count

MAX_TPR = 512


def _regular(c: int) -> bool:
    return c == 128 or (c > 128 and c % 256 == 0 and _regular(c // 2))


class CoopEmitter(LoopEmitter):
    def __init__(self, region, vec, tpr, rpc, row_shape, C):
        super().__init__(region, vec_loads=False)
        self.vec = vec
        self.tpr = tpr
        self.rpc = rpc
        self.P = 8 // vec
        self.Ts = row_shape
        self.C = C
        self.cb = Var("cb", 1, align=vec)     # thread's first column (128*l + h*VEC)
        self.coop_m: Optional[Var] = None
        self.coop_v: Optional[Var] = None
        self.staged = {}
        self.discovered = []
        self.n_sh = 0
        # paired element loops: (v, v+1) of a thread's VEC elements as one
        # gr::f2 — sums, differences, products and the shared-divisor
        # division issue once per pair (FADD2/FMUL2/FFMA2)
        self.coop_pair = False

    # col coordinate of the current coop loops
    def coop_col(self, m: Var, v: Var) -> Aff:
        if self.half is not None and v.name == self.half.name[len("gr_half_"):]:
            return Aff.of(self.cb) + Aff.of(m).scale(8) + Aff.of(v).scale(2) + Aff.of(self.half)
        return Aff.of(self.cb) + Aff.of(m).scale(8) + Aff.of(v)

    def close_coop(self, mm, vv):
        self.close(vv[1], vv[2])
        self.close(mm[1], mm[2])
        if self.half is not None and self.half.name == "gr_half_" + vv[0].name:
            self.half = None

    def prestage(self, leaves, tma_layout=None, async_layout=None, block=256):
        """Load whole row segments of ``leaves`` into registers up front: from
        the shared-memory stage filled by bulk copies (``tma_layout``: leaf id ->
        (byte offset of the leaf block, leaf stride in elements, row bytes)),
        from the per-thread cp.async stage (``async_layout``: leaf id -> byte
        offset; the fast pass reads it, then starts the next row group's
        copies), or from global memory."""
        rowkey = Aff.of(Var("r", 1)).scale(self.C).key()
        if async_layout is not None:
            names = []
            for leaf in leaves:
                name = self.fresh("S")
                self.stmt(1, f"{leaf.dtype.ctype} {name}[16][{self.vec}];")
                names.append(name)
                self.staged[(leaf.id, rowkey)] = name
            self.stmt(1, "if constexpr (FAST) {")
            self.stmt(1, "  gr::cp_async_wait_all();")
            for leaf, name in zip(leaves, names):
                T = leaf.dtype.ctype
                self.stmt(1, f"  #pragma unroll\n    for (int mm = 0; mm < 16; ++mm) gr::ldsv<{T}, {self.vec}>({name}[mm], "
                             f"reinterpret_cast<const {T}*>(stage + {async_layout[leaf.id]}) + "
                             f"((long long)mm * {block} + threadIdx.x) * {self.vec});")
            self.stmt(1, "  if (gnext < NG) copy_group(p, stage, gnext);")
            self.stmt(1, "} else {")
            for leaf, name in zip(leaves, names):
                T = leaf.dtype.ctype
                idx = self.leaf_index[leaf.id]
                self.stmt(1, f"  #pragma unroll\n    for (int mm = 0; mm < 16; ++mm) "
                             f"gr::ldv<{T}, {self.vec}>({name}[mm], p.in{idx} + r * {self.C}LL + cb + 8 * mm);")
            self.stmt(1, "}")
            return
        for leaf in leaves:
            name = self.fresh("S")
            T = leaf.dtype.ctype
            self.stmt(1, f"{T} {name}[16][{self.vec}];")
            if tma_layout is not None and leaf.id in tma_layout:
                boff, ls, rowb = tma_layout[leaf.id]
                idx = self.leaf_index[leaf.id]
                if self.div_fast:
                    self.stmt(1, "if constexpr (FAST) {")
                self.stmt(1, f"{{ const {T}* sp = reinterpret_cast<const {T}*>(stage + {boff} + (long long)ri * {rowb}) + "
                             f"(tr / {self.P}) * {ls} + (tr % {self.P}) * {self.vec};")
                self.stmt(1, f"#pragma unroll\n    for (int mm = 0; mm < 16; ++mm) gr::ldsv<{T}, {self.vec}>({name}[mm], sp + 8 * mm); }}")
                if self.div_fast:
                    # redo pass: the stage already holds the next group
                    self.stmt(1, "} else {")
                    self.stmt(1, f"#pragma unroll\n    for (int mm = 0; mm < 16; ++mm) "
                                 f"gr::ldv<{T}, {self.vec}>({name}[mm], p.in{idx} + r * {self.C}LL + cb + 8 * mm);")
                    self.stmt(1, "}")
            else:
                idx = self.leaf_index[leaf.id]
                self.stmt(1, f"#pragma unroll\n    for (int mm = 0; mm < 16; ++mm) "
                             f"gr::ldv<{T}, {self.vec}>({name}[mm], p.in{idx} + r * {self.C}LL + cb + 8 * mm);")
            self.staged[(leaf.id, rowkey)] = name

    def load_leaf(self, leaf: Node, off: Aff):
        if self.half is not None and off.coef(self.half):
            # paired loop: elements (2*vp, 2*vp + 1) of the staged segment
            for m, v in self._coop_pairs():
                if (off.coef(self.half) == 1 and off.coef(v) == 2 and off.coef(m) == 8
                        and off.coef(self.cb) == 1 and leaf.dtype is DType.f32):
                    rest = off.without(v).without(m).without(self.cb).without(self.half)
                    name = self.staged.get((leaf.id, rest.key()))
                    if name is not None and rest.level <= 1:
                        return self.emit_pair(v.level, f"gr::pk({name}[{m.name}][2 * {v.name}], "
                                                        f"{name}[{m.name}][2 * {v.name} + 1])"), v.level
            raise NotPairable("paired leaf outside the staged row segment")
        # staged row segment: offset = rest + cb + 8*m + v with m, v the coop loop vars
        for m, v in self._coop_pairs():
            if off.coef(v) == 1 and off.coef(m) == 8 and off.coef(self.cb) == 1:
                rest = off.without(v).without(m).without(self.cb)
                if rest.level <= 1 and rest.alignment() % self.vec == 0:
                    key = (leaf.id, rest.key())
                    name = self.staged.get(key)
                    if name is None:
                        self.discovered.append((leaf, rest.key()))
                        name = self.fresh("S")
                        T = leaf.dtype.ctype
                        idx = self.leaf_index[leaf.id]
                        self.stmt(1, f"{T} {name}[16][{self.vec}];")
                        self.stmt(1, f"#pragma unroll\n    for (int mm = 0; mm < 16; ++mm) "
                                     f"gr::ldv<{T}, {self.vec}>({name}[mm], p.in{idx} + {rest.c()} + cb + 8 * mm);")
                        self.staged[key] = name
                    return f"{name}[{m.name}][{v.name}]", max(v.level, off.level)
        return super().load_leaf(leaf, off)

    def _coop_pairs(self):
        out = []
        for i in range(2, len(self.stack) - 1):
            a, b = self.stack[i], self.stack[i + 1]
            if (a is not None and b is not None and a.kind == "for" and b.kind == "for" and a.trip == 16
                    and b.trip in (self.vec, self.vec // 2) and getattr(a, "coop", False)):
                out.append((a.var, b.var))
        return out

    def open_coop(self, level, paired=False):
        """Open the (m < 16, v < VEC) loops over this thread's row elements;
        ``paired``: v walks element pairs (v < VEC/2) with the pair's half as
        the symbolic ``self.half`` (values become gr::f2)."""
        m, sm, savm = self.open(level, "for", trip=16, unroll=True)
        sm.coop = True
        v, sv, savv = self.open(m.level, "for", trip=self.vec // 2 if paired else self.vec, unroll=True)
        if paired:
            self.half = Var("gr_half_" + v.name, v.level)
        return (m, sm, savm), (v, sv, savv)

    def pairable_sum(self, x: Node, rop, T: DType) -> bool:
        return (self.coop_pair and rop is ReduceOp.sum and T is DType.f32 and x.dtype is DType.f32
                and self.vec % 2 == 0)

    def _pair_map(self, n: Node, coords):
        """Packed element ops; a division by a row-level divisor keeps the
        shared-reciprocal Markstein form (two FFMA2 per pair) instead of the
        per-lane IEEE division."""
        v = shared_div_pair(self, n, coords)
        return v if v is not None else super()._pair_map(n, coords)

    # -- row-complete reductions ---------------------------------------------------
    def _row_complete(self, r: Node, axes) -> bool:
        x = r.preds[0]
        return (tuple(x.shape[:len(self.Ts)]) == self.Ts and len(x.shape) == len(self.Ts) + 1
                and x.shape[-1] == self.C and tuple(axes) == (len(self.Ts),))

    def reduce(self, r: Node, coords):
        rop, axes, keepdims, odt = r.op.attrs
        if not self._row_complete(r, axes):
            return super().reduce(r, coords)
        kept = [c for i, c in enumerate(coords) if i not in axes] if keepdims else list(coords)
        if any(c.level > 1 for c in kept):
            raise NotFusable(r, "row reduction consumed per column")
        rk = self.reduction_key(r, kept)
        hit = self.memo_get(rk)
        if hit is not None:
            return hit
        return self.memo_put(rk, (self.coop_reduce(r.preds[0], rop, r.dtype, kept), 1))

    def coop_reduce(self, x: Node, rop, T: DType, row_coords, identity=True):
        """Reduce x over this row's C columns across the TPR threads; float sums
        in NumPy pairwise order (``identity``: apply NumPy's 0.0 start)."""
        ct = T.ctype
        acc = self.fresh("acc")
        self.stmt(1, f"{ct} {acc}[{self.vec}];")
        if self.pairable_sum(x, rop, T):
            # the thread's VEC accumulators as VEC/2 packed pairs: lane v of
            # pair vp is accumulator 2*vp + v, same adds in the same order
            acc2 = self.fresh("acc")
            self.stmt(1, f"gr::f2 {acc2}[{self.vec // 2}];")
            mm, vv = self.open_coop(1, paired=True)
            m, v = mm[0], vv[0]
            val = self.value(x, list(row_coords) + [self.coop_col(m, v)])
            pv = self.splat(val)
            self.stmt(v.level, f"{acc2}[{v.name}] = ({m.name} == 0) ? {pv} : gr::p2::add({acc2}[{v.name}], {pv});")
            self.close_coop(mm, vv)
            for k in range(self.vec // 2):
                self.stmt(1, f"{acc}[{2 * k}] = gr::lo({acc2}[{k}]); {acc}[{2 * k + 1}] = gr::hi({acc2}[{k}]);")
            return self.finish_coop(acc, rop, T, identity)
        mm, vv = self.open_coop(1)
        m, v = mm[0], vv[0]
        val = self.cast(self.value(x, list(row_coords) + [self.coop_col(m, v)]), x.dtype, T)
        comb = _COMBINE[rop]
        self.stmt(v.level, f"{acc}[{v.name}] = ({m.name} == 0) ? {val[0]} : {comb}<{ct}>({acc}[{v.name}], {val[0]});")
        self.close_coop(mm, vv)
        return self.finish_coop(acc, rop, T, identity)

    def finish_coop(self, acc: str, rop, T: DType, identity=True):
        """Cross-thread combine of per-thread accumulators acc[VEC] for one row."""
        ct = T.ctype
        comb = _COMBINE[rop]
        sh = self._sh(T)
        if rop is ReduceOp.sum and T.is_float:
            tree = self.emit(1, ct, f"gr::row_sum<{ct}, {self.vec}, {self.P}, {self.tpr}, GR_ROWSUM_TRAIL>({acc}, {sh}, ri)")
            if not identity:
                return tree
            return self.emit(1, ct, f"gr::add<{ct}>({c_literal(0, T)}, {tree})")
        loc = self.fresh("lo")
        self.stmt(1, f"{ct} {loc} = {acc}[0];")
        for i in range(1, self.vec):
            self.stmt(1, f"{loc} = {comb}<{ct}>({loc}, {acc}[{i}]);")
        return self.emit(1, ct, f"gr::row_tree<{_OPS[rop]}, {ct}, {self.tpr}>({loc}, {sh}, ri)")

    def _sh(self, T: DType) -> str:
        self.n_sh += 1
        nw = max(self.tpr // 32, 1)
        name = f"sh{self.n_sh}"
        self.stmt(1, f"__shared__ {T.ctype} {name}[{self.rpc * nw}];")
        return name

    def argreduce(self, r: Node, coords):
        which, axis, keepdims = r.op.attrs
        x = r.preds[0]
        if axis is None or not self._row_complete(r, (axis,)):
            return super().argreduce(r, coords)
        kept = [c for i, c in enumerate(coords) if i != axis] if keepdims else list(coords)
        if any(c.level > 1 for c in kept):
            raise NotFusable(r, "row arg-reduction consumed per column")
        T = x.dtype.ctype
        best = self.fresh("bv")
        bi = self.fresh("bi")
        self.stmt(1, f"{T} {best} = 0; long long {bi} = -1;")
        mm, vv = self.open_coop(1)
        m, v = mm[0], vv[0]
        col = self.coop_col(m, v)
        val = self.value(x, list(kept) + [col])
        pred = "gr::arg_better_max" if which == "max" else "gr::arg_better_min"
        # within a thread the columns visit in increasing order per v lane, so
        # combine with the index-aware predicate
        self.stmt(v.level, f"{{ const long long ci = {col.c()}; if ({bi} < 0 || gr::arg_take_b<{'true' if which == 'max' else 'false'}, {T}>({best}, {bi}, {val[0]}, ci)) {{ {best} = {val[0]}; {bi} = ci; }} }}")
        self.close_coop(mm, vv)
        nw = max(self.tpr // 32, 1)
        self.n_sh += 1
        shv, shi = f"shv{self.n_sh}", f"shi{self.n_sh}"
        self.stmt(1, f"__shared__ {T} {shv}[{self.rpc * nw}]; __shared__ long long {shi}[{self.rpc * nw}];")
        mx = "true" if which == "max" else "false"
        return self.emit(1, "long long", f"gr::row_arg<{mx}, {T}, {self.tpr}>({best}, {bi}, {shv}, {shi}, ri)"), 1


def _qualifies(region: Region):
    try:
        Ts, totals, virtual = thread_space(region)
    except NotFusable:
        return None
    if virtual is not None or not Ts:
        return None
    tot_ids = {t.id for t in totals}
    C = None
    for n in region.nodes:
        if n.kind in (OpKind.REDUCE, OpKind.ARGREDUCE) and n.id not in tot_ids:
            x = n.preds[0]
            if len(x.shape) != len(Ts) + 1 or tuple(x.shape[:len(Ts)]) != Ts:
                return None
            axes = n.op.attrs[1] if n.kind is OpKind.REDUCE else (n.op.attrs[1],)
            if tuple(axes) != (len(Ts),):
                return None
            if C is None:
                C = x.shape[-1]
            elif C != x.shape[-1]:
                return None
    if C is None or C < 256 or not _regular(C):
        return None
    for r in region.roots:
        if r.id in tot_ids:
            x = r.preds[0]
            if tuple(x.shape) not in (Ts, Ts + (C,)) and element_count(x.shape[len(Ts):]) != 1:
                return None
            continue
        if tuple(r.shape) not in (Ts, Ts + (C,)) and not (tuple(r.shape[:len(Ts)]) == Ts and element_count(r.shape[len(Ts):]) == 1):
            return None
    sizes = [n.dtype.itemsize for n in region.nodes + region.leaves]
    vec = 4 if max(sizes) <= 4 else 2
    vec = min(vec, int(os.environ.get("GRUMPY_COOP_VEC", vec)))
    tpr = (C // 128) * (8 // vec)
    if tpr > MAX_TPR:
        return None
    return Ts, totals, C, vec, tpr


SMEM_PER_CTA = 110 * 1024   # two CTAs per SM keep 16 warps resident
ASYNC_SMEM_PER_CTA = 72 * 1024   # cp.async stage: three CTAs per SM
PREFETCH_GROUPS = int(os.environ.get("GRUMPY_PREFETCH_GROUPS", "2"))


def _pad_bytes(isz: int, P: int) -> int:
    """Leaf padding so a warp's 16-byte reads of the staged leaves are
    conflict-free: (leaf stride / 16) ≡ P (mod 8)."""
    base = 128 * isz // 16
    pad = 0
    while (base + pad) % 8 != P % 8:
        pad += 1
    return pad * 16


def try_generate(region: Region, kname="gr_region") -> Optional[KernelSource]:
    q = _qualifies(region)
    if q is None:
        return None
    # pass 1 discovers the row-contiguous leaves; pass 2 stages them up front,
    # through a bulk-copy ring when they fit in shared memory
    first = _generate(region, q, kname, None, None)
    if first is None:
        return None
    ks, em = first
    Ts, totals, C, vec, tpr = q
    rowkey = Aff.of(Var("r", 1)).scale(C).key()
    leaves = []
    for leaf, key in em.discovered:
        if key == rowkey and tuple(leaf.shape) == Ts + (C,) and leaf not in leaves:
            leaves.append(leaf)
    if not leaves:
        return ks
    block = max(COOP_BLOCK, tpr)
    rpc = block // tpr
    P = 8 // vec
    layout = {}
    off = 0
    for l in leaves:
        lsb = 128 * l.dtype.itemsize + _pad_bytes(l.dtype.itemsize, P)
        rowb = (C // 128) * lsb
        layout[l.id] = (off, lsb // l.dtype.itemsize, rowb)
        off += rpc * rowb
    # measured (profiles/r01_rownorm_modes.md): register staging at 3 CTAs/SM
    # 0.270 ms; per-thread cp.async stage 0.371 ms (MIO-bound); bulk-copy ring
    # 0.427 ms; L2 bulk prefetch 0.333 ms
    mode = os.environ.get("GRUMPY_COOP_MODE", "plain")
    tma = layout if (off <= SMEM_PER_CTA and mode == "tma") else None
    async_layout = None
    if mode == "async" and all(vec * l.dtype.itemsize == 16 for l in leaves):
        async_layout, aoff = {}, 0
        for l in leaves:
            async_layout[l.id] = aoff
            aoff += 16 * block * 16
        if aoff > ASYNC_SMEM_PER_CTA:
            async_layout = None
    if async_layout is not None:
        second = _generate(region, q, kname, leaves, None, smem_bytes=aoff, async_layout=async_layout)
    else:
        second = _generate(region, q, kname, leaves, tma, smem_bytes=off if tma else 0,
                           l2_prefetch=(mode == "l2" and tma is None))
    return second[0] if second is not None else ks


COOP_PAIR = os.environ.get("GRUMPY_COOP_PAIR", "1") == "1"
# debug bounds checks run the unpaired element loops
if os.environ.get("GRUMPY_DEBUG_BOUNDS", "0") == "1":
    COOP_PAIR = False
COOP_BLOCKED_TOTAL = os.environ.get("GRUMPY_COOP_BLOCKED_TOTAL", "0") == "1"
TOT_BLOCK = 4096          # rows per first-level block of a cooperative kernel's total
COOP_BLOCK = int(os.environ.get("GRUMPY_COOP_BLOCK", "256"))


def _generate(region: Region, q, kname, prestage, tma, smem_bytes=0, l2_prefetch=False, async_layout=None):
    """Generate with packed element pairs when every paired value has a packed
    form (f32), else with scalar element loops."""
    if COOP_PAIR and q[3] % 2 == 0:
        try:
            return _generate1(region, q, kname, prestage, tma, smem_bytes, l2_prefetch, async_layout, pair=True)
        except NotPairable:
            pass
    return _generate1(region, q, kname, prestage, tma, smem_bytes, l2_prefetch, async_layout, pair=False)


def _generate1(region: Region, q, kname, prestage, tma, smem_bytes=0, l2_prefetch=False, async_layout=None,
               pair=False):
    Ts, totals, C, vec, tpr = q
    tot_ids = {t.id for t in totals}
    block = max(COOP_BLOCK, tpr)
    rpc = block // tpr
    R = element_count(Ts)
    em = CoopEmitter(region, vec, tpr, rpc, Ts, C)
    em.coop_pair = pair
    em.div_fast = os.environ.get("GRUMPY_DIV_TWO_PASS", "1") != "0"
    rvar = Var("r", 1)
    if len(Ts) == 1:
        row_coords = [Aff.of(rvar)]
    else:
        row_coords = []
        rest = "r"
        for d in range(len(Ts) - 1, -1, -1):
            if d == 0:
                row_coords.append(Aff.of(Var(rest, 1)))
            else:
                c = em.emit(1, "long long", f"{rest} % {Ts[d]}")
                row_coords.append(Aff.of(Var(c, 1)))
                rest = em.emit(1, "long long", f"{rest} / {Ts[d]}")
        row_coords.reverse()

    if prestage and l2_prefetch:
        # bulk-prefetch this row's segment of the group PREFETCH_GROUPS ahead into
        # L2 (cp.async.bulk.prefetch.L2): the register staging loads of later
        # groups then hit L2, keeping HBM busy while this group is reduced
        for l in prestage:
            idx = em.leaf_index[l.id]
            isz = l.dtype.itemsize
            em.stmt(1, f"if (tr == 0) {{ const long long rp = (rb / {rpc} + {PREFETCH_GROUPS}LL * gridDim.x) * {rpc} + ri; "
                       f"if (rp < NROWS) gr::prefetch_l2(p.in{idx} + rp * {C}LL, {C * isz}u); }}")
    if prestage:
        em.prestage(prestage, tma, async_layout, block)
        if tma:
            # the stage is in registers now: release it and start the bulk copy
            # of the next row group, which then overlaps this group's compute
            em.stmt(1, "__syncthreads();")
            em.stmt(1, f"if ({'FAST' if em.div_fast else 'true'}) {{ gr::fence_proxy_async(); if (gnext < NG) issue(p, stage, bar, gnext, threadIdx.x); }}")

    # totals whose operand is itself a stored root accumulate in the store loop
    # (the value is computed once per element)
    fused_tot = {}
    for t in totals:
        x = t.preds[0]
        if (t.kind is OpKind.REDUCE and tuple(x.shape) == Ts + (C,)
                and any(x is r for r in region.roots if r.id not in tot_ids)):
            fused_tot.setdefault(x.id, []).append(t)
    tot_partials = {}
    for ri, r in enumerate(region.roots):
        if r.id in tot_ids:
            continue
        T = r.dtype.ctype
        if tuple(r.shape) == Ts + (C,):
            o = em.fresh("O")
            accs = []
            for t in fused_tot.get(r.id, []):
                a = em.fresh("acc")
                em.stmt(1, f"{t.dtype.ctype} {a}[{vec}];")
                accs.append((t, a))
            paired = (em.coop_pair and r.dtype is DType.f32 and vec % 2 == 0
                      and all(em.pairable_sum(r, t.op.attrs[0], t.dtype) for t, _a in accs))
            m, sm, savm = em.open(1, "for", trip=16, unroll=True)
            sm.coop = True
            em.stmt(m.level, f"{T} {o}[{vec}];")
            if paired:
                pacc = []
                for t, a in accs:
                    a2 = em.fresh("acc")
                    em.stmt(1, f"gr::f2 {a2}[{vec // 2}];")
                    pacc.append(a2)
                v, sv, savv = em.open(m.level, "for", trip=vec // 2, unroll=True)
                em.half = Var("gr_half_" + v.name, v.level)
                val = em.value(r, row_coords + [em.coop_col(m, v)])
                pv = em.splat(val)
                em.stmt(v.level, f"{o}[2 * {v.name}] = gr::lo({pv}); {o}[2 * {v.name} + 1] = gr::hi({pv});")
                for a2 in pacc:
                    em.stmt(v.level, f"{a2}[{v.name}] = ({m.name} == 0) ? {pv} : gr::p2::add({a2}[{v.name}], {pv});")
                em.close(sv, savv)
                em.half = None
            else:
                v, sv, savv = em.open(m.level, "for", trip=vec, unroll=True)
                val = em.value(r, row_coords + [em.coop_col(m, v)])
                em.stmt(v.level, f"{o}[{v.name}] = {val[0]};")
                for t, a in accs:
                    tv = em.cast(val, r.dtype, t.dtype)
                    comb = _COMBINE[t.op.attrs[0]]
                    em.stmt(v.level, f"{a}[{v.name}] = ({m.name} == 0) ? {tv[0]} : {comb}<{t.dtype.ctype}>({a}[{v.name}], {tv[0]});")
                em.close(sv, savv)
            em.stmt(m.level, f"if (valid) gr::stv<{T}, {vec}>(p.out{ri} + r * {C}LL + cb + 8 * {m.name}, {o});")
            em.close(sm, savm)
            if paired:
                for (t, a), a2 in zip(accs, pacc):
                    for k in range(vec // 2):
                        em.stmt(1, f"{a}[{2 * k}] = gr::lo({a2}[{k}]); {a}[{2 * k + 1}] = gr::hi({a2}[{k}]);")
            for t, a in accs:
                tot_partials[t.id] = em.finish_coop(a, t.op.attrs[0], t.dtype, identity=False)
        else:
            val = em.value(r, row_coords + [Aff.of(0)] * (len(r.shape) - len(Ts)))
            em.stmt(1, f"if (valid && tr == 0) gr::st<{T}>(p.out{ri} + r, {val[0]});")

    scratch_off = 0
    tot_meta = []
    for ri, r in enumerate(region.roots):
        if r.id not in tot_ids:
            continue
        x = r.preds[0]
        if r.kind is OpKind.ARGREDUCE:
            raise NotFusable(r, "argmax over all axes with cooperative rows")
        rop = r.op.attrs[0]
        T = r.dtype
        ct = T.ctype
        if r.id in tot_partials:
            part = tot_partials[r.id]
        elif tuple(x.shape) == Ts + (C,):
            # the partial is the bare pairwise row sum: NumPy's 0.0 start is
            # applied once, to the grand total
            part = em.coop_reduce(x, rop, T, row_coords, identity=False)
        else:
            part = em.cast(em.value(x, row_coords + [Aff.of(0)] * (len(x.shape) - len(Ts))), x.dtype, T)[0]
        off = scratch_off
        em.stmt(1, f"if (valid && tr == 0) reinterpret_cast<{ct}*>(static_cast<char*>(p.scratch) + {off})[r] = {part};")
        tot_meta.append((ri, rop, T, off))
        scratch_off += ((R * T.itemsize + 255) // 256) * 256

    P = 8 // vec
    NG = -(-R // rpc)
    two_pass = em.used_div_fast
    # (experiment, off: GRUMPY_COOP_BLOCKED_TOTAL=1) totals folded per block
    # of TOT_BLOCK rows by the warp whose row completes the block (the
    # total's perfect tree restricted to aligned blocks, so the same
    # association), then over the blocks by the last block-folder.  The
    # single last-CTA fold of every row partial was a serial tail (rownorm:
    # 0.048 of 0.235 ms); batching its loads (gr::chunk_tree) removed most of
    # it, while the per-row release atomic (MEMBAR.ALL.GPU) and row-uniform
    # redo vote of this scheme cost more (0.239 vs 0.225 ms)
    blocked_tot = (COOP_BLOCKED_TOTAL and bool(tot_meta) and R % TOT_BLOCK == 0 and 2 <= R // TOT_BLOCK <= 1000
                   and TOT_BLOCK % rpc == 0 and (R & (R - 1)) == 0)
    tot_block_off = {}
    if blocked_tot:
        for ri, rop, T, off in tot_meta:
            tot_block_off[ri] = scratch_off
            scratch_off += ((R // TOT_BLOCK) * T.itemsize + 255) // 256 * 256
    templ = two_pass or async_layout is not None
    lines = [("template <bool FAST> static __device__ __forceinline__ bool rows(" if templ else
              "static __device__ __forceinline__ void rows(") +
             "const Params& p, const long long rb, unsigned char* stage, unsigned long long* bar, const long long gnext) {",
             f"  const int tr = threadIdx.x % {tpr};",
             f"  const int ri = threadIdx.x / {tpr};",
             "  const bool valid = rb + ri < NROWS;",
             "  const long long r = valid ? rb + ri : NROWS - 1;",
             f"  const long long cb = (long long)(tr / {P}) * 128 + (tr % {P}) * {vec};",
             "  (void)stage; (void)bar; (void)gnext;"]
    if templ:
        lines.append("  bool bad = false;")
    lines += ["  " + c for c in em.consts]
    lines += render(em.row, 1)
    # a row sum's trailing barrier protects its smem slots until the next
    # barrier of the row; with two or more cross-thread combines per row
    # group another combine's barrier always comes first.  Measured: without
    # it rownorm (reductions only) 0.2377 -> 0.2358 ms, but rownorm-y (row
    # stores between the combines) 0.421 -> 0.434 ms, so only the former drops it
    stores_rows = any(tuple(r.shape) == Ts + (C,) for r in region.roots if r.id not in tot_ids)
    trail = "false" if em.n_sh >= 2 and not stores_rows else "true"
    lines = [l.replace("GR_ROWSUM_TRAIL", trail) for l in lines]
    if templ:
        lines += ["  " + l for l in em.div_finalize]
        if blocked_tot:
            NWR = max(1, tpr // 32)
            lines += [f"  __shared__ int gr_shbad[{rpc * NWR}];",
                      f"  if constexpr (FAST) bad = gr::row_tree<gr::OpMax, int, {tpr}>(bad ? 1 : 0, gr_shbad, ri) != 0;",
                      "  // count this row's final partial into its block of rows; the warp",
                      "  // whose row completes the block folds it",
                      "  {",
                      "    int kf = -1;",
                      f"    if (tr == 0 && valid && (FAST ? !bad : (((-1 - gnext) >> ri) & 1) != 0)) {{",
                      f"      const int k = (int)(r / {TOT_BLOCK});",
                      f"      if (gr::atom_add_release(p.ticket + 1 + k, 1u) + 1u == {TOT_BLOCK}u) kf = k;",
                      "    }",
                      "    if (tr < 32) {",
                      "      kf = __shfl_sync(0xffffffffu, kf, 0);",
                      "      if (kf >= 0) fold_block(p, kf);",
                      "    }",
                      "  }"]
        lines.append("  return bad;")
    lines.append("}")
    if blocked_tot:
        nb = R // TOT_BLOCK
        fb = ["static __device__ __noinline__ void fold_block(const Params& p, const int k) {",
              "  gr::fence_acq_rel();"]
        for ri, rop, T, off in tot_meta:
            ct = T.ctype
            ident = c_literal(_IDENT[rop](T), T)
            fb += [f"  {{ const {ct} v = gr::warp_range_tree<{_OPS[rop]}, {ct}, {TOT_BLOCK}LL>("
                   f"reinterpret_cast<const {ct}*>(static_cast<const char*>(p.scratch) + {off}) + (long long)k * {TOT_BLOCK}, {ident});",
                   f"    if ((threadIdx.x & 31) == 0) reinterpret_cast<{ct}*>(static_cast<char*>(p.scratch) + {tot_block_off[ri]})[k] = v; }}"]
        fb += ["  int last = 0;",
               "  if ((threadIdx.x & 31) == 0) {",
               "    p.ticket[1 + k] = 0u;",
               f"    last = gr::atom_add_release(p.ticket, 1u) + 1u == {nb}u;",
               "  }",
               "  if (__shfl_sync(0xffffffffu, last, 0)) {",
               "    gr::fence_acq_rel();"]
        for ri, rop, T, off in tot_meta:
            ct = T.ctype
            ident = c_literal(_IDENT[rop](T), T)
            fin = f"gr::add<{ct}>({c_literal(0, T)}, t{ri})" if rop is ReduceOp.sum else f"t{ri}"
            fb += [f"    const {ct} t{ri} = gr::warp_range_tree<{_OPS[rop]}, {ct}, {nb}LL>("
                   f"reinterpret_cast<const {ct}*>(static_cast<const char*>(p.scratch) + {tot_block_off[ri]}), {ident});",
                   f"    if ((threadIdx.x & 31) == 0) p.out{ri}[0] = {fin};"]
        fb += ["    if ((threadIdx.x & 31) == 0) p.ticket[0] = 0u;", "  }", "}"]
        lines = fb + lines
    issue = []
    if async_layout is not None:
        issue = ["static __device__ __forceinline__ void copy_group(const Params& p, unsigned char* stage, const long long g) {",
                 f"  const int tr = threadIdx.x % {tpr};",
                 f"  const int ri = threadIdx.x / {tpr};",
                 f"  const long long r0 = g * {rpc} + ri;",
                 "  const long long r = r0 < NROWS ? r0 : NROWS - 1;",
                 f"  const long long cb = (long long)(tr / {P}) * 128 + (tr % {P}) * {vec};"]
        for l in prestage:
            idx = region.leaves.index(l)
            issue += ["#pragma unroll",
                      f"  for (int mm = 0; mm < 16; ++mm) gr::cp_async16(stage + {async_layout[l.id]} + "
                      f"((long long)mm * {block} + threadIdx.x) * 16, p.in{idx} + r * {C}LL + cb + 8 * mm);"]
        issue += ["  gr::cp_async_commit();", "}"]
    if tma:
        nleaf = C // 128
        total = sum(nleaf * 128 * l.dtype.itemsize for l in prestage)
        # every thread issues its share of the per-leaf bulk copies: the copy
        # instruction is uniform-operand, so one warp issuing them all
        # serialises them (0.328 -> 0.251 ms on rownorm when spread)
        issue = ["static __device__ __forceinline__ void issue(const Params& p, unsigned char* stage, unsigned long long* bar, const long long g, const int lane) {",
                 f"  const long long nvalid = (g * {rpc} + {rpc} <= NROWS) ? {rpc} : (NROWS - g * {rpc});",
                 f"  if (lane == 0) gr::mbar_arrive_expect_tx(bar, (unsigned)(nvalid * {total}));"]
        for l in prestage:
            boff, ls, rowb = tma[l.id]
            lsb = ls * l.dtype.itemsize
            idx = region.leaves.index(l)
            issue += [f"  for (int c = lane; c < {rpc * nleaf}; c += {block}) {{",
                      f"    const int qq = c / {nleaf}, lf = c % {nleaf};",
                      f"    if (qq < nvalid) gr::bulk_g2s(stage + {boff} + (long long)qq * {rowb} + (long long)lf * {lsb}, "
                      f"p.in{idx} + (g * {rpc} + qq) * {C}LL + (long long)lf * 128, {128 * l.dtype.itemsize}u, bar);",
                      "  }"]
        issue.append("}")
    # per-row redo flags (two-pass division) replace a CTA-wide vote per row
    # group: rows whose fast pass saw a dividend outside the shared-divisor
    # window are flagged and redone exactly after the CTA's last group
    row_redo = two_pass and async_layout is None
    params = _params_struct(region).replace("    void* __restrict__ scratch;",
                                             "    void* __restrict__ scratch;\n    unsigned int* ticket;"
                                             + ("\n    unsigned int* redo;" if row_redo else ""))
    src = [HEADER, '#include "gr_reduce.cuh"\n#include "gr_tma.cuh"\n', "struct K {", params,
           f"  static constexpr long long NROWS = {R}LL;",
           f"  static constexpr long long NG = {NG}LL;"]
    if issue:
        src.append("  " + "\n  ".join(issue))
    src.append("  " + "\n  ".join(lines))
    src.append("};")
    def _redo_tail(smem_arg, bar_arg, next_arg="K::NG"):
        """flag bad rows during the loop; after it, redo flagged row groups
        (uniform per group: the flags are read after a CTA barrier) and clear
        the flags, so the buffer is zero again for the next launch"""
        # the CTA's threads first check all its groups' flags at once (one L2
        # round trip; a loop of dependent flag loads was a serial tail of
        # ~20 us), and walk the groups only when one is flagged
        return ["  __syncthreads();",
                "  bool gr_any = false;",
                "  for (long long g = blockIdx.x + (long long)threadIdx.x * gridDim.x; g < K::NG; g += (long long)blockDim.x * gridDim.x)",
                f"    gr_any |= ((__ldcg(p.redo + ((g * {rpc}) >> 5)) >> ((g * {rpc}) & 31)) & {(1 << rpc) - 1}u) != 0u;",
                "  if (__syncthreads_or(gr_any))",
                "  for (long long g = blockIdx.x; g < K::NG; g += gridDim.x) {",
                f"    const unsigned bits = (__ldcg(p.redo + ((g * {rpc}) >> 5)) >> ((g * {rpc}) & 31)) & {(1 << rpc) - 1}u;",
                "    if (bits) {",
                "      __syncthreads();",
                f"      if (threadIdx.x == 0) atomicAnd(p.redo + ((g * {rpc}) >> 5), ~({(1 << rpc) - 1}u << ((g * {rpc}) & 31)));",
                f"      K::rows<false>(p, g * {rpc}, {smem_arg}, {bar_arg}, {next_arg});",
                "    }",
                "  }"]

    def _flag(call):
        return [f"    if ({call}) atomicOr(p.redo + ((g * {rpc} + threadIdx.x / {tpr}) >> 5), 1u << ((g * {rpc} + threadIdx.x / {tpr}) & 31));"]
    if tma:
        # residency is set by the stage size: cap registers to match it
        tminb = max(1, min(4, (227 * 1024) // (smem_bytes + 2048)))
        kern = [f'extern "C" __global__ void __launch_bounds__({block}, {tminb}) {kname}(const K::Params p) {{',
                "  extern __shared__ __align__(128) unsigned char smem[];",
                "  __shared__ unsigned long long bar;",
                "  if (threadIdx.x == 0) { gr::mbar_init(&bar, 1); gr::fence_mbar_init(); }",
                "  __syncthreads();",
                "  long long g = blockIdx.x;",
                "  if (g < K::NG) K::issue(p, smem, &bar, g, threadIdx.x);",
                "  for (int it = 0; g < K::NG; g += gridDim.x, ++it) {",
                "    gr::mbar_wait(&bar, (unsigned)(it & 1));"]
        if two_pass:
            # the redo pass re-reads its rows from global memory
            kern += _flag(f"K::rows<true>(p, g * {rpc}, smem, &bar, g + gridDim.x)")
            kern.append("  }")
            kern += _redo_tail("smem", "&bar")
        else:
            kern.append(f"    K::rows(p, g * {rpc}, smem, &bar, g + gridDim.x);")
            kern.append("  }")
    elif async_layout is not None:
        minb = int(os.environ.get("GRUMPY_COOP_MINBLOCKS", "3"))
        kern = [f'extern "C" __global__ void __launch_bounds__({block}, {minb}) {kname}(const K::Params p) {{',
                "  extern __shared__ __align__(128) unsigned char smem[];",
                "  if (blockIdx.x < K::NG) K::copy_group(p, smem, blockIdx.x);",
                "  for (long long g = blockIdx.x; g < K::NG; g += gridDim.x) {"]
        if two_pass:
            kern += [f"    if (__syncthreads_or(K::rows<true>(p, g * {rpc}, smem, nullptr, g + gridDim.x)))",
                     f"      K::rows<false>(p, g * {rpc}, smem, nullptr, g + gridDim.x);"]
        else:
            kern.append(f"    K::rows<true>(p, g * {rpc}, smem, nullptr, g + gridDim.x);")
        kern.append("  }")
    else:
        # register staging holds 16*VEC elements per staged leaf; with one f32
        # leaf (64 registers) capping the kernel at 80 registers fits three
        # CTAs per SM: 0.270 ms vs 0.307 ms at two (profiles/r01_rownorm_modes.md)
        data_regs = sum(16 * vec * l.dtype.itemsize // 4 for l in (prestage or []))
        minb = int(os.environ.get("GRUMPY_COOP_MINBLOCKS", str(768 // block) if 0 < data_regs <= 64 else "0"))
        lb = f"{block}, {minb}" if minb else f"{block}"
        kern = [f'extern "C" __global__ void __launch_bounds__({lb}) {kname}(const K::Params p) {{',
                f"  for (long long g = blockIdx.x; g < K::NG; g += gridDim.x) {{"]
        if two_pass:
            # fast pass; rows where a dividend left the shared-divisor window
            # (gr::div_sh) are flagged and redone exactly after the loop
            # (a CTA-wide vote per group cost 0.269 vs 0.243 ms on rownorm)
            kern += _flag(f"K::rows<true>(p, g * {rpc}, nullptr, nullptr, 0)")
            kern.append("  }")
            # blocked totals: the redo pass counts only the redone rows (their
            # mask travels in gnext as -1 - bits)
            kern += _redo_tail("nullptr", "nullptr", "-1 - (long long)bits" if blocked_tot else "K::NG")
        else:
            kern.append(f"    K::rows(p, g * {rpc}, nullptr, nullptr, 0);")
            kern.append("  }")
    if tot_meta and blocked_tot:
        pass      # the warps completing a block fold it (K::fold_block); no grid-end fold
    elif tot_meta:
        kern.append("  if (gr::last_block(p.ticket)) {")
        for ri, rop, T, off in tot_meta:
            ct = T.ctype
            ident = c_literal(_IDENT[rop](T), T)
            kern.append(f"    const {ct} v{ri} = gr::block_tree<{_OPS[rop]}, {ct}>("
                        f"reinterpret_cast<const {ct}*>(static_cast<const char*>(p.scratch) + {off}), K::NROWS, {ident});")
            fin = f"gr::add<{ct}>({c_literal(0, T)}, v{ri})" if rop is ReduceOp.sum else f"v{ri}"
            kern.append(f"    if (threadIdx.x == 0) p.out{ri}[0] = {fin};")
        kern.append("  }")
    kern.append("}")
    src += kern
    ks = KernelSource("coop", "\n".join(src) + "\n", kname,
                      leaf_slots=list(range(len(region.leaves))),
                      root_slots=list(range(len(region.roots))),
                      block=block, groups=NG * block, vec=vec, unroll=1, scratch_bytes=scratch_off,
                      meta={"rows": R, "row_shape": Ts, "cols": C, "tpr": tpr, "rows_per_cta": rpc,
                            "redo_words": -(-R // 32) if row_redo else 0,
                            "totals": len(tot_meta), "ticket": bool(tot_meta), "smem": smem_bytes,
                            "bulk_copy": bool(tma), "cp_async": async_layout is not None,
                            "label": "coop-tma" if tma else ("coop-async" if async_layout is not None else "coop")})
    return ks, em


def shared_div_pair(em, n: Node, coords):
    """A packed division by a row-level (shared) divisor: one reciprocal per
    row, the Markstein correction as two FFMA2 per pair; with the emitter's
    two-pass division (``div_fast``) the dividends' range is tracked and the
    row is redone exactly when any left the window.  None when ``n`` is not
    such a division."""
    from .dag import ElemCode
    if not (n.op.code is ElemCode.div and n.loop[0] is DType.f32 and n.dtype is DType.f32):
        return None
    a = em.cast(em.value(n.preds[0], bcast_coords(coords, n.shape, n.preds[0].shape)), n.preds[0].dtype, n.loop[0])
    b = em.cast(em.value(n.preds[1], bcast_coords(coords, n.shape, n.preds[1].shape)), n.preds[1].dtype, n.loop[1])
    if not (em.is_pair(a) and not em.is_pair(b) and b[1] < a[1]):
        return None
    rk = ("rcp", b[0])
    r = em.const_memo.get(rk)
    if r is None or b[1] > 0:
        r = em.emit(b[1], "gr::DivShared<float>", f"gr::div_prep<float>({b[0]})")
        if b[1] == 0:
            em.const_memo[rk] = r
    r2 = em.const_memo.get(("rcp2", r))
    if r2 is None:
        r2 = em.emit(max(b[1], 0), "gr::p2::DivShared2", f"gr::p2::div_prep2({r})")
        em.const_memo[("rcp2", r)] = r2
    if em.div_fast and b[1] == 1:
        w = em.const_memo.get(("divrange", r))
        if w is None:
            w = em.fresh("w")
            em.stmt(1, f"gr::DivRange<float> {w} = gr::div_range_init<float>();")
            em.const_memo[("divrange", r)] = w
            em.div_finalize.append(f"bad |= gr::div_range_bad<float>({w}, {r});")
        em.used_div_fast = True
        return em.emit_pair(a[1], f"gr::p2::div_shr<FAST>({a[0]}, {r2}, {w})"), a[1]
    if not em.div_fast:
        return em.emit_pair(a[1], f"gr::p2::div_shared({a[0]}, {r2})"), a[1]
    raise NotPairable("paired division outside the row-divisor form")
