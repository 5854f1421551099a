"""Row-streaming family (K3 on B200): one warp per row, rows fed by TMA bulk copies.

Regions whose reductions all reduce one long contiguous row axis
(row-normalise (x - mean)/std + total, softmax/argmax over wide rows, row
sums) are bandwidth-bound; the design goal is to keep HBM busy while rows are
reduced in several dependent phases (mean → variance → normalised output):

* each warp owns whole rows (32 lanes ↔ the row's 128-element leaves, so
  every cross-lane combine is a warp shuffle — no CTA barriers);
* every input read along the row is streamed into a per-warp shared-memory
  ring of NS stages by ``cp.async.bulk`` (one 512 B bulk copy per leaf, issued
  by the lanes in parallel, completion on an mbarrier with expect_tx); the
  copy for row g+NS-1 is issued before row g is processed, so NS-1 rows per
  warp are always in flight;
* leaves sit 16 B apart in shared memory (stride 528 B for f32) so the lanes'
  8-element reads (two LDS.128) are bank-conflict free;
* sums follow NumPy's pairwise order exactly: lane-owned leaf = 8 sequential
  accumulators combined ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), leaves in a
  perfect binary tree (in-lane, then shuffles) — bit-identical to
  numpy.add.reduce along the row.
"""

from __future__ import annotations

import os
from typing import Optional

from .codegen import HEADER, Aff, KernelSource, NotPairable, Region, Var, _params_struct, c_literal
from .codegen_rows import _COMBINE, _IDENT, _OPS, LoopEmitter, NotFusable, render, thread_space
from .dag import Node, OpKind, ReduceOp
from .tensor import DType, element_count

SMEM_BUDGET = 200 * 1024
WROW_DIV_TWO_PASS = os.environ.get("GRUMPY_WROW_TWO_PASS", "1") == "1"


def _regular(c: int) -> bool:
    return c == 128 or (c > 128 and c % 256 == 0 and _regular(c // 2))


class WrowEmitter(LoopEmitter):
    def __init__(self, region, Ts, C, lpr, lpl, rpw):
        super().__init__(region, vec_loads=False)
        self.Ts = Ts
        self.C = C
        self.lpr = lpr          # lanes per row
        self.lpl = lpl          # leaves per lane
        self.rpw = rpw          # rows per warp
        self.lfb = Var("lfb", 1, align=128)   # first column of this lane's leaves
        self.staged = []        # leaf nodes streamed through shared memory
        self.staged_ptr = {}
        self.pair = False       # float row sums over element pairs (f32x2)

    # -- the (li, m, j) loops over a lane's elements --------------------------------
    def open_elem(self, level=1):
        li, sli, a = self.open(level, "for", trip=self.lpl, unroll=True)
        sli.coop = "li"
        m, sm, b = self.open(li.level, "for", trip=16, unroll=True)
        sm.coop = "m"
        j, sj, c = self.open(m.level, "for", trip=8, unroll=True)
        sj.coop = "j"
        return (li, sli, a), (m, sm, b), (j, sj, c)

    def close_elem(self, L):
        for v, s, saved in reversed(L):
            self.close(s, saved)

    def col(self, li: Var, m: Var, j: Var) -> Aff:
        return Aff.of(self.lfb) + Aff.of(li).scale(128) + Aff.of(m).scale(8) + Aff.of(j)

    def _roles(self):
        roles = {}
        for s in self.stack[2:]:
            if s is not None and s.coop:
                roles[s.coop] = s
        return roles

    def load_leaf(self, leaf: Node, off: Aff):
        roles = self._roles()
        if {"li", "m", "jp"} <= set(roles) and self.half is not None:
            li, m, jp = roles["li"].var, roles["m"].var, roles["jp"].var
            if (off.coef(jp) == 2 and off.coef(self.half) == 1 and off.coef(m) == 8 and off.coef(li) == 128
                    and off.coef(self.lfb) == 1 and tuple(leaf.shape) == self.Ts + (self.C,)
                    and leaf.dtype is DType.f32):
                rest = off.without(jp).without(self.half).without(m).without(li).without(self.lfb)
                if rest.key() == Aff.of(Var("r", 1)).scale(self.C).key():
                    name = self._lds(leaf, li, m)
                    return self.emit_pair(jp.level, f"gr::pk({name}[2 * {jp.name}], {name}[2 * {jp.name} + 1])"), jp.level
            raise NotPairable("paired row element off the staged leaf")
        if {"li", "m", "j"} <= set(roles):
            li, m, j = roles["li"].var, roles["m"].var, roles["j"].var
            if (off.coef(j) == 1 and off.coef(m) == 8 and off.coef(li) == 128 and off.coef(self.lfb) == 1
                    and tuple(leaf.shape) == self.Ts + (self.C,) and leaf.dtype.itemsize in (4, 8)):
                rest = off.without(j).without(m).without(li).without(self.lfb)
                if rest.key() == Aff.of(Var("r", 1)).scale(self.C).key():
                    return f"{self._lds(leaf, li, m)}[{j.name}]", j.level
        return super().load_leaf(leaf, off)

    def _lds(self, leaf: Node, li: Var, m: Var) -> str:
        """The 8 staged elements (li, m, 0..7) of ``leaf`` in registers."""
        if leaf.id not in self.staged_ptr:
            self.staged_ptr[leaf.id] = len(self.staged)
            self.staged.append(leaf)
        k = self.staged_ptr[leaf.id]
        T = leaf.dtype.ctype
        key = ("lds", leaf.id, m.name, li.name)
        hit = self.memo_get(key)
        if hit is None:
            name = self.fresh("L")
            ls = 128 + 16 // leaf.dtype.itemsize
            self.stmt(m.level, f"{T} {name}[8];")
            self.stmt(m.level, f"gr::lds8<{T}>({name}, reinterpret_cast<const {T}*>(sst{k}) + "
                               f"(lf0 + {li.name}) * {ls} + 8 * {m.name});")
            hit = self.memo_put(key, (name, m.level))
        return hit[0]

    def _pair_map(self, n: Node, coords):
        from .codegen_coop import shared_div_pair
        v = shared_div_pair(self, n, coords)
        return v if v is not None else super()._pair_map(n, coords)

    # -- row-complete reductions -------------------------------------------------------
    def _row_complete(self, x: Node, axes) -> bool:
        return (tuple(x.shape[:len(self.Ts)]) == self.Ts and len(x.shape) == len(self.Ts) + 1
                and x.shape[-1] == self.C and tuple(axes) == (len(self.Ts),))

    def reduce(self, r: Node, coords):
        rop, axes, keepdims, odt = r.op.attrs
        if not self._row_complete(r.preds[0], axes):
            return super().reduce(r, coords)
        kept = [c for i, c in enumerate(coords) if i not in axes] if keepdims else list(coords)
        if any(c.level > 1 for c in kept):
            raise NotFusable(r, "row reduction consumed per column")
        rk = self.reduction_key(r, kept)
        hit = self.memo_get(rk)
        if hit is not None:
            return hit
        return self.memo_put(rk, (self.row_reduce(r.preds[0], rop, r.dtype, kept), 1))

    def row_reduce(self, x: Node, rop, T: DType, row_coords, identity=True, value_fn=None):
        """Reduce x over the row (NumPy order for float sums)."""
        if self.pair and rop is ReduceOp.sum and T is DType.f32 and x.dtype is DType.f32:
            return self._row_reduce_pair(x, T, row_coords, identity)
        ct = T.ctype
        lsum = self.fresh("ls")
        self.stmt(1, f"{ct} {lsum}[{self.lpl}];")
        acc = self.fresh("acc")
        L = self.open_elem(1)
        (li, sli, _), (m, sm, _), (j, sj, _) = L
        self.stmt(li.level, f"{ct} {acc}[8];")
        val = self.cast(self.value(x, list(row_coords) + [self.col(li, m, j)]), x.dtype, T)
        comb = _COMBINE[rop]
        self.stmt(j.level, f"{acc}[{j.name}] = ({m.name} == 0) ? {val[0]} : {comb}<{ct}>({acc}[{j.name}], {val[0]});")
        self.close(sj, L[2][2])
        self.close(sm, L[1][2])
        if rop is ReduceOp.sum and T.is_float:
            self.stmt(li.level, f"{lsum}[{li.name}] = gr::leaf_local<{ct}, 8>({acc});")
        else:
            self.stmt(li.level, f"{{ {ct} t = {acc}[0]; for (int q = 1; q < 8; ++q) t = {comb}<{ct}>(t, {acc}[q]); "
                                f"{lsum}[{li.name}] = t; }}")
        self.close(sli, L[0][2])
        op = _OPS[rop]
        s = self.emit(1, ct, f"gr::lane_tree<{op}, {ct}, {self.lpl}>({lsum})")
        s = self.emit(1, ct, f"gr::warp_tree<{op}, {ct}>({s}, {self.lpr})")
        if identity and rop is ReduceOp.sum and T.is_float:
            s = self.emit(1, ct, f"gr::add<{ct}>({c_literal(0, T)}, {s})")
        return s

    def _row_reduce_pair(self, x: Node, T: DType, row_coords, identity):
        """Float row sum with element pairs: NumPy's eight leaf accumulators
        as four gr::f2 (FADD2), unpacked for the leaf combine."""
        lsum = self.fresh("ls")
        self.stmt(1, f"float {lsum}[{self.lpl}];")
        acc = self.fresh("acc")
        li, sli, a = self.open(1, "for", trip=self.lpl, unroll=True)
        sli.coop = "li"
        m, sm, b = self.open(li.level, "for", trip=16, unroll=True)
        sm.coop = "m"
        jp, sj, c = self.open(m.level, "for", trip=4, unroll=True)
        sj.coop = "jp"
        self.stmt(li.level, f"gr::f2 {acc}[4];")
        self.half = Var("gr_half_" + jp.name, jp.level)
        try:
            col = Aff.of(self.lfb) + Aff.of(li).scale(128) + Aff.of(m).scale(8) + Aff.of(jp).scale(2) + Aff.of(self.half)
            val = self.value(x, list(row_coords) + [col])
            pv = self.splat(val)
            self.stmt(jp.level, f"{acc}[{jp.name}] = ({m.name} == 0) ? {pv} : gr::p2::add({acc}[{jp.name}], {pv});")
        finally:
            self.half = None
        self.close(sj, c)
        self.close(sm, b)
        self.stmt(li.level, f"{{ float a8[8]; for (int q = 0; q < 4; ++q) {{ a8[2 * q] = gr::lo({acc}[q]); "
                            f"a8[2 * q + 1] = gr::hi({acc}[q]); }} {lsum}[{li.name}] = gr::leaf_local<float, 8>(a8); }}")
        self.close(sli, a)
        s = self.emit(1, "float", f"gr::lane_tree<gr::OpSum, float, {self.lpl}>({lsum})")
        s = self.emit(1, "float", f"gr::warp_tree<gr::OpSum, float>({s}, {self.lpr})")
        if identity:
            s = self.emit(1, "float", f"gr::add<float>({c_literal(0, T)}, {s})")
        return s

    def argreduce(self, r: Node, coords):
        which, axis, keepdims = r.op.attrs
        x = r.preds[0]
        if axis is None or not self._row_complete(x, (axis,)):
            return super().argreduce(r, coords)
        kept = [c for i, c in enumerate(coords) if i != axis] if keepdims else list(coords)
        if any(c.level > 1 for c in kept):
            raise NotFusable(r, "row arg-reduction consumed per column")
        T = x.dtype.ctype
        best, bi = self.fresh("bv"), self.fresh("bi")
        self.stmt(1, f"{T} {best} = 0; long long {bi} = -1;")
        L = self.open_elem(1)
        (li, _, _), (m, _, _), (j, _, _) = L
        col = self.col(li, m, j)
        val = self.value(x, list(kept) + [col])
        mx = "true" if which == "max" else "false"
        self.stmt(j.level, f"{{ const long long ci = {col.c()}; if ({bi} < 0 || gr::arg_take_b<{mx}, {T}>({best}, {bi}, {val[0]}, ci)) "
                           f"{{ {best} = {val[0]}; {bi} = ci; }} }}")
        self.close_elem(L)
        return self.emit(1, "long long", f"gr::warp_arg<{mx}, {T}>({best}, {bi}, {self.lpr})"), 1


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
    if C is None or C < 128 or not _regular(C):
        return None
    for r in region.roots:
        x = r.preds[0] if r.id in tot_ids else r
        if tuple(x.shape) != Ts + (C,) and not (tuple(x.shape[:len(Ts)]) == Ts and element_count(x.shape[len(Ts):]) == 1):
            return None
    for l in region.leaves:
        if tuple(l.shape) == Ts + (C,) and l.dtype.itemsize not in (4, 8):
            return None
    return Ts, totals, C


def _params_with(region):
    return _params_struct(region).replace("    void* __restrict__ scratch;",
                                          "    void* __restrict__ scratch;\n    unsigned int* ticket;")


WROW_PAIR = os.environ.get("GRUMPY_WROW_PAIR", "1") == "1"


def try_generate(region: Region, kname="gr_region") -> Optional[KernelSource]:
    if WROW_PAIR:
        try:
            return _try_generate(region, kname, pair=True)
        except NotPairable:
            pass
    return _try_generate(region, kname, pair=False)


def _try_generate(region: Region, kname="gr_region", pair=False) -> Optional[KernelSource]:
    q = _qualifies(region)
    if q is None:
        return None
    Ts, totals, C = q
    tot_ids = {t.id for t in totals}
    nleaf = C // 128
    lpr = min(32, nleaf)
    lpl = nleaf // lpr
    rpw = 32 // lpr
    R = element_count(Ts)
    em = WrowEmitter(region, Ts, C, lpr, lpl, rpw)
    # two-pass division by row-level divisors: the fast pass tracks the
    # dividends' range; a warp whose rows left the exact window redoes its
    # rows from the stage it still holds (no flags, no second launch)
    em.div_fast = WROW_DIV_TWO_PASS and lpr == 32
    em.pair = pair and lpr == 32
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
            accs = []
            for t in fused_tot.get(r.id, []):
                accs.append((t, em.fresh("tacc"), em.fresh("tls")))
                em.stmt(1, f"{t.dtype.ctype} {accs[-1][2]}[{lpl}];")
            L = em.open_elem(1)
            (li, sli, _), (m, sm, _), (j, sj, _) = L
            for t, a, ls in accs:
                em.stmt(li.level, f"{t.dtype.ctype} {a}[8];")
            o = em.fresh("O")
            em.stmt(m.level, f"{T} {o}[8];")
            val = em.value(r, row_coords + [em.col(li, m, j)])
            em.stmt(j.level, f"{o}[{j.name}] = {val[0]};")
            for t, a, ls in accs:
                tv = em.cast(val, r.dtype, t.dtype)
                comb = _COMBINE[t.op.attrs[0]]
                em.stmt(j.level, f"{a}[{j.name}] = ({m.name} == 0) ? {tv[0]} : {comb}<{t.dtype.ctype}>({a}[{j.name}], {tv[0]});")
            em.close(sj, L[2][2])
            em.stmt(m.level, f"if (valid) gr::st8<{T}>(p.out{ri} + r * {C}LL + lfb + 128 * {li.name} + 8 * {m.name}, {o});")
            em.close(sm, L[1][2])
            for t, a, ls in accs:
                rop = t.op.attrs[0]
                ct = t.dtype.ctype
                if rop is ReduceOp.sum and t.dtype.is_float:
                    em.stmt(li.level, f"{ls}[{li.name}] = gr::leaf_local<{ct}, 8>({a});")
                else:
                    cb = _COMBINE[rop]
                    em.stmt(li.level, f"{{ {ct} tt = {a}[0]; for (int q = 1; q < 8; ++q) tt = {cb}<{ct}>(tt, {a}[q]); {ls}[{li.name}] = tt; }}")
            em.close(sli, L[0][2])
            for t, a, ls in accs:
                op = _OPS[t.op.attrs[0]]
                ct = t.dtype.ctype
                s = em.emit(1, ct, f"gr::lane_tree<{op}, {ct}, {lpl}>({ls})")
                tot_partials[t.id] = em.emit(1, ct, f"gr::warp_tree<{op}, {ct}>({s}, {lpr})")
        else:
            val = em.value(r, row_coords + [Aff.of(0)] * (len(r.shape) - len(Ts)))
            em.stmt(1, f"if (valid && lr == 0) gr::st<{T}>(p.out{ri} + r, {val[0]});")

    scratch_off = 0
    tot_meta = []
    for ri, r in enumerate(region.roots):
        if r.id not in tot_ids:
            continue
        x = r.preds[0]
        if r.kind is OpKind.ARGREDUCE:
            raise NotFusable(r, "argmax over all axes with streamed rows")
        rop = r.op.attrs[0]
        T = r.dtype
        ct = T.ctype
        if r.id in tot_partials:
            part = tot_partials[r.id]
        elif tuple(x.shape) == Ts + (C,):
            part = em.row_reduce(x, rop, T, row_coords, identity=False)
        else:
            part = em.cast(em.value(x, row_coords + [Aff.of(0)] * (len(x.shape) - len(Ts))), x.dtype, T)[0]
        off = scratch_off
        em.stmt(1, f"if (valid && lr == 0) reinterpret_cast<{ct}*>(static_cast<char*>(p.scratch) + {off})[r] = {part};")
        tot_meta.append((ri, rop, T, off))
        scratch_off += ((R * T.itemsize + 255) // 256) * 256

    # ---- shared-memory ring geometry
    staged = em.staged
    leaf_bytes = [128 * l.dtype.itemsize + 16 for l in staged]
    row_bytes = sum(nleaf * b for b in leaf_bytes)
    slot_bytes = rpw * row_bytes                      # one stage of one warp
    if slot_bytes == 0:
        return None
    best = None
    for W in (8, 6, 4, 2, 1):
        for NS in (3, 2):
            if W * NS * slot_bytes <= SMEM_BUDGET:
                cand = (W * (NS - 1), W, NS)
                if best is None or cand > best:
                    best = cand
    if best is None:
        return None
    _, W, NS = best
    if os.environ.get("GRUMPY_WROW_WNS"):       # experiments: "W,NS"
        W, NS = (int(v) for v in os.environ["GRUMPY_WROW_WNS"].split(","))
    smem = W * NS * slot_bytes

    # stage pointers for the staged leaves, per row of this lane
    ptr_lines = []
    off = 0
    for k, l in enumerate(staged):
        ptr_lines.append(f"  const unsigned char* sst{k} = stage + {off} + (long long)q * {nleaf * leaf_bytes[k]};")
        off += rpw * nleaf * leaf_bytes[k]

    two_pass = em.used_div_fast
    lines = [("template <bool FAST> static __device__ __forceinline__ bool" if two_pass else
              "static __device__ __forceinline__ void") +
             " rows(const Params& p, const unsigned char* stage, const long long g, const int lane) {",
             f"  const int q = lane / {lpr};",
             f"  const int lr = lane % {lpr};",
             f"  const long long r0 = g * {rpw} + q;",
             "  const bool valid = r0 < NROWS;",
             "  const long long r = valid ? r0 : NROWS - 1;",
             f"  const int lf0 = lr * {lpl};",
             "  const long long lfb = (long long)lf0 * 128;"]
    lines += ptr_lines
    if two_pass:
        lines.append("  bool bad = false;")
    lines += ["  " + c for c in em.consts]
    lines += render(em.row, 1)
    if two_pass:
        lines += ["  " + l for l in em.div_finalize]
        lines.append("  return bad;")
    lines.append("}")

    # bulk-copy issue for one row group: copies spread over the 32 lanes
    issue = ["static __device__ __forceinline__ void issue(const Params& p, unsigned char* stage, unsigned long long* bar, const long long g, const int lane) {",
             f"  const long long nvalid = (g * {rpw} + {rpw} <= NROWS) ? {rpw} : (NROWS - g * {rpw});",
             f"  if (lane == 0) gr::mbar_arrive_expect_tx(bar, (unsigned)(nvalid * {sum(nleaf * 128 * l.dtype.itemsize for l in staged)}));"]
    off = 0
    for k, l in enumerate(staged):
        T = l.dtype.ctype
        idx = region.leaves.index(l)
        lb = leaf_bytes[k]
        issue.append(f"  for (int c = lane; c < {rpw * nleaf}; c += 32) {{")
        issue.append(f"    const int qq = c / {nleaf}, lf = c % {nleaf};")
        issue.append(f"    if (qq < nvalid) gr::bulk_g2s(stage + {off} + (long long)qq * {nleaf * lb} + (long long)lf * {lb}, "
                     f"p.in{idx} + (g * {rpw} + qq) * {C}LL + (long long)lf * 128, {128 * l.dtype.itemsize}u, bar);")
        issue.append("  }")
        off += rpw * nleaf * lb
    issue.append("}")

    src = [HEADER, '#include "gr_reduce.cuh"\n#include "gr_tma.cuh"\n', "struct K {", _params_with(region),
           f"  static constexpr long long NROWS = {R}LL;"]
    src.append("  " + "\n  ".join(lines))
    src.append("  " + "\n  ".join(issue))
    src.append("};")
    ngroups = -(-R // rpw)
    kern = [f'extern "C" __global__ void __launch_bounds__({W * 32}) {kname}(const K::Params p) {{',
            "  extern __shared__ __align__(128) unsigned char smem[];",
            f"  __shared__ unsigned long long bars[{W * NS}];",
            "  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;",
            f"  if (lane == 0) {{ for (int s = 0; s < {NS}; ++s) gr::mbar_init(&bars[warp * {NS} + s], 1); gr::fence_mbar_init(); }}",
            "  __syncwarp();",
            f"  const long long gw = (long long)blockIdx.x * {W} + warp, nwg = (long long)gridDim.x * {W};",
            f"  const long long NG = {ngroups}LL;",
            f"  unsigned char* wbase = smem + (long long)warp * {NS * slot_bytes};",
            f"  for (int s = 0; s < {NS - 1}; ++s) {{ const long long g = gw + s * nwg; if (g < NG) K::issue(p, wbase + s * {slot_bytes}, &bars[warp * {NS} + s], g, lane); }}",
            "  int it = 0;",
            "  for (long long g = gw; g < NG; g += nwg, ++it) {",
            f"    const int s = it % {NS};",
            "    {",
            f"      const long long gn = g + {NS - 1} * nwg;",
            f"      const int sn = (it + {NS - 1}) % {NS};",
            "      __syncwarp();",
            "      gr::fence_proxy_async();",
            f"      if (gn < NG) K::issue(p, wbase + sn * {slot_bytes}, &bars[warp * {NS} + sn], gn, lane);",
            "    }",
            f"    gr::mbar_wait(&bars[warp * {NS} + s], (unsigned)((it / {NS}) & 1));",
            (f"    if (__any_sync(0xffffffffu, K::rows<true>(p, wbase + s * {slot_bytes}, g, lane))) "
             f"K::rows<false>(p, wbase + s * {slot_bytes}, g, lane);" if two_pass else
             f"    K::rows(p, wbase + s * {slot_bytes}, g, lane);"),
            "  }"]
    if tot_meta:
        kern.append("  if (gr::last_block(p.ticket)) {")
        for ri, rop, T, off_ in tot_meta:
            ct = T.ctype
            ident = c_literal(_IDENT[rop](T), T)
            kern.append(f"    const {ct} v{ri} = gr::block_tree<{_OPS[rop]}, {ct}>("
                        f"reinterpret_cast<const {ct}*>(static_cast<const char*>(p.scratch) + {off_}), K::NROWS, {ident});")
            fin = f"gr::add<{ct}>({c_literal(0, T)}, v{ri})" if rop is ReduceOp.sum else f"v{ri}"
            kern.append(f"    if (threadIdx.x == 0) p.out{ri}[0] = {fin};")
        kern.append("  }")
    kern.append("}")
    src += kern
    return KernelSource("wrow", "\n".join(src) + "\n", kname,
                        leaf_slots=list(range(len(region.leaves))),
                        root_slots=list(range(len(region.roots))),
                        block=W * 32, groups=ngroups * W * 32 // W, vec=1, unroll=1, scratch_bytes=scratch_off,
                        meta={"rows": R, "row_shape": Ts, "cols": C, "lanes_per_row": lpr, "rows_per_warp": rpw,
                              "warps": W, "stages": NS, "smem": smem, "totals": len(tot_meta),
                              "ticket": bool(tot_meta), "persistent": True, "label": "wrow"})
