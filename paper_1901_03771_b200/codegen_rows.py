"""Row family: fused regions that contain reductions (K2 / K3 / K4 / K5).

Reference: run_map_reduce (per-thread fold
from the identity, partials folded in a fixed order), arg-reductions as
"reduce + select" and the paper's GPU reduction with a
separate final kernel.  The B200 design replaces the
"cut at every reduction" of Algorithm 1 with loop nests:

* the region's *thread space* T is the leading shape every reduction keeps
  (rows); one thread owns one row and evaluates the whole region for it;
* a reduction is evaluated where its kept coordinates live — values depending
  only on the row are computed once per row and reused by every element of the
  row (mean/std broadcast back in row-normalise, max/sum in softmax);
* float sums follow NumPy's association exactly (``gr::pairwise`` along the
  contiguous axis, sequential along the others, identity-initialised), so
  reductions of IEEE-exact terms are bit-identical to the oracle; arg-
  reductions keep the first index and treat NaN as extreme like np.argmax;
* full reductions of the region ("totals", e.g. ``y.sum()``) are accumulated
  as one partial per row and folded by the last CTA to finish (atomic ticket,
  no float atomics) in a fixed tree: one launch, deterministic.

The cooperative variant for long rows (one CTA per row, row staged in
registers) lives in ``codegen_coop.py``.
"""

from __future__ import annotations

import os
import re
from typing import Dict, List, Optional, Sequence, Tuple

from .codegen import (
    _PAIR_BIN, _PAIR_UN, HEADER, Aff, KernelSource, NotPairable, Region, ValueEmitter, Var, _params_struct,
    bcast_coords, c_literal,
)
from .dag import ElemCode, Node, OpKind, ReduceOp
from .errors import UnsupportedNodeInFusedStep
from .tensor import DType, element_count, row_major_strides


class NotFusable(UnsupportedNodeInFusedStep):
    """Raised when ``node`` cannot live inside this region; the planner cuts it."""

    def __init__(self, node: Node, why: str):
        super().__init__(f"node {node.id} ({node.op!r}) not fusable here: {why}")
        self.node = node


# Certified nearest-centre argmin (gr_nearest.cuh): argmin_j sum_k (u_k - C[j,k])^2
# over a constant-bank centre table ranks the centres by an expanded key (four
# FFMA2 per centre pair instead of 4 sub + 4 mul + 3 add per centre) and runs
# the exact NumPy-order scan only for rows whose label the key's error bound
# cannot certify.  Labels are np.argmin's in every case.
NEAREST = os.environ.get("GRUMPY_NEAREST", "1") == "1"
NEAREST_MAX_D = 8
# CTAs per SM asked of ptxas (__launch_bounds__ min blocks) for row kernels
# with a nearest-centre search (0: none).  With the exact fallback scan out
# of line (gr::nearest_exact, __noinline__) the k-means kernel needs 32
# registers and runs at full occupancy uncapped.
NEAREST_MIN_BLOCKS = int(os.environ.get("GRUMPY_NEAREST_MINB", "0"))
# (experiment, off) the kernel's row loop takes two rows per step and
# searches both rows' centres together (gr::nearest_centre_n<.., 2>): 444
# instead of 496 hot-loop instructions per point, but 40 registers and the
# row body's own reload of the point: 1.636 vs 1.601 ms on k-means 2^26 x 64
NEAREST_PAIR_ROWS = os.environ.get("GRUMPY_NEAREST_PAIR", "0") == "1"
NEAREST_MAX_K = 256


def match_nearest(x: Node, axes):
    """(u, centre leaf, K, D) when ``x`` is ((u - c) ** 2).sum(-1) with u of
    shape (N, 1, D) and c a (1, K, D) / (K, D) view of an f32 leaf, reduced
    over axis 1 of x's (N, K); else None."""
    if (x.kind is not OpKind.REDUCE or x.dtype is not DType.f32 or len(x.shape) != 2 or tuple(axes) != (1,)):
        return None
    rop, raxes, keepdims, _odt = x.op.attrs
    s = x.preds[0]
    if rop is not ReduceOp.sum or keepdims or tuple(raxes) != (2,) or len(s.shape) != 3:
        return None
    N, K, D = s.shape
    if not (2 <= K <= NEAREST_MAX_K and K % 2 == 0 and 1 <= D <= NEAREST_MAX_D):
        return None
    if s.kind is not OpKind.MAP or s.dtype is not DType.f32 or s.loop[0] is not DType.f32:
        return None
    if s.op.code is ElemCode.square:
        d = s.preds[0]
    elif s.op.code is ElemCode.mul and s.preds[0].id == s.preds[1].id:
        d = s.preds[0]
    else:
        return None
    if (d.kind is not OpKind.MAP or d.op.code is not ElemCode.sub or d.dtype is not DType.f32
            or tuple(d.loop) != (DType.f32, DType.f32)):
        return None
    for u, c in (d.preds, d.preds[::-1]):
        if tuple(u.shape) != (N, 1, D) or tuple(c.shape) not in ((1, K, D), (K, D)):
            continue
        while c.kind is OpKind.RESHAPE and not c.is_materialized:
            c = c.preds[0]
        if c.dtype is DType.f32 and tuple(c.shape) in ((K, D), (1, K, D)) and c.is_materialized:
            return u, c, K, D
    return None


def is_total(n: Node) -> bool:
    """A reduction to a single value (all axes), e.g. y.sum() or argmax(axis=None)."""
    if n.kind is OpKind.REDUCE:
        return len(n.op.attrs[1]) == len(n.preds[0].shape) if n.preds else element_count(n.shape) == 1
    if n.kind is OpKind.ARGREDUCE:
        return n.op.attrs[1] is None
    return False


_IDENT = {
    ReduceOp.sum: lambda dt: 0,
    ReduceOp.prod: lambda dt: 1,
    ReduceOp.max: lambda dt: float("-inf") if dt.is_float else (False if dt.is_bool else (-(2**31) if dt is DType.i32 else -(2**63))),
    ReduceOp.min: lambda dt: float("inf") if dt.is_float else (True if dt.is_bool else (2**31 - 1 if dt is DType.i32 else 2**63 - 1)),
}
_COMBINE = {ReduceOp.sum: "gr::add", ReduceOp.prod: "gr::mul", ReduceOp.max: "gr::maximum", ReduceOp.min: "gr::minimum"}
_OPS = {ReduceOp.sum: "gr::OpSum", ReduceOp.prod: "gr::OpProd", ReduceOp.max: "gr::OpMax", ReduceOp.min: "gr::OpMin"}

ARG_UNROLL = 64        # arg-reductions up to this length are fully unrolled
SMALL_RECOMPUTE = 64   # a reduction re-evaluated per column may reduce at most this many points
MAX_GRID = int(os.environ.get("GRUMPY_KEYED_MAX_GRID", str(148 * 16)))  # grid cap for kernels with per-CTA partial slots (keyed sums)
KEYED_GROUP = 32       # CTAs per first-level fold of the keyed-sum partials (tickets: 1 + MAX_GRID / 32 words)


# Skinny products z = A @ B (A [R, K] streamed, B [K, N] small) computed as
# the first stage of their consumers' row kernel (gr_skinny.cuh) instead of a
# cuBLAS call whose output the consumers read back (C4 layer 2 + softmax).
SKINNY = os.environ.get("GRUMPY_SKINNY", "1") == "1"
SKINNY_MAX_N = 16
SKINNY_MIN_ROWS = 4096
# "<B placement>,<threads per CTA>,<rows per thread>,<stages>".  MLP layer 2
# (65536 x 1024 @ 1024 x 10 + softmax + argmax, tools/skinny_sweep.sh):
# cbank,64,1,3 102 us (LDCU latency: 71% short-scoreboard stalls); cbank
# 64,2,3 97; smem,64,2,3 78; smem,128,1,3 76; smem,64,4,2 65; smem,128,2,2
# 58.5 us (256-row boxes, 2 CTAs/SM) — against cuBLAS SIMT 111 + R2 9 us.
_SK = os.environ.get("GRUMPY_SKINNY_CFG", "smem,128,2,2").split(",")
SKINNY_B = _SK[0]          # B's k-pairs: "cbank" (64-bit uniform operands) or "smem" (broadcast LDS)
SKINNY_BLOCK = int(_SK[1])  # threads per CTA
SKINNY_RT = int(_SK[2])    # rows per thread (each B operand feeds RT rows)
SKINNY_STAGES = int(_SK[3])  # TMA boxes in flight per CTA
SKINNY_CBANK_BYTES = 48 * 1024


def skinny_ok(n: Node) -> bool:
    """Planner hook: may the product ``n`` be the in-kernel prologue of its
    consumers' row region (rather than a library step)?"""
    if not SKINNY or n.kind is not OpKind.MATMUL or len(n.preds) != 2:
        return False
    a, b = n.preds
    if a.dtype is not DType.f32 or b.dtype is not DType.f32 or len(a.shape) != 2 or len(b.shape) != 2:
        return False
    if any(p.kind is OpKind.TRANSPOSE and not p.is_materialized for p in (a, b)):
        return False                      # transposed operands keep the library's trans flags
    R, K = a.shape
    N = b.shape[1]
    return (R >= SKINNY_MIN_ROWS and K >= 32 and K % 32 == 0 and 0 < N <= SKINNY_MAX_N
            and K * N * 4 <= SKINNY_CBANK_BYTES and R < 2 ** 31)


def _skinny_nodes(region: Region) -> List[Node]:
    return [n for n in region.nodes if n.kind is OpKind.MATMUL and n.id not in region.leaf_ids]


class CBankMiss(Exception):
    """A leaf staged in constant memory is read at a row-dependent offset."""

    def __init__(self, leaf: Node):
        super().__init__(f"leaf {leaf.id} read per row")
        self.leaf = leaf


# Row kernels whose rows are short contiguous slices of a leaf prefetch the
# next grid-stride row of that leaf into L1 before evaluating the current one
# (hides the load latency at the low occupancy of register-heavy row bodies)
ROW_PREFETCH = os.environ.get("GRUMPY_ROW_PREFETCH", "1") == "1"
ROW_PREFETCH_MAX_BYTES = 128
# bincount keys are matched as 32-bit words (keys outside every histogram map
# to one ignored word): MATCH.ANY on 32 bits instead of 64
MATCH32 = os.environ.get("GRUMPY_MATCH32", "1") == "1"

CBANK_LEAF_BYTES = 16 * 1024   # per leaf
CBANK_TOTAL_BYTES = 48 * 1024  # per kernel (the user constant bank is 64 KB)
CBANK_MIN_ROWS = 4096          # staging pays only when many rows reuse the leaf


def cbank_candidates(region: Region, rows: int) -> Dict[int, str]:
    """Small leaves that may be staged in the constant bank (leaf id -> symbol)."""
    if rows < CBANK_MIN_ROWS:
        return {}
    out, total = {}, 0
    for i, l in enumerate(region.leaves):
        nb = element_count(l.shape) * l.dtype.itemsize
        if 0 < nb <= CBANK_LEAF_BYTES and total + nb <= CBANK_TOTAL_BYTES and l.dtype.itemsize in (4, 8):
            out[l.id] = f"gr_cin{i}"
            total += nb
    return out


class Scope:
    __slots__ = ("level", "kind", "header", "lines", "ret", "unroll", "var", "trip", "coop")

    def __init__(self, level, kind="block", header="", unroll=False, var=None, trip=None):
        self.coop = False
        self.level = level
        self.kind = kind
        self.header = header
        self.lines: list = []
        self.ret = None
        self.unroll = unroll
        self.var = var
        self.trip = trip


def render(scope: Scope, indent: int) -> List[str]:
    pad = "  " * indent
    out = []
    for l in scope.lines:
        if isinstance(l, Scope):
            if l.kind == "for":
                if l.unroll:
                    out.append("#pragma unroll")
                out.append(f"{pad}{l.header} {{")
                out += render(l, indent + 1)
                out.append(f"{pad}}}")
            elif l.kind == "lambda":
                out.append(f"{pad}{l.header} {{")
                out += render(l, indent + 1)
                out.append(f"{pad}  return {l.ret};")
                out.append(f"{pad}}};")
            else:
                out.append(f"{pad}{{")
                out += render(l, indent + 1)
                out.append(f"{pad}}}")
        else:
            out.append(pad + l)
    return out


class LoopEmitter(ValueEmitter):
    """Scoped emitter: level 0 kernel constants, level 1 the row, 2+ loops."""

    def __init__(self, region: Region, vec_loads=True, cbank=None):
        super().__init__(region)
        self.row = Scope(1)
        self.stack: List[Optional[Scope]] = [None, self.row]
        self.vec_loads = vec_loads
        # leaf id -> __constant__ symbol for small leaves every row reads at
        # the same (row-independent) offsets, e.g. the k-means centroids
        self.cbank: Dict[int, str] = dict(cbank or {})
        self.cbank_pair: Dict[int, int] = {}   # leaf id -> pair stride of its pair-adjacent copy
        self.uniform_vars = set()   # loop indices with row-independent values
        # loop pairing: an unrolled f32 arg-reduction loop walks index PAIRS
        # (2i, 2i+1); values that depend on the logical index (2*iv + half)
        # are gr::f2 and run as FADD2/FMUL2/FFMA2 (gr_pair.cuh)
        self.pair_loops = False
        self.half: Optional[Var] = None
        self.pairs = set()            # emitted names holding a gr::f2
        # skinny product computed by the tile prologue: (canonical id, row key)
        self.skinny: Optional[tuple] = None
        # centre leaf id -> (K, D, table symbol) of certified nearest-centre searches
        self.nearest: Dict[int, tuple] = {}
        # two rows per nearest-centre search, done by the kernel loop
        self.nn_rows2 = False
        self.nn_pair: Optional[tuple] = None   # (row operand, K, D, table symbol, centre symbol)

    # -- scopes ------------------------------------------------------------------
    def emit(self, level, ctype, expr):
        name = self.fresh()
        if level <= 0:
            self.consts.append(f"const {ctype} {name} = {expr};")
            return name
        self.stack[level].lines.append(f"const {ctype} {name} = {expr};")
        return name

    def stmt(self, level, text):
        if level <= 0:
            self.consts.append(text)
        else:
            self.stack[level].lines.append(text)

    def var_decl(self, level, ctype, init) -> str:
        name = self.fresh("a")
        self.stmt(level, f"{ctype} {name} = {init};")
        return name

    def open(self, parent_level, kind, trip=None, unroll=False, ret_type=None):
        saved = self.stack[parent_level + 1:]
        del self.stack[parent_level + 1:]
        lvl = parent_level + 1
        name = self.fresh("i")
        var = Var(name, lvl)
        if kind == "for":
            tstr = f"{trip}LL" if isinstance(trip, int) else trip
            header = f"for (long long {name} = 0; {name} < {tstr}; ++{name})"
        else:
            header = f"auto f{name} = [&](long long {name}) -> {ret_type}"
        if kind != "for" or isinstance(trip, int):
            self.uniform_vars.add(name)
        s = Scope(lvl, kind, header, unroll=unroll, var=var, trip=trip)
        self.stack.append(s)
        return var, s, saved

    def close(self, s: Scope, saved, ret=None):
        assert self.stack[-1] is s
        self.stack.pop()
        s.ret = ret
        self.stack[-1].lines.append(s)
        self.stack.extend(saved)

    def value(self, n: Node, coords):
        key = (self.cid(n), tuple(c.key() for c in coords))
        hit = self.memo.get(key)
        if hit is not None:
            expr, lvl, sc = hit
            if lvl == 0 or (lvl < len(self.stack) and self.stack[lvl] is sc):
                return expr, lvl
        v = self._value(n, list(coords))
        self.memo[key] = (v[0], v[1], self.stack[v[1]] if 0 < v[1] < len(self.stack) else None)
        return v

    def derived_var(self, level, expr) -> Var:
        name = self.emit(level, "long long", expr)
        return Var(name, level)

    def memo_get(self, key):
        hit = self.memo.get(key)
        if hit is not None:
            expr, lvl, sc = hit
            if lvl == 0 or (lvl < len(self.stack) and self.stack[lvl] is sc):
                return expr, lvl
        return None

    def memo_put(self, key, v):
        self.memo[key] = (v[0], v[1], self.stack[v[1]] if 0 < v[1] < len(self.stack) else None)
        return v

    def reduction_key(self, r: Node, kept) -> tuple:
        """keepdims-independent identity of a reduction value: the same fold of
        the same operand at the same kept coordinates."""
        a = r.op.attrs
        return ("red", r.kind, self.cid(r.preds[0]), a[0], a[1], r.dtype, tuple(k.key() for k in kept))

    # -- loads ----------------------------------------------------------------------
    def load_leaf(self, leaf: Node, off: Aff):
        idx = self.leaf_index[leaf.id]
        T = leaf.dtype.ctype
        ptr = f"p.in{idx}"
        lvl = off.level
        sym = self.cbank.get(leaf.id)
        if self.half is not None and off.coef(self.half):
            # the two logical indices of a paired loop
            if leaf.dtype is not DType.f32:
                raise NotPairable("non-f32 leaf in a paired loop")
            lo = off.without(self.half)
            hi = lo + off.coef(self.half)
            if sym is not None:
                if any(v.name not in self.uniform_vars for v, _ in lo.terms):
                    raise CBankMiss(leaf)
                B = off.coef(self.half)
                n = element_count(leaf.shape)
                if B > 0 and n % (2 * B) == 0 and self.cbank_pair.get(leaf.id, B) == B:
                    # pair-adjacent copy of the leaf: (x[lo], x[lo+B]) is one
                    # 64-bit constant -> a uniform-register pair operand
                    self.cbank_pair[leaf.id] = B
                    psym = sym + "_p"
                    expr = (f"((({lo.c()}) / {B}) % 2 == 0 ? gr::f2{{{psym}[(({lo.c()}) / {2 * B}) * {B} + (({lo.c()}) % {B})]}} "
                            f": gr::pk({sym}[{lo.c()}], {sym}[{hi.c()}]))")
                    return self.emit_pair(lvl, expr), lvl
                raise NotPairable("constant-bank leaf without a pair-adjacent copy")
            else:
                # gathered pairs of a row-invariant leaf get hoisted out of the
                # row loop by ptxas (254 registers, 4.14 vs 3.25 ms for k-means)
                raise NotPairable("paired operand outside the constant bank")
            return self.emit_pair(lvl, f"gr::pk({a}, {b})"), lvl
        if sym is not None:
            if any(v.name not in self.uniform_vars for v, _ in off.terms):
                raise CBankMiss(leaf)
            # warp-uniform address: a constant-bank operand (LDCU / c[3][]),
            # no per-thread load instruction
            return self.emit(lvl, T, f"{sym}[{off.c()}]"), lvl
        if self.vec_loads and lvl >= 2:
            sc = self.stack[lvl]
            if sc.kind == "for" and sc.unroll and sc.var is not None:
                cv = off.coef(sc.var)
                rest = off.without(sc.var)
                trip = sc.trip
                nbytes = trip * leaf.dtype.itemsize
                if (cv == 1 and rest.level < lvl and trip in (2, 4, 8, 16) and nbytes in (2, 4, 8, 16)
                        and rest.alignment() % trip == 0):
                    key = ("vec", leaf.id, rest.key(), trip)
                    hit = self.memo.get(key)
                    if hit is not None and (hit[1] == 0 or self.stack[hit[1]] is hit[2]):
                        return f"{hit[0]}[{sc.var.name}]", lvl
                    name = self.fresh("L")
                    plvl = max(rest.level, 1)
                    self.stmt(plvl, f"{T} {name}[{trip}];")
                    self.stmt(plvl, f"gr::ldv<{T}, {trip}>({name}, {ptr} + {rest.c()});")
                    self.memo[key] = (name, plvl, self.stack[plvl] if plvl > 0 else None)
                    return f"{name}[{sc.var.name}]", lvl
        # a scalar read covered by a vector load already issued in scope
        # (k-means: the bincount weights P[r, d] after the row's P[r, :] load)
        for trip in (16, 8, 4, 2):
            for j in range(trip):
                rest = off + Aff.of(-j)
                if rest.const % trip or rest.alignment() % trip:
                    continue
                hit = self.memo.get(("vec", leaf.id, rest.key(), trip))
                if hit is not None and (hit[1] == 0 or (hit[1] < len(self.stack) and self.stack[hit[1]] is hit[2])):
                    return f"{hit[0]}[{j}]", max(lvl, hit[1])
        return self.emit(lvl, T, f"gr::ld<{T}>({ptr} + {off.c()})"), lvl

    # -- reductions -------------------------------------------------------------------
    def _value(self, n: Node, coords):
        if n.id not in self.leaf_index:
            if n.kind is OpKind.MATMUL:
                return self.skinny_value(n, coords)
            if n.kind is OpKind.REDUCE:
                return self.reduce(n, coords)
            if n.kind is OpKind.ARGREDUCE:
                return self.argreduce(n, coords)
            if (self.half is not None and n.kind is OpKind.MAP and n.op.code is not ElemCode.const_splat
                    and any(c.coef(self.half) for c in coords)):
                return self._pair_map(n, coords)
        return super()._value(n, coords)

    def skinny_value(self, n: Node, coords):
        """z[row, j] of the region's skinny product: register zk[j] filled by
        the CTA's tile prologue (gr::Skinny) before the row body runs."""
        if self.skinny is None or self.cid(n) != self.skinny[0]:
            raise NotFusable(n, "one skinny product per row region")
        if coords[0].key() != self.skinny[1]:
            raise NotFusable(n, "skinny product read at another row")
        col = coords[1]
        if self.half is not None and col.coef(self.half):
            raise NotPairable("skinny product read in a paired loop")
        return f"zk[{col.c()}]", max(col.level, 1)

    # -- paired loops ---------------------------------------------------------------
    def emit_pair(self, level, expr) -> str:
        name = self.emit(level, "gr::f2", expr)
        self.pairs.add(name)
        return name

    def is_pair(self, val) -> bool:
        return val[0] in self.pairs

    def splat(self, val) -> str:
        return val[0] if self.is_pair(val) else f"gr::splat({val[0]})"

    def cast(self, val, frm: DType, to: DType):
        if frm is not to and self.is_pair(val):
            raise NotPairable("cast of a paired value")
        return super().cast(val, frm, to)

    def _pair_map(self, n: Node, coords):
        code = n.op.code
        args = []
        for p, lt in zip(n.preds, n.loop):
            v = self.value(p, bcast_coords(coords, n.shape, p.shape))
            args.append(self.cast(v, p.dtype, lt))
        lvl = max(a[1] for a in args)
        if not any(self.is_pair(a) for a in args):
            return super()._value(n, coords)
        if n.dtype is not DType.f32 or any(lt is not DType.f32 for lt in n.loop):
            raise NotPairable(f"{code} on {n.loop}")
        names = [self.splat(a) for a in args]
        if code in (ElemCode.mul, ElemCode.square) and self._feeds_add(n):
            fn = "gr::p2::mul_nc" if code is ElemCode.mul else "gr::p2::square_nc"
            return self.emit_pair(lvl, f"{fn}({', '.join(names)})"), lvl
        if code in (ElemCode.add, ElemCode.sub, ElemCode.mul, ElemCode.div, ElemCode.maximum, ElemCode.minimum):
            return self.emit_pair(lvl, f"{_PAIR_BIN[code]}({names[0]}, {names[1]})"), lvl
        if code in _PAIR_UN:
            return self.emit_pair(lvl, f"{_PAIR_UN[code]}({names[0]})"), lvl
        raise NotPairable(f"no packed form for {code}")

    def _operand_coords(self, r: Node, coords, axes, keepdims):
        x = r.preds[0]
        if keepdims:
            kept = [c for i, c in enumerate(coords) if i not in axes]
        else:
            kept = list(coords)
        # loops need a real scope: reductions at constant coordinates live in the row scope
        lvl = max(max((c.level for c in kept), default=0), 1)
        return x, kept, lvl

    def loop_coords(self, level, dims, trip_unroll=16):
        """Open nested for-loops over ``dims`` (C order) under ``level``;
        returns (vars, scopes)."""
        vars_, opened = [], []
        cur = level
        for ext in dims:
            v, s, saved = self.open(cur, "for", trip=ext, unroll=(ext <= trip_unroll))
            vars_.append(v)
            opened.append((s, saved))
            cur = v.level
        return vars_, opened

    def close_all(self, opened):
        for s, saved in reversed(opened):
            self.close(s, saved)

    def reduce(self, r: Node, coords):
        rop, axes, keepdims, odt = r.op.attrs
        x, kept, L = self._operand_coords(r, coords, axes, keepdims)
        rk = self.reduction_key(r, kept)
        hit = self.memo_get(rk)
        if hit is not None:
            return hit
        return self.memo_put(rk, self._reduce(r, x, kept, L))

    def _reduce(self, r: Node, x: Node, kept, L):
        rop, axes, keepdims, odt = r.op.attrs
        T = r.dtype
        ct = T.ctype
        So = x.shape
        red_sizes = [So[a] for a in axes]
        nred = element_count(red_sizes)
        if L >= 2 and nred > SMALL_RECOMPUTE:
            raise NotFusable(r, f"reduction over {nred} points would be recomputed per column")
        if nred == 0:
            return self.const(_IDENT[rop](T), T)
        ident = c_literal(_IDENT[rop](T), T)
        if self.half is not None and any(c.coef(self.half) for c in kept):
            return self._reduce_pair(r, x, kept, L)
        # coalesce: NumPy merges adjacent reduced axes; the innermost group is
        # pairwise-summed when it contains the last (contiguous) axis.
        groups: List[List[int]] = []
        for a in axes:
            if groups and groups[-1][-1] == a - 1:
                groups[-1].append(a)
            else:
                groups.append([a])
        pairwise = (rop is ReduceOp.sum and T.is_float and groups and groups[-1][-1] == len(So) - 1
                    and element_count([So[a] for a in groups[-1]]) > 1)
        outer_axes = [a for g in (groups[:-1] if pairwise else groups) for a in g]
        compared_fold = (pairwise and element_count([So[a] for a in groups[-1]]) < 8 and not outer_axes
                         and self._only_compared(r))
        acc = None if compared_fold else self.var_decl(L, ct, ident)
        # sequential loops over outer reduced axes (C order)
        ovars, opened = self.loop_coords(L, [So[a] for a in outer_axes])
        loop_lvl = ovars[-1].level if ovars else L
        amap = dict(zip(outer_axes, ovars))

        def full_coords(inner_map):
            out = []
            k = 0
            for i in range(len(So)):
                if i in amap:
                    out.append(Aff.of(amap[i]))
                elif i in inner_map:
                    out.append(inner_map[i])
                else:
                    out.append(kept[k])
                    k += 1
            return out

        comb = _COMBINE[rop]
        if compared_fold:
            # consumed only by arg-reductions (ordered compares): NumPy's 0.0
            # identity add changes nothing but the sign of a zero sum, which no
            # compare sees — the sequential fold is the value (k-means: one
            # FADD less per centroid)
            g = groups[-1]
            gdims = [So[a] for a in g]
            Lg = element_count(gdims)
            part = self.var_decl(loop_lvl, ct, c_literal(-0.0, T))
            iv, s, saved = self.open(loop_lvl, "for", trip=Lg, unroll=True)
            inner = self._delin(iv, g, gdims)
            v = self.cast(self.value(x, full_coords(inner)), x.dtype, T)
            self.stmt(iv.level, f"{part} = {iv.name} == 0 ? {v[0]} : gr::add<{ct}>({part}, {v[0]});")
            self.close(s, saved)
            return part, L
        if pairwise and element_count([So[a] for a in groups[-1]]) < 8:
            # NumPy: n < 8 is a sequential fold from -0.0 — an unrolled loop, so
            # contiguous operands become one vector load
            g = groups[-1]
            gdims = [So[a] for a in g]
            Lg = element_count(gdims)
            part = self.var_decl(loop_lvl, ct, c_literal(-0.0, T))
            iv, s, saved = self.open(loop_lvl, "for", trip=Lg, unroll=True)
            inner = self._delin(iv, g, gdims)
            v = self.cast(self.value(x, full_coords(inner)), x.dtype, T)
            # -0.0 + t == t (up to a NaN payload): the first term seeds the fold
            self.stmt(iv.level, f"{part} = {iv.name} == 0 ? {v[0]} : gr::add<{ct}>({part}, {v[0]});")
            self.close(s, saved)
            self.stmt(loop_lvl, f"{acc} = gr::add<{ct}>({acc}, {part});")
        elif pairwise:
            g = groups[-1]
            gdims = [So[a] for a in g]
            Lg = element_count(gdims)
            iv, s, saved = self.open(loop_lvl, "lambda", ret_type=ct)
            inner = self._delin(iv, g, gdims)
            v = self.cast(self.value(x, full_coords(inner)), x.dtype, T)
            self.close(s, saved, ret=v[0])
            self.stmt(loop_lvl, f"{acc} = gr::add<{ct}>({acc}, gr::pairwise<{ct}, {Lg}LL>(f{iv.name}, 0));")
        else:
            v = self.cast(self.value(x, full_coords({})), x.dtype, T)
            self.stmt(loop_lvl, f"{acc} = {comb}<{ct}>({acc}, {v[0]});")
        self.close_all(opened)
        return acc, L

    def _only_compared(self, r: Node) -> bool:
        """Is every consumer of ``r`` in this region an arg-reduction?"""
        if any(q.id == r.id for q in self.region.roots):
            return False
        cid = self.cid(r)
        users = [n for n in self.region.nodes if any(self.cid(q) == cid for q in n.preds)]
        return bool(users) and all(n.kind is OpKind.ARGREDUCE for n in users)

    def _reduce_pair(self, r: Node, x: Node, kept, L):
        """A reduction evaluated for both indices of a paired loop: sums of f32
        along a short contiguous axis (NumPy's sequential n < 8 fold from -0.0,
        then the 0.0 identity), as packed adds."""
        rop, axes, keepdims, odt = r.op.attrs
        T = r.dtype
        So = x.shape
        if (rop is not ReduceOp.sum or T is not DType.f32 or x.dtype is not DType.f32
                or list(axes) != [len(So) - 1] or So[-1] >= 8):
            raise NotPairable("paired reduction other than a short f32 sum")
        n = So[-1]
        part = self.fresh("a")
        self.stmt(L, f"gr::f2 {part} = gr::splat({c_literal(-0.0, T)});")
        self.pairs.add(part)
        # consumed only by ordered compares: the 0.0 identity add only
        # changes the sign of a zero sum, which no compare sees
        compared = self._only_compared(r)
        if not compared:
            acc = self.fresh("a")
            self.stmt(L, f"gr::f2 {acc} = gr::splat({c_literal(0, T)});")
            self.pairs.add(acc)
        iv, s, saved = self.open(L, "for", trip=n, unroll=True)
        v = self.value(x, list(kept) + [Aff.of(iv)])
        # -0.0 + t == t: the first term seeds the fold (the packed add is
        # inline asm, which ptxas does not fold)
        self.stmt(iv.level, f"{part} = {iv.name} == 0 ? {self.splat(v)} : gr::p2::add({part}, {self.splat(v)});")
        self.close(s, saved)
        if compared:
            return part, L
        self.stmt(L, f"{acc} = gr::p2::add({acc}, {part});")
        return acc, L

    def _delin(self, iv: Var, group, gdims) -> Dict[int, Aff]:
        if len(group) == 1:
            return {group[0]: Aff.of(iv)}
        out = {}
        rest = Aff.of(iv)
        for a, ext in zip(reversed(group), reversed(gdims)):
            if a == group[0]:
                out[a] = rest
            else:
                out[a] = Aff.of(self.derived_var(iv.level, f"{rest.c()} % {ext}"))
                rest = Aff.of(self.derived_var(iv.level, f"{rest.c()} / {ext}"))
        return out

    def _delin_pair(self, iv: Var, group, gdims) -> Dict[int, Aff]:
        """Coordinates of the logical index 2*iv + half along one axis."""
        if len(group) != 1:
            raise NotPairable("paired loop over merged axes")
        return {group[0]: Aff.of(iv).scale(2) + Aff.of(self.half)}

    def argreduce(self, r: Node, coords):
        which, axis, keepdims = r.op.attrs
        x = r.preds[0]
        So = x.shape
        if axis is None:
            axes = tuple(range(len(So)))
            kept = []
        else:
            axes = (axis,)
            kept = [c for i, c in enumerate(coords) if i != axis] if keepdims else list(coords)
        L = max(max((c.level for c in kept), default=0), 1)
        n = element_count([So[a] for a in axes])
        if L >= 2 and n > SMALL_RECOMPUTE:
            raise NotFusable(r, f"arg-reduction over {n} points would be recomputed per column")
        if NEAREST and which == "min" and self.half is None:
            nn = self._nearest(x, axes, kept, L)
            if nn is not None:
                return nn
        return self._argreduce_exact(x, which, axes, kept, L, n)

    def _nearest(self, x: Node, axes, kept, L):
        """argmin over ((u - C) ** 2).sum(-1) with C a constant-bank centre
        table: the certified expanded-key search of gr_nearest.cuh, the exact
        NumPy-order scan only for rows it cannot certify."""
        m = match_nearest(x, axes)
        if m is None:
            return None
        u, leaf, K, D = m
        sym = self.cbank.get(leaf.id)
        if sym is None or len(kept) != 1 or kept[0].level != L:
            return None
        tsym = sym + "_nn"
        self.nearest[leaf.id] = (K, D, tsym)
        if self.nn_rows2 and self.nn_pair is None and kept[0].key() == Aff.of(Var("r", 1)).key():
            # the kernel loop searches two rows' centres at once (sharing every
            # table load) and hands this row its label
            self.nn_pair = (u, K, D, tsym, sym)
            return self.emit(L, "long long", "nnlab"), L
        pv = self.fresh("P")
        self.stmt(L, f"float {pv}[{D}];")
        iv, s, saved = self.open(L, "for", trip=D, unroll=True)
        v = self.cast(self.value(u, [kept[0], Aff.of(0), Aff.of(iv)]), u.dtype, DType.f32)
        self.stmt(iv.level, f"{pv}[{iv.name}] = {v[0]};")
        self.close(s, saved)
        lab = self.fresh("a")
        self.stmt(L, f"int {lab}; const bool {lab}ok = gr::nearest_centre<{K}, {D}>({pv}, {tsym}, {lab});")
        # uncertified rows: the exact NumPy-order scan, out of line
        self.stmt(L, f"if (!{lab}ok) {lab} = gr::nearest_exact<{K}, {D}>({pv}, {sym});")
        return self.emit(L, "long long", lab), L

    def _argreduce_exact(self, x: Node, which, axes, kept, L, n):
        """First-index arg-reduction in NumPy's order (the value compared is
        the operand exactly as NumPy computes it)."""
        So = x.shape
        T = x.dtype.ctype
        best = self.var_decl(L, T, "0")
        bi = self.var_decl(L, "long long", "0")

        def operand(iv):
            inner = self._delin(iv, list(axes), [So[a] for a in axes])
            full = []
            k = 0
            for i in range(len(So)):
                if i in inner:
                    full.append(inner[i])
                else:
                    full.append(kept[k])
                    k += 1
            return self.value(x, full)

        iv, s, saved = self.open(L, "for", trip=n, unroll=(n <= ARG_UNROLL))
        v = operand(iv)
        if not x.dtype.is_float:
            pred = "gr::arg_better_max" if which == "max" else "gr::arg_better_min"
            self.stmt(iv.level, f"if ({iv.name} == 0 || {pred}<{T}>({v[0]}, {best})) {{ {best} = {v[0]}; {bi} = {iv.name}; }}")
            self.close(s, saved)
            return bi, L
        # floats: the scan is a plain ordered compare (first index wins ties)
        # plus one add whose result is NaN whenever an operand is NaN; only
        # then is the operand rescanned for np.argmax's answer, its first NaN
        cmp = ">" if which == "max" else "<"
        nanop = "gr::max_nan" if which == "max" else "gr::min_nan"
        if self.pair_loops and n % 2 == 0 and n <= ARG_UNROLL and x.dtype is DType.f32 and self.half is None:
            # paired scan: drop the scalar loop opened above and walk pairs
            self.close(s, saved)
            self.stack[L].lines.pop()
            nacc = self.fresh("a")
            self.stmt(L, f"gr::f2 {nacc} = gr::splat(0.0f);")
            iv, s, saved = self.open(L, "for", trip=n // 2, unroll=True)
            self.half = Var("gr_half_" + iv.name, iv.level)
            try:
                inner = self._delin_pair(iv, list(axes), [So[a] for a in axes])
                full = []
                k = 0
                for i in range(len(So)):
                    if i in inner:
                        full.append(inner[i])
                    else:
                        full.append(kept[k])
                        k += 1
                v = self.value(x, full)
            finally:
                self.half = None
            pv = self.splat(v)
            self.stmt(iv.level, f"{{ const float vlo = gr::lo({pv}), vhi = gr::hi({pv}); "
                                f"if ({iv.name} != 0 && vlo {cmp} {best}) {bi} = 2 * {iv.name}; "
                                f"{best} = {iv.name} == 0 ? vlo : {nanop}({best}, vlo); "
                                f"if (vhi {cmp} {best}) {bi} = 2 * {iv.name} + 1; "
                                f"{best} = {nanop}({best}, vhi); }}")
            self.stmt(L, f"(void){nacc};")
            self.close(s, saved)
            nan_test = f"{best} != {best}"
        else:
            nacc = self.var_decl(L, T, "0")
            self.stmt(iv.level, f"if ({iv.name} == 0 || {v[0]} {cmp} {best}) {{ {best} = {v[0]}; {bi} = {iv.name}; }}")
            self.stmt(iv.level, f"{nacc} = {nacc} + {v[0]};")
            self.close(s, saved)
            nan_test = f"{nacc} != {nacc}"
        saved_if = self.stack[L + 1:]
        del self.stack[L + 1:]
        sif = Scope(L + 1, "for", header=f"if ({nan_test})")
        self.stack.append(sif)
        iv2, s2, saved2 = self.open(L + 1, "for", trip=n)
        v2 = operand(iv2)
        self.stmt(iv2.level, f"if ({v2[0]} != {v2[0]}) {{ {best} = {v2[0]}; {bi} = {iv2.name}; break; }}")
        self.close(s2, saved2)
        self.close(sif, saved_if)
        return bi, L


# ---------------------------------------------------------------------------
# Thread space analysis
# ---------------------------------------------------------------------------


def _blame(region: Region, node: Node) -> Node:
    """The node the planner should cut: an interior reduction that fixed the
    row space when possible (roots cannot be cut, only split off)."""
    root_ids = {r.id for r in region.roots}
    if node.id in root_ids:
        inner = [n for n in _reductions(region) if n.id not in root_ids and not is_total(n)]
        if inner:
            return inner[0]
    return node


def _reductions(region: Region):
    return [n for n in region.nodes if n.kind in (OpKind.REDUCE, OpKind.ARGREDUCE)]


def thread_space(region: Region):
    """(Ts, totals, rows_roots): the row shape every non-total reduction keeps."""
    totals = [r for r in region.roots if is_total(r)]
    tot_ids = {t.id for t in totals}
    reds = [n for n in _reductions(region) if n.id not in tot_ids]
    for n in _reductions(region):
        if n.id not in tot_ids and is_total(n):
            raise NotFusable(n, "a full reduction consumed inside the region")
    keyed = [r for r in region.roots if r.kind is OpKind.KEYED_SUM]
    mms = _skinny_nodes(region)
    if mms:
        for m in mms:
            if not skinny_ok(m) or any(p.id not in region.leaf_ids for p in m.preds):
                raise NotFusable(m, "product is not a skinny prologue")
        if keyed or len({m.preds[0].shape[0] for m in mms}) != 1:
            raise NotFusable(mms[0], "skinny product with keyed sums / other row spaces")
        Rm = (mms[0].preds[0].shape[0],)
        if not reds:
            for t in totals:
                if t.kind is OpKind.REDUCE and t.op.attrs[0] is ReduceOp.sum and t.dtype.is_float:
                    C = element_count(t.preds[0].shape[1:]) if len(t.preds[0].shape) >= 1 else 1
                    if not rows_tile_pairwise(Rm[0], C):
                        raise NotFusable(mms[0], "total does not split on row boundaries")
            return Rm, totals, None
    if keyed and not reds:
        return tuple(keyed[0].preds[0].shape), totals, None
    if (len(reds) == 1 and reds[0] in region.roots and len(region.roots) == 1 + len(totals) and not totals
            and not mms):
        # a lone reduction root: one thread per output element, loops over the
        # reduced axes in NumPy order (covers sum(axis=0) and middle axes)
        return tuple(reds[0].shape), totals, None
    if reds:
        prefixes = []
        for r in reds:
            x = r.preds[0]
            if r.kind is OpKind.REDUCE:
                lo = min(r.op.attrs[1])
            else:
                lo = r.op.attrs[1]
            prefixes.append((r, tuple(x.shape[:lo])))
        Ts = min((p for _, p in prefixes), key=len)
        for r, p in prefixes:
            if p[:len(Ts)] != Ts:
                raise NotFusable(_blame(region, r), f"keeps {p}, not the row shape {Ts}")
        if not Ts:
            bad = next(r for r, p in prefixes if not p)
            raise NotFusable(_blame(region, bad), "reduction over the leading axis shares a region with other outputs")
        # a float total folds one pairwise partial per row with a perfect
        # binary tree: exact only when NumPy's pairwise recursion over the
        # flattened operand splits on row boundaries all the way down.
        # Otherwise cut the row reductions out (they become a small step of
        # their own) and the total runs in the flattened-tree mode below.
        R = element_count(Ts)
        for t in totals:
            if t.kind is OpKind.REDUCE and t.op.attrs[0] is ReduceOp.sum and t.dtype.is_float:
                C = element_count(t.preds[0].shape[len(Ts):]) if len(t.preds[0].shape) >= len(Ts) else 1
                if not rows_tile_pairwise(R, C):
                    raise NotFusable(_blame(region, reds[0]),
                                     f"total over {R}x{C} does not split on row boundaries")
        virtual = None
        if mms and tuple(Ts) != Rm:
            raise NotFusable(mms[0], f"skinny product rows {Rm} differ from the region's rows {Ts}")
    else:
        # maps + totals: rows are the subtrees of NumPy's pairwise tree over the
        # flattened space at depth D, so per-row partials combined by a
        # perfect binary tree reproduce np.sum exactly for any length
        shapes = [t.preds[0].shape for t in totals] + [r.shape for r in region.roots if r.id not in tot_ids]
        S = max(shapes, key=len)
        N = element_count(S)
        D, sizes = tree_chunks(N)
        Ts = (1 << D,)
        virtual = (tuple(S), D, sizes)
    return tuple(Ts), totals, virtual


def _split(n: int) -> int:
    h = n // 2
    return h - h % 8


def rows_tile_pairwise(R: int, C: int) -> bool:
    """True iff NumPy's pairwise sum over R*C flattened elements is a perfect
    binary tree whose leaves are the R rows of C elements (oracle/pairwise.py):
    every multi-row node has > 128 elements (so it splits) and splits at a
    row boundary into two equal halves."""
    if R <= 1:
        return True
    stack = [R * C]
    while stack:
        m = stack.pop()
        if m == C:
            continue
        if m <= 128 or m % C:
            return False
        a = _split(m)
        if a % C or a != m - a:
            return False
        stack.append(a)
    return True


def tree_chunks(N: int, cmax: int = 2048):
    """(D, sorted distinct chunk sizes) for the depth-D nodes of NumPy's
    pairwise recursion over N elements (oracle/pairwise.py), D the smallest
    depth whose nodes all hold <= cmax elements.  All nodes above depth D have
    > 128 elements, so every one of them splits and there are exactly 2^D."""
    D = 0
    level = {N}
    while max(level) > cmax:
        nxt = set()
        for n in level:
            if n <= 256:
                return D, sorted(level)
            a = _split(n)
            nxt.add(a)
            nxt.add(n - a)
        level = nxt
        D += 1
    return D, sorted(level)


# ---------------------------------------------------------------------------
# Generator
# ---------------------------------------------------------------------------


def gen_rows(region: Region, kname="gr_region", block=128) -> KernelSource:
    """Thread-per-row kernel; small row-invariant leaves go to the constant
    bank (retried without a leaf that turns out to be read per row)."""
    Ts, _totals, virtual = thread_space(region)
    cbank = cbank_candidates(region, element_count(Ts)) if virtual is None else {}
    pair = PAIR_LOOPS
    while True:
        try:
            return _gen_rows(region, kname, block, cbank, pair)
        except CBankMiss as e:
            del cbank[e.leaf.id]
        except NotPairable:
            pair = False


# Paired arg-reduction loops (two candidates per packed FADD2/FFMA2): used when
# every paired operand is a constant-bank leaf, read from a pair-adjacent copy
# (one 64-bit constant = one uniform-register pair operand) that a repack
# kernel of the same module writes before each launch; the running best is
# kept with min.NaN/max.NaN so a NaN candidate needs no extra add.  Measured on
# k-means 2^26 x 64: scalar 3.25 ms; pairs gathered from the leaf layout
# 4.14 ms (254 regs, refused now); pairs from a pair-adjacent smem copy
# 2.99 ms; pair-adjacent constant bank 2.41 ms (profiles/r01s2_kmeans_variants.md).
PAIR_LOOPS = os.environ.get("GRUMPY_PAIR_LOOPS", "1") == "1"
# debug bounds checks run the unpaired element loops
if os.environ.get("GRUMPY_DEBUG_BOUNDS", "0") == "1":
    PAIR_LOOPS = False


def _gen_rows(region: Region, kname, block, cbank, pair=False) -> KernelSource:
    Ts, totals, virtual = thread_space(region)
    tot_ids = {t.id for t in totals}
    R = element_count(Ts)
    mms = _skinny_nodes(region)
    if mms:
        block, RT = SKINNY_BLOCK, SKINNY_RT
        mm = mms[0]
        ai, bi = region.leaves.index(mm.preds[0]), region.leaves.index(mm.preds[1])
        KD, NZ = mm.preds[0].shape[1], mm.preds[1].shape[1]
        cbank = {k: v for k, v in cbank.items() if k != mm.preds[1].id}
    em = LoopEmitter(region, cbank=cbank)
    em.pair_loops = pair
    em.nn_rows2 = NEAREST_PAIR_ROWS and virtual is None and len(Ts) == 1 and not mms
    rvar = Var("r", 1)
    # row coordinates
    if virtual is None:
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
    else:
        # descend NumPy's pairwise tree along the bits of r: (vo, vn) = this
        # row's chunk of the flattened space
        S, D, sizes = virtual
        N = element_count(S)
        em.stmt(1, f"long long vo = 0, vn = {N}LL;")
        if D:
            em.stmt(1, f"for (int d = {D - 1}; d >= 0; --d) {{ const long long h = vn / 2, n2 = h - h % 8; "
                       f"if ((r >> d) & 1) {{ vo += n2; vn -= n2; }} else {{ vn = n2; }} }}")

    if mms:
        if virtual is not None or len(Ts) != 1:
            raise NotFusable(mms[0], "skinny product outside a 1-D row space")
        em.skinny = (em.cid(mms[0]), row_coords[0].key())

    def full_root_coords(shape):
        """Open loops over the columns of a root of ``shape`` (shape[:len(Ts)] == Ts)."""
        cols = shape[len(Ts):]
        vars_, opened = em.loop_coords(1, list(cols))
        return row_coords + [Aff.of(v) for v in vars_], opened, cols

    def virtual_coords(S, kind="for", ret_type=None):
        if kind == "for":
            iv, s, saved = em.open(1, "for", trip="vn")
        else:
            iv, s, saved = em.open(1, "lambda", ret_type=ret_type)
        return _flat_coords(em, S, Aff.of(Var("vo", 1)) + Aff.of(iv), iv), (s, saved), iv

    for ri, r in enumerate(region.roots):
        if r.id in tot_ids or r.kind is OpKind.KEYED_SUM:
            continue
        T = r.dtype.ctype
        if virtual is not None:
            S = virtual[0]
            if tuple(r.shape) != S:
                raise NotFusable(r, "map root shape differs from the reduced space")
            coords, (s, saved), iv = virtual_coords(S)
            v = em.value(r, coords)
            em.stmt(iv.level, f"gr::st<{T}>(p.out{ri} + vo + {iv.name}, {v[0]});")
            em.close(s, saved)
            continue
        if tuple(r.shape[:len(Ts)]) != Ts:
            raise NotFusable(_blame(region, r), f"root shape {r.shape} does not start with the row shape {Ts}")
        cols = r.shape[len(Ts):]
        if element_count(cols) == 1:
            v = em.value(r, row_coords + [Aff.of(0)] * len(cols))
            em.stmt(1, f"gr::st<{T}>(p.out{ri} + r, {v[0]});")
        else:
            coords, opened, cols = full_root_coords(r.shape)
            v = em.value(r, coords)
            st = row_major_strides(cols)
            off = Aff.of(rvar).scale(element_count(cols))
            for c, s_ in zip(coords[len(Ts):], st):
                off = off + c.scale(s_)
            em.stmt(max(v[1], opened[-1][0].level), f"gr::st<{T}>(p.out{ri} + {off.c()}, {v[0]});")
            em.close_all(opened)

    # totals: one partial per row
    scratch_off = 0
    tot_meta = []
    for ri, r in enumerate(region.roots):
        if r.id not in tot_ids:
            continue
        x = r.preds[0]
        if r.kind is OpKind.ARGREDUCE:
            which = r.op.attrs[0]
            xt = x.dtype
            if virtual is not None:
                S = virtual[0]
                if tuple(x.shape) != S:
                    raise NotFusable(r, "total operand shape differs")
                best, bi = _arg_partial(em, x, which, None, S, "vn")
                glob = f"vo + {bi}"
            else:
                if tuple(x.shape[:len(Ts)]) != Ts:
                    raise NotFusable(_blame(region, r), f"total operand {x.shape} does not start with rows {Ts}")
                cols = x.shape[len(Ts):]
                C = element_count(cols)
                best, bi = _arg_partial(em, x, which, row_coords, None, C, cols)
                glob = f"r * {C}LL + {bi}"
            voff = scratch_off
            scratch_off += ((R * xt.itemsize + 255) // 256) * 256
            ioff = scratch_off
            scratch_off += ((R * 8 + 255) // 256) * 256
            em.stmt(1, f"reinterpret_cast<{xt.ctype}*>(static_cast<char*>(p.scratch) + {voff})[r] = {best};")
            em.stmt(1, f"reinterpret_cast<long long*>(static_cast<char*>(p.scratch) + {ioff})[r] = {glob};")
            tot_meta.append((ri, ("arg", which), xt, (voff, ioff)))
            continue
        rop = r.op.attrs[0]
        T = r.dtype
        ct = T.ctype
        if virtual is not None:
            S, D, sizes = virtual
            if tuple(x.shape) != S:
                raise NotFusable(r, "total operand shape differs")
            # partial = NumPy pairwise over this row's subtree of the flat space
            part = _chunk_partial(em, x, rop, T, S, sizes)
        else:
            if tuple(x.shape[:len(Ts)]) != Ts:
                raise NotFusable(_blame(region, r), f"total operand {x.shape} does not start with rows {Ts}")
            cols = x.shape[len(Ts):]
            if element_count(cols) == 1:
                v = em.cast(em.value(x, row_coords + [Aff.of(0)] * len(cols)), x.dtype, T)
                part = v[0]
            else:
                part = _row_partial(em, x, rop, T, row_coords, cols)
        off = scratch_off
        em.stmt(1, f"reinterpret_cast<{ct}*>(static_cast<char*>(p.scratch) + {off})[r] = {part};")
        tot_meta.append((ri, rop, T, off))
        scratch_off += ((R * T.itemsize + 255) // 256) * 256

    # keyed sums (np.bincount): deterministic warp histograms.  Each warp owns
    # a private shared-memory histogram; per 32 rows the (key, weight) pairs
    # are broadcast in lane order and lane (key % 32) adds them — no atomics,
    # fixed order.  Warps fold in warp order, CTAs in CTA order (last CTA).
    keyed = [(ri, r) for ri, r in enumerate(region.roots) if r.kind is OpKind.KEYED_SUM]
    warps = block // 32
    kmeta = []
    if keyed:
        NB = max(r.op.attrs[0] for _, r in keyed)
        if warps * NB * 8 * len(keyed) > 40 * 1024:
            raise UnsupportedNodeInFusedStep(f"bincount with {NB} bins exceeds the shared-memory histogram")
        key_node = keyed[0][1].preds[0]
        kv = em.cast(em.value(key_node, row_coords), key_node.dtype, DType.i64)
        em.stmt(1, f"const long long kkey = valid ? {kv[0]} : -1LL;")
        wnames = []
        for j, (ri, r) in enumerate(keyed):
            if r.preds[0] is not key_node and r.preds[0].id != key_node.id:
                raise NotFusable(r, "bincounts of one region must share their keys")
            w_ = r.preds[1] if len(r.preds) == 2 else None
            if (w_ is not None and w_.kind is OpKind.CAST and w_.dtype is DType.f64
                    and w_.preds[0].dtype in (DType.f32, DType.i32)):
                w_ = w_.preds[0]
            if w_ is not None and w_.dtype in (DType.f32, DType.i32):
                # exactly representable in f64: shuffled at 4 bytes, widened on add
                wv = em.value(w_, row_coords)
                em.stmt(1, f"const {w_.dtype.ctype} kw{j} = {wv[0]};")
            elif len(r.preds) == 2:
                wv = em.cast(em.value(r.preds[1], row_coords), r.preds[1].dtype, DType.f64)
                em.stmt(1, f"const double kw{j} = {wv[0]};")
            else:
                em.stmt(1, f"const long long kw{j} = 1LL;")
            wnames.append((j, r))
        # lanes holding the same key form a group (__match_any_sync); the
        # group's lowest lane sums the group's weights in lane order (one
        # shuffle round per extra member, rounds = largest group - 1) and
        # alone updates the bin, so every bin sees a fixed order of adds.
        # Counts are the group's population count.
        NBmax = max(r.op.attrs[0] for _j, r in wnames)
        mkey = (f"(kkey >= 0 && kkey < {NBmax}LL) ? (unsigned)kkey : 0xffffffffu" if MATCH32 and NBmax < 2 ** 31
                else "(unsigned long long)kkey")
        body = [f"const unsigned kpeers = __match_any_sync(0xffffffffu, {mkey});",
                "const unsigned klane = threadIdx.x & 31u;",
                "const bool klead = (kpeers & ((1u << klane) - 1u)) == 0u;",
                "unsigned krest = klead ? (kpeers & (kpeers - 1u)) : 0u;"]
        weighted = [(j, r) for j, r in wnames if len(r.preds) == 2]
        for j, r in weighted:
            body.append(f"double ks{j} = (double)kw{j};")
        if weighted:
            body.append("while (__any_sync(0xffffffffu, krest != 0u)) {")
            body.append("  const int ksrc = krest ? __ffs(krest) - 1 : (int)klane;")
            for j, r in weighted:
                body.append(f"  const auto kv{j} = __shfl_sync(0xffffffffu, kw{j}, ksrc);")
            body.append("  if (krest) {")
            for j, r in weighted:
                body.append(f"    ks{j} += (double)kv{j};")
            body.append("    krest &= krest - 1u;")
            body.append("  }")
            body.append("}")
        body.append("if (klead && kkey >= 0) {")
        for j, r in wnames:
            NBj = r.op.attrs[0]
            val = f"ks{j}" if len(r.preds) == 2 else "(long long)__popc(kpeers)"
            body.append(f"  if (kkey < {NBj}LL) khist{j}[(threadIdx.x >> 5) * {NBj} + kkey] += {val};")
        body.append("}")
        for line in body:
            em.stmt(1, line)
        for j, r in wnames:
            NBj = r.op.attrs[0]
            off = scratch_off
            scratch_off += ((MAX_GRID * NBj * 8 + 255) // 256) * 256
            kmeta.append((j, r, NBj, off))

    if mms and kmeta:
        raise NotFusable(mms[0], "skinny product with keyed sums")
    # leaves read as short contiguous row slices: prefetched a row ahead
    pref = []
    if ROW_PREFETCH and virtual is None and len(Ts) == 1 and not mms:
        body_txt = "\n".join(render(em.row, 1))
        for i, l in enumerate(region.leaves):
            if len(l.shape) < 1 or l.shape[0] != R or l.id in cbank:
                continue
            W = element_count(l.shape[1:])
            if W * l.dtype.itemsize > ROW_PREFETCH_MAX_BYTES:
                continue
            pat = f"p.in{i} + ({W}*r" if W > 1 else f"p.in{i} + (r"
            if pat in body_txt:
                pref.append((i, W))
    lines = ["static __device__ __forceinline__ void row(const Params& p, const long long r, const bool valid"
             + "".join(f", {r.dtype.ctype}* khist{j}" for j, r, _, _ in kmeta)
             + (f", const float (&zk)[{NZ}]" if mms else "") + (", const int nnlab" if em.nn_pair else "") + ") {",
             "  (void)valid;"]
    lines += ["  " + c for c in em.consts]
    lines += render(em.row, 1)
    lines.append("}")
    if em.nn_pair:
        u, K_, D_, tsym, csym = em.nn_pair
        pe = LoopEmitter(region, cbank=cbank)
        iv, sc, saved = pe.open(1, "for", trip=D_, unroll=True)
        v = pe.cast(pe.value(u, [Aff.of(Var("r", 1)), Aff.of(0), Aff.of(iv)]), u.dtype, DType.f32)
        pe.stmt(iv.level, f"pv[{iv.name}] = {v[0]};")
        pe.close(sc, saved)
        lines += [f"static __device__ __forceinline__ void point(const Params& p, const long long r, float (&pv)[{D_}]) {{"]
        lines += ["  " + c for c in pe.consts]
        lines += render(pe.row, 1)
        lines += ["}",
                  "// two rows' nearest centres: each table record loaded once for both",
                  "static __device__ __forceinline__ void nn_labels(const Params& p, const long long r0, const long long r1, int (&lab)[2]) {",
                  f"  float P[2][{D_}];",
                  "  point(p, r0, P[0]);",
                  "  point(p, r1, P[1]);",
                  "  bool ok[2];",
                  f"  gr::nearest_centre_n<{K_}, {D_}, 2>(P, {tsym}, lab, ok);",
                  f"  if (!ok[0]) lab[0] = gr::nearest_exact<{K_}, {D_}>(P[0], {csym});",
                  f"  if (!ok[1]) lab[1] = gr::nearest_exact<{K_}, {D_}>(P[1], {csym});",
                  "}"]
    params = _params_struct(region).replace("    void* __restrict__ scratch;",
                                             "    void* __restrict__ scratch;\n    unsigned int* ticket;")
    used_cb = []
    for i, l in enumerate(region.leaves):
        sym = cbank.get(l.id)
        if sym is not None and re.search(rf"\b{sym}\b(?!_)", "\n".join(lines)):
            used_cb.append((i, sym, element_count(l.shape) * l.dtype.itemsize))
    cdecl = "".join(f"__constant__ {region.leaves[i].dtype.ctype} {sym}[{nb // region.leaves[i].dtype.itemsize}];\n"
                    for i, sym, nb in used_cb)
    used_pair = []
    for i, sym, nb in used_cb:
        B = em.cbank_pair.get(region.leaves[i].id)
        if B and sym + "_p[" in "\n".join(lines):
            npairs = nb // region.leaves[i].dtype.itemsize // 2
            used_pair.append((i, sym + "_p", B, npairs, f"gr_repack{i}"))
            cdecl += (f"__constant__ unsigned long long {sym}_p[{npairs}];\n"
                      f'extern "C" __global__ void gr_repack{i}(const float* __restrict__ src, unsigned long long* dst) {{\n'
                      f"  for (int i = threadIdx.x; i < {npairs}; i += blockDim.x) {{\n"
                      f"    const int lo = (i / {B}) * {2 * B} + i % {B};\n"
                      f"    dst[i] = (unsigned long long)__float_as_uint(src[lo]) | ((unsigned long long)__float_as_uint(src[lo + {B}]) << 32);\n"
                      "  }\n}\n")
    inc = '#include "gr_reduce.cuh"\n'
    for lid, (K_, D_, tsym) in em.nearest.items():
        # certified nearest-centre table (gr_nearest.cuh), packed per launch
        i = next(j for j, l in enumerate(region.leaves) if l.id == lid)
        H_ = (D_ + 3) // 2 + ((D_ + 3) // 2) % 2
        words = H_ + K_ // 2 * ((D_ + 2) + (D_ + 2) % 2)
        cdecl += (f"__constant__ float2 {tsym}[{words}];\n"
                  f'extern "C" __global__ void gr_nnpack{i}(const float* __restrict__ src, float2* dst) {{\n'
                  f"  gr::nearest_pack<{K_}, {D_}>(src, dst);\n}}\n")
        used_pair.append((i, tsym, 0, words, f"gr_nnpack{i}"))
    if em.nearest:
        inc += '#include "gr_nearest.cuh"\n'
    if mms:
        # A by TMA (tensor map first in the parameter block), B as k-pairs in
        # the constant bank written by a one-CTA repack kernel of the module
        params = params.replace("  struct Params {\n", "  struct Params {\n    gr::TMap tmap0;\n", 1)
        inc += '#include "gr_tma.cuh"\n#include "gr_skinny.cuh"\n'
        psym, npairs = f"gr_skb{bi}_p", KD * NZ // 2
        cdecl += (f"__constant__ unsigned long long {psym}[{npairs}];\n"
                  f'extern "C" __global__ void gr_repack{bi}(const float* __restrict__ src, unsigned long long* dst) {{\n'
                  f"  for (int i = threadIdx.x; i < {npairs}; i += blockDim.x) {{\n"
                  f"    const int lo = (i / {NZ}) * {2 * NZ} + i % {NZ};\n"
                  f"    dst[i] = (unsigned long long)__float_as_uint(src[lo]) | ((unsigned long long)__float_as_uint(src[lo + {NZ}]) << 32);\n"
                  "  }\n}\n")
        if SKINNY_B == "cbank":
            used_pair.append((bi, psym, NZ, npairs, f"gr_repack{bi}"))
    src = [HEADER, inc, cdecl, "struct K {", params,
           f"  static constexpr long long NROWS = {R}LL;"]
    src.append("  " + "\n  ".join(lines))
    src.append("};")
    lb = f"{block}, {NEAREST_MIN_BLOCKS}" if em.nearest and NEAREST_MIN_BLOCKS > 0 else f"{block}"
    kern = [f'extern "C" __global__ void __launch_bounds__({lb}) {kname}(const K::Params p) {{',
            "  const long long stride = (long long)gridDim.x * blockDim.x;"]
    skinny_smem = 0
    if mms:
        S_ = SKINNY_STAGES
        kern = [f'extern "C" __global__ void __launch_bounds__({block}) {kname}(const __grid_constant__ K::Params p) {{',
                "  const long long stride = (long long)gridDim.x * blockDim.x;"]
        if SKINNY_B == "smem" or S_ * block * RT * 128 > 40 * 1024:
            skinny_smem = S_ * block * RT * 128 + (KD * NZ * 4 if SKINNY_B == "smem" else 0) + 1024 + 64
            kern += ["  extern __shared__ unsigned char gr_dyn[];",
                     "  float* gr_ring = reinterpret_cast<float*>(gr_dyn + ((1024u - (gr::smem_u32(gr_dyn) & 1023u)) & 1023u));",
                     f"  unsigned long long* gr_bs = reinterpret_cast<unsigned long long*>(gr_ring + {S_ * block * RT * 32});",
                     f"  unsigned long long* gr_full = gr_bs + {KD * NZ // 2 if SKINNY_B == 'smem' else 0};"]
            if SKINNY_B == "smem":
                kern.append(f"  gr::Skinny<{block}, {KD}, {NZ}, {S_}, {RT}>::load_pairs(gr_bs, p.in{bi});")
            bsrc = "gr_bs" if SKINNY_B == "smem" else psym
        else:
            kern += [f"  __shared__ __align__(1024) float gr_ring[{S_ * block * RT * 32}];",
                     f"  __shared__ __align__(8) unsigned long long gr_full[{S_}];"]
            bsrc = psym
        kern += [f"  gr::Skinny<{block}, {KD}, {NZ}, {S_}, {RT}> sk;",
                 "  sk.init(gr_ring, gr_full, &p.tmap0, K::NROWS);",
                 f"  for (long long base = (long long)blockIdx.x * {block * RT}; base < K::NROWS; base += stride * {RT}) {{",
                 f"    float zk[{RT}][{NZ}];",
                 f"    sk.tile(zk, {bsrc});",
                 "#pragma unroll",
                 f"    for (int j = 0; j < {RT}; ++j) {{",
                 f"      const long long r = base + threadIdx.x + j * {block};",
                 "      if (r < K::NROWS) K::row(p, r, true, zk[j]);",
                 "    }",
                 "  }"]
    elif kmeta:
        for j, r, NBj, off in kmeta:
            kern.append(f"  __shared__ {r.dtype.ctype} khist{j}[{warps * NBj}];")
            kern.append(f"  for (int i = threadIdx.x; i < {warps * NBj}; i += blockDim.x) khist{j}[i] = 0;")
        kern.append("  __syncthreads();")
        hargs = "".join(f", khist{j}" for j, _, _, _ in kmeta)
        if em.nn_pair:
            kern += ["  for (long long base = (long long)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < K::NROWS; base += 2 * stride) {",
                     "    const long long r = base + (threadIdx.x & 31), r1 = r + stride;"]
            kern += [f"    if (r + 2 * stride < K::NROWS) gr::prefetch_l1(p.in{i} + (r + 2 * stride) * {W}LL);" for i, W in pref]
            kern += [f"    if (r1 + 2 * stride < K::NROWS) gr::prefetch_l1(p.in{i} + (r1 + 2 * stride) * {W}LL);" for i, W in pref]
            kern += ["    const long long rc = r < K::NROWS ? r : K::NROWS - 1, r1c = r1 < K::NROWS ? r1 : K::NROWS - 1;",
                     "    int nl[2];",
                     "    K::nn_labels(p, rc, r1c, nl);",
                     f"    K::row(p, rc, r < K::NROWS{hargs}, nl[0]);",
                     f"    if (base + stride < K::NROWS) K::row(p, r1c, r1 < K::NROWS{hargs}, nl[1]);",
                     "  }",
                     "  __syncthreads();"]
        else:
            kern += ["  for (long long base = (long long)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < K::NROWS; base += stride) {",
                     "    const long long r = base + (threadIdx.x & 31);"]
            kern += [f"    if (r + stride < K::NROWS) gr::prefetch_l1(p.in{i} + (r + stride) * {W}LL);" for i, W in pref]
            kern += [f"    K::row(p, r < K::NROWS ? r : K::NROWS - 1, r < K::NROWS{hargs});",
                     "  }",
                     "  __syncthreads();"]
        for j, r, NBj, off in kmeta:
            ct = r.dtype.ctype
            kern += [f"  for (int b = threadIdx.x; b < {NBj}; b += blockDim.x) {{",
                     f"    {ct} s = khist{j}[b];",
                     f"    for (int w = 1; w < {warps}; ++w) s += khist{j}[w * {NBj} + b];",
                     f"    reinterpret_cast<{ct}*>(static_cast<char*>(p.scratch) + {off})[(long long)blockIdx.x * {NBj} + b] = s;",
                     "  }"]
    elif em.nn_pair:
        kern += ["  for (long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x; r < K::NROWS; r += 2 * stride) {",
                 "    const long long r1 = r + stride;",
                 "    int nl[2];",
                 "    K::nn_labels(p, r, r1 < K::NROWS ? r1 : r, nl);",
                 "    K::row(p, r, true, nl[0]);",
                 "    if (r1 < K::NROWS) K::row(p, r1, true, nl[1]);",
                 "  }"]
    else:
        if pref:
            kern += ["  for (long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x; r < K::NROWS; r += stride) {"]
            kern += [f"    if (r + stride < K::NROWS) gr::prefetch_l1(p.in{i} + (r + stride) * {W}LL);" for i, W in pref]
            kern += ["    K::row(p, r, true);", "  }"]
        else:
            kern += ["  for (long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x; r < K::NROWS; r += stride)",
                     "    K::row(p, r, true);"]
    if kmeta:
        # two-level fold of the per-CTA histograms: the last CTA of each group
        # of KEYED_GROUP folds its group's partials (in CTA order), the last
        # group to finish folds the group partials (in group order) — a fixed
        # association whose serial tail is two short folds, not one over the grid
        gscr = []
        for j, r, NBj, off in kmeta:
            gscr.append(scratch_off)
            scratch_off += ((-(-MAX_GRID // KEYED_GROUP)) * NBj * 8 + 255) // 256 * 256
        kern += [f"  const unsigned kgid = blockIdx.x / {KEYED_GROUP}u;",
                 f"  const unsigned kgn = min({KEYED_GROUP}u, gridDim.x - kgid * {KEYED_GROUP}u);",
                 f"  const unsigned kng = (gridDim.x + {KEYED_GROUP - 1}u) / {KEYED_GROUP}u;",
                 "  if (!gr::last_arrival(p.ticket + 1 + kgid, kgn)) return;"]
        for (j, r, NBj, off), goff in zip(kmeta, gscr):
            ct = r.dtype.ctype
            kern += [f"  for (int b = threadIdx.x; b < {NBj}; b += blockDim.x) {{",
                     f"    {ct} s = 0;",
                     f"    s = gr::seq_fold<{ct}>(s, reinterpret_cast<const {ct}*>(static_cast<const char*>(p.scratch) + {off}) + (long long)kgid * {KEYED_GROUP * NBj} + b, kgn, {NBj});",
                     f"    reinterpret_cast<{ct}*>(static_cast<char*>(p.scratch) + {goff})[(long long)kgid * {NBj} + b] = s;",
                     "  }"]
        kern.append("  if (gr::last_arrival(p.ticket, kng)) {")
        for (j, r, NBj, off), goff in zip(kmeta, gscr):
            ri = region.roots.index(r)
            ct = r.dtype.ctype
            kern += [f"    for (int b = threadIdx.x; b < {NBj}; b += blockDim.x) {{",
                     f"      {ct} s = 0;",
                     f"      s = gr::seq_fold<{ct}>(s, reinterpret_cast<const {ct}*>(static_cast<const char*>(p.scratch) + {goff}) + b, kng, {NBj});",
                     f"      p.out{ri}[b] = s;",
                     "    }"]
    elif tot_meta:
        kern.append("  if (gr::last_block(p.ticket)) {")
    if tot_meta or kmeta:
        for ri, rop, T, off in tot_meta:
            ct = T.ctype
            if isinstance(rop, tuple):
                mx = "true" if rop[1] == "max" else "false"
                voff, ioff = off
                kern.append(f"    const long long v{ri} = gr::block_arg<{mx}, {ct}>("
                            f"reinterpret_cast<const {ct}*>(static_cast<const char*>(p.scratch) + {voff}), "
                            f"reinterpret_cast<const long long*>(static_cast<const char*>(p.scratch) + {ioff}), K::NROWS);")
                kern.append(f"    if (threadIdx.x == 0) p.out{ri}[0] = v{ri};")
                continue
            ident = c_literal(_IDENT[rop](T), T)
            kern.append(f"    const {ct} v{ri} = gr::block_tree<{_OPS[rop]}, {ct}>("
                        f"reinterpret_cast<const {ct}*>(static_cast<const char*>(p.scratch) + {off}), K::NROWS, {ident});")
            fin = f"gr::add<{ct}>({c_literal(0, T)}, v{ri})" if rop is ReduceOp.sum else f"v{ri}"
            kern.append(f"    if (threadIdx.x == 0) p.out{ri}[0] = {fin};")
        kern.append("  }")
    kern.append("}")
    src += kern
    return KernelSource("rows", "\n".join(src) + "\n", kname,
                        leaf_slots=list(range(len(region.leaves))),
                        root_slots=list(range(len(region.roots))),
                        block=block, groups=R, vec=1, unroll=RT if mms else 1, scratch_bytes=scratch_off,
                        meta={"rows": R, "row_shape": Ts, "totals": len(tot_meta), "ticket": bool(tot_meta or kmeta),
                              "virtual": virtual, "block_pow2": True, "keyed": len(kmeta),
                              "max_grid": MAX_GRID if kmeta else None, "cbank": used_cb, "cbank_pair": used_pair,
                              "tmaps": [(ai, KD, R, 32, block * RT, 128)] if mms else [],
                              "skinny": (KD, NZ, SKINNY_B, block, RT, SKINNY_STAGES) if mms else None,
                              **({"smem": skinny_smem} if skinny_smem else {})})


def _row_partial(em: LoopEmitter, x: Node, rop, T: DType, row_coords, cols):
    """Reduction of x over the row's columns with NumPy order (a total's partial)."""
    ct = T.ctype
    ident = c_literal(_IDENT[rop](T), T)
    if rop is ReduceOp.sum and T.is_float:
        C = element_count(cols)
        iv, s, saved = em.open(1, "lambda", ret_type=ct)
        inner = em._delin(iv, list(range(len(row_coords), len(row_coords) + len(cols))), list(cols))
        coords = row_coords + [inner[i] for i in range(len(row_coords), len(row_coords) + len(cols))]
        v = em.cast(em.value(x, coords), x.dtype, T)
        em.close(s, saved, ret=v[0])
        return em.emit(1, ct, f"gr::pairwise<{ct}, {C}LL>(f{iv.name}, 0)")
    acc = em.var_decl(1, ct, ident)
    vars_, opened = em.loop_coords(1, list(cols))
    v = em.cast(em.value(x, row_coords + [Aff.of(v_) for v_ in vars_]), x.dtype, T)
    em.stmt(max(v[1], vars_[-1].level), f"{acc} = {_COMBINE[rop]}<{ct}>({acc}, {v[0]});")
    em.close_all(opened)
    return acc


def _flat_coords(em: LoopEmitter, S, lin: Aff, iv: Var):
    """Coordinates in S of the flat (row-major) index ``lin``."""
    if len(S) == 1:
        return [lin]
    coords = []
    rest = lin
    for d in range(len(S) - 1, -1, -1):
        if d == 0:
            coords.append(rest)
        else:
            coords.append(Aff.of(em.derived_var(iv.level, f"{rest.c()} % {S[d]}")))
            rest = Aff.of(em.derived_var(iv.level, f"{rest.c()} / {S[d]}"))
    coords.reverse()
    return coords


def _chunk_partial(em: LoopEmitter, x: Node, rop, T: DType, S, sizes):
    """Reduction of x over this row's subtree (vo, vn) of the flattened space."""
    ct = T.ctype
    ident = c_literal(_IDENT[rop](T), T)
    pw = rop is ReduceOp.sum and T.is_float
    if pw:
        iv, s, saved = em.open(1, "lambda", ret_type=ct)
    else:
        acc = em.var_decl(1, ct, ident)
        iv, s, saved = em.open(1, "for", trip="vn")
    coords = _flat_coords(em, S, Aff.of(Var("vo", 1)) + Aff.of(iv), iv)
    v = em.cast(em.value(x, coords), x.dtype, T)
    if pw:
        em.close(s, saved, ret=v[0])
        part = em.var_decl(1, ct, ident)
        cases = " ".join(f"case {n}LL: {part} = gr::pairwise<{ct}, {n}LL>(f{iv.name}, 0); break;" for n in sizes)
        em.stmt(1, f"switch (vn) {{ {cases} default: break; }}")
        return part
    em.stmt(iv.level, f"{acc} = {_COMBINE[rop]}<{ct}>({acc}, {v[0]});")
    em.close(s, saved)
    return acc


def _arg_partial(em: LoopEmitter, x: Node, which, row_coords, S, C, cols=None):
    """First-index arg-reduction of x over this row's columns (row mode) or its
    chunk (vo, vn) of the flattened space (virtual mode); returns (best, local index)."""
    T = x.dtype.ctype
    best = em.var_decl(1, T, "0")
    bi = em.var_decl(1, "long long", "0")
    iv, s, saved = em.open(1, "for", trip=C, unroll=(isinstance(C, int) and C <= 16))
    if row_coords is None:
        coords = _flat_coords(em, S, Aff.of(Var("vo", 1)) + Aff.of(iv), iv)
    else:
        nrow = len(row_coords)
        inner = em._delin(iv, list(range(nrow, nrow + len(cols))), list(cols))
        coords = list(row_coords) + [inner[i] for i in range(nrow, nrow + len(cols))]
    v = em.value(x, coords)
    pred = "gr::arg_better_max" if which == "max" else "gr::arg_better_min"
    em.stmt(iv.level, f"if ({iv.name} == 0 || {pred}<{T}>({v[0]}, {best})) {{ {best} = {v[0]}; {bi} = {iv.name}; }}")
    em.close(s, saved)
    return best, bi
