"""kernel-lowering + code generation: region → CUDA C++ for the sm_100a skeletons.

Reference module ``kernel-lowering``:
``lower`` builds an iteration space from the root shape
and composes index maps root→leaves for transpose, slice, broadcast and reshape
(PAPER.md:463-483); constants are splatted into the body
(SPEC.md:337).  The spec then interprets or natively emits the point program
("execution strategy ... is an implementation decision").

The B200 path always emits native code: the point program becomes C++ calls to
the hand-written device-function templates in ``csrc/kernels/gr_ops.cuh`` and is
instantiated into a hand-written fused-loop skeleton (``gr_map.cuh`` …), then
compiled by NVRTC for sm_100a through the C-ABI shim.

Index maps are kept *symbolic and affine* (``Aff``: Σ coef·var + const over the
kernel's coordinate variables); reshapes that cannot stay affine introduce
derived div/mod variables.  Every emitted value records the set of loop
variables it depends on and is placed in the outermost scope where those are
bound — constants at kernel scope, per-group values once per group, per-point
values inside the vector-lane loop — so broadcast operands and row-level
values are computed once, not once per point.
"""

from __future__ import annotations

import math
import os
import re
import struct
from typing import Dict, List, Optional, Sequence, Tuple

from .dag import ElemCode, Node, OpKind, ReduceOp
from .errors import UnsupportedNodeInFusedStep
from .tensor import DType, element_count, row_major_strides

# ---------------------------------------------------------------------------
# Coordinate algebra
# ---------------------------------------------------------------------------


class Var:
    """A coordinate variable of the generated kernel.

    ``level`` is the scope that binds it (0 kernel, 1 group, 2 lane, 3+ loops);
    ``align`` a known divisor of its value.
    """

    __slots__ = ("name", "level", "align", "ctype")

    def __init__(self, name, level, align=1, ctype="long long"):
        self.name = name
        self.level = level
        self.align = align
        self.ctype = ctype

    def __repr__(self):
        return self.name


class Aff:
    """Affine integer expression Σ coef·var + const (immutable)."""

    __slots__ = ("terms", "const")

    def __init__(self, terms=(), const=0):
        # terms: tuple of (Var, coef) with coef != 0, sorted by name
        self.terms = terms
        self.const = const

    @staticmethod
    def of(x):
        if isinstance(x, Aff):
            return x
        if isinstance(x, Var):
            return Aff(((x, 1),), 0)
        return Aff((), int(x))

    def __add__(self, other):
        o = Aff.of(other)
        d = {v.name: [v, c] for v, c in self.terms}
        for v, c in o.terms:
            if v.name in d:
                d[v.name][1] += c
            else:
                d[v.name] = [v, c]
        terms = tuple(sorted(((v, c) for v, c in d.values() if c != 0), key=lambda t: t[0].name))
        return Aff(terms, self.const + o.const)

    def scale(self, k):
        k = int(k)
        if k == 0:
            return Aff((), 0)
        return Aff(tuple((v, c * k) for v, c in self.terms), self.const * k)

    def coef(self, var):
        for v, c in self.terms:
            if v is var:
                return c
        return 0

    @property
    def is_const(self):
        return not self.terms

    @property
    def level(self):
        return max((v.level for v, _ in self.terms), default=0)

    def without(self, var):
        return Aff(tuple((v, c) for v, c in self.terms if v is not var), self.const)

    def alignment(self):
        """Largest known divisor of the value (0 when identically 0)."""
        g = abs(self.const)
        for v, c in self.terms:
            g = math.gcd(g, abs(c) * v.align)
        return g

    def key(self):
        return (tuple((v.name, c) for v, c in self.terms), self.const)

    def c(self, ctype="long long"):
        parts = []
        for v, c in self.terms:
            if c == 1:
                parts.append(v.name)
            elif c == -1:
                parts.append(f"-{v.name}")
            else:
                parts.append(f"{c}*{v.name}")
        if self.const or not parts:
            parts.append(str(self.const))
        s = " + ".join(parts).replace("+ -", "- ")
        return f"({s})"


def bcast_coords(coords: Sequence[Aff], out_shape, in_shape) -> List[Aff]:
    """Right-aligned broadcast index map (SPEC.md:70, 284 'constant 0')."""
    off = len(out_shape) - len(in_shape)
    return [Aff.of(0) if in_shape[d] == 1 else coords[off + d] for d in range(len(in_shape))]


# ---------------------------------------------------------------------------
# Literal formatting (bit-exact constants)
# ---------------------------------------------------------------------------


def c_literal(value, dtype: DType) -> str:
    if dtype is DType.f32:
        (u,) = struct.unpack("<I", struct.pack("<f", float(value)))
        return f"gr::f32_bits(0x{u:08x}u)"
    if dtype is DType.f64:
        (u,) = struct.unpack("<Q", struct.pack("<d", float(value)))
        return f"gr::f64_bits(0x{u:016x}ull)"
    if dtype is DType.i32:
        v = int(value)
        return "(-2147483647 - 1)" if v == -(2**31) else f"{v}"
    if dtype is DType.i64:
        v = int(value)
        return "(-9223372036854775807LL - 1)" if v == -(2**63) else f"{v}LL"
    return "true" if value else "false"


_BIN = {
    ElemCode.add: "gr::add<{T}>", ElemCode.sub: "gr::sub<{T}>", ElemCode.mul: "gr::mul<{T}>",
    ElemCode.div: "gr::div<{T}>", ElemCode.floordiv: "gr::floordiv<{T}>", ElemCode.mod: "gr::mod<{T}>",
    ElemCode.pow: "gr::pow_<{T}>", ElemCode.maximum: "gr::maximum<{T}>", ElemCode.minimum: "gr::minimum<{T}>",
    ElemCode.cmp_lt: "gr::lt<{T}>", ElemCode.cmp_gt: "gr::gt<{T}>", ElemCode.cmp_le: "gr::le<{T}>",
    ElemCode.cmp_ge: "gr::ge<{T}>", ElemCode.cmp_eq: "gr::eq<{T}>", ElemCode.cmp_ne: "gr::ne<{T}>",
    ElemCode.logical_and: "gr::land<{T}>", ElemCode.logical_or: "gr::lor<{T}>",
    ElemCode.logical_xor: "gr::lxor<{T}>",
}
_UN = {
    ElemCode.neg: "gr::neg<{T}>", ElemCode.abs: "gr::abs_", ElemCode.exp: "gr::exp_",
    ElemCode.log: "gr::log_", ElemCode.sqrt: "gr::sqrt_", ElemCode.square: "gr::square<{T}>",
    ElemCode.sin: "gr::sin_", ElemCode.cos: "gr::cos_", ElemCode.tanh: "gr::tanh_",
    ElemCode.erf: "gr::erf_", ElemCode.floor: "gr::floor_", ElemCode.ceil: "gr::ceil_",
    ElemCode.isnan: "gr::isnan_<{T}>", ElemCode.logical_not: "gr::lnot<{T}>",
}


# ---------------------------------------------------------------------------
# Region descriptor
# ---------------------------------------------------------------------------


class Region:
    """A fused step: roots (outputs), interior nodes, leaves (inputs).

    Leaves are nodes whose values come from buffers at execution time
    (materialized before the step runs, SPEC.md:195 leaves-only invariant).
    """

    def __init__(self, roots: Sequence[Node], leaves: Sequence[Node], nodes: Sequence[Node]):
        self.roots = list(roots)
        self.leaves = list(leaves)
        self.nodes = list(nodes)
        self.leaf_ids = {n.id for n in self.leaves}

    def __repr__(self):
        return f"Region(roots={[r.id for r in self.roots]}, leaves={[l.id for l in self.leaves]}, n={len(self.nodes)})"


# ---------------------------------------------------------------------------
# Generated kernel description
# ---------------------------------------------------------------------------


class KernelSource:
    """Generated source plus everything the executor needs to launch it."""

    def __init__(self, family, source, name, leaf_slots, root_slots, block, groups, vec, unroll,
                 scratch_bytes=0, meta=None):
        self.family = family
        self.source = source
        self.name = name
        self.leaf_slots = leaf_slots    # list of leaf positions (index into region.leaves)
        self.root_slots = root_slots    # list of root positions (index into region.roots)
        self.block = block
        self.groups = groups            # number of work items the grid walks
        self.vec = vec
        self.unroll = unroll
        self.scratch_bytes = scratch_bytes
        self.meta = meta or {}


# ---------------------------------------------------------------------------
# Value emission shared by all families
# ---------------------------------------------------------------------------


class ValueEmitter:
    """Emits C++ for node values at symbolic coordinates.

    Subclasses decide where statements go (``place``) and how leaves are
    loaded (``load_leaf``).  A value is (expr, level): the C expression naming
    it and the deepest scope level it depends on.
    """

    def __init__(self, region: Region):
        self.region = region
        self.memo: Dict[tuple, Tuple[str, int]] = {}
        self.counter = 0
        self.leaf_index = {n.id: i for i, n in enumerate(region.leaves)}
        self.consts: List[str] = []
        self.const_memo: Dict[tuple, str] = {}
        # families that can redo a work item emit the two-pass division
        # (gr::div_sh<FAST>) and set this before emission
        self.div_fast = False
        self.used_div_fast = False
        self.div_finalize: List[str] = []   # row-end checks of the fast division
        self.ns = ""              # name prefix (two emitters in one function)
        # fast mode (map family): slice-assigns assume the whole lane group is
        # inside the assigned region and read the value branch at unclamped,
        # affine coordinates; each assumption adds a guard the kernel checks
        # before taking the result (else the clamped, general group runs)
        self.fast = False
        self.guards: List[str] = []
        # hash-consing: structurally identical nodes (same op over the same
        # operands) share one value — e.g. the two mean computations of
        # (x - x.mean(1)) / x.std(1).  Evaluation is pure, so this is exact.
        self.canon: Dict[int, int] = {}
        seen: Dict[tuple, int] = {}
        for n in sorted(region.nodes, key=lambda x: x.id):
            if n.id in self.leaf_index:
                continue
            key = (n.op, n.shape, n.dtype, tuple(self.canon.get(p.id, p.id) for p in n.preds))
            self.canon[n.id] = seen.setdefault(key, n.id)

    def cid(self, n: Node) -> int:
        return self.canon.get(n.id, n.id)

    def _feeds_add(self, n: Node) -> bool:
        """Does a packed add/sub/neg of this region consume ``n``?"""
        cons = getattr(self, "_cons", None)
        if cons is None:
            cons = self._cons = {}
            for m in self.region.nodes:
                adds = ((m.op.kind is OpKind.MAP and m.op.code in (ElemCode.add, ElemCode.sub, ElemCode.neg))
                        or (m.op.kind is OpKind.REDUCE and m.op.attrs[0] is ReduceOp.sum))
                if adds:
                    for q in m.preds:
                        cons[self.cid(q)] = True   # hash-consed twins share the value
        return cons.get(self.cid(n), False)

    def fresh(self, prefix="t"):
        self.counter += 1
        return f"{self.ns}{prefix}{self.counter}"

    # -- to implement
    def emit(self, level: int, ctype: str, expr: str) -> str:
        raise NotImplementedError

    def load_leaf(self, leaf: Node, offset: Aff) -> Tuple[str, int]:
        raise NotImplementedError

    def bounds_exempt(self, leaf: Node) -> bool:
        """Leaves not read from global memory at ``offset`` (staged copies)."""
        return False

    # -- shared
    def const(self, value, dtype: DType) -> Tuple[str, int]:
        key = (value, dtype)
        if key not in self.const_memo:
            name = self.fresh("k")
            self.consts.append(f"const {dtype.ctype} {name} = {c_literal(value, dtype)};  // {value!r}")
            self.const_memo[key] = name
        return self.const_memo[key], 0

    def cast(self, val: Tuple[str, int], frm: DType, to: DType) -> Tuple[str, int]:
        if frm is to:
            return val
        expr, lvl = val
        return self.emit(lvl, to.ctype, f"gr::cast<{to.ctype}, {frm.ctype}>({expr})"), lvl

    def value(self, n: Node, coords: Sequence[Aff]) -> Tuple[str, int]:
        key = (self.cid(n), tuple(c.key() for c in coords))
        hit = self.memo.get(key)
        if hit is not None:
            return hit
        v = self._value(n, list(coords))
        self.memo[key] = v
        return v

    def _value(self, n: Node, coords: List[Aff]) -> Tuple[str, int]:
        if n.id in self.leaf_index:
            st = row_major_strides(n.shape)
            off = Aff.of(0)
            for c, s, ext in zip(coords, st, n.shape):
                if ext != 1:
                    off = off + c.scale(s)
            if DEBUG_BOUNDS and not self.bounds_exempt(n):
                # debug runs: every leaf read checked against its extent
                # (SPEC.md:286, 314); a violation prints and traps
                self.emit(off.level, "bool", f"gr::bounds_ok((long long)({off.c()}), {element_count(n.shape)}LL, "
                                              f"{self.leaf_index[n.id]})")
            return self.load_leaf(n, off)
        k = n.op.kind
        if k is OpKind.MAP:
            code = n.op.code
            if code is ElemCode.const_splat:
                return self.const(n.op.attrs[0], n.dtype)
            fused = self._fma(n, coords) if getattr(self, "fma_ok", False) else None
            if fused is not None:
                return fused
            args = []
            for p, lt in zip(n.preds, n.loop):
                v = self.value(p, bcast_coords(coords, n.shape, p.shape))
                args.append(self.cast(v, p.dtype, lt))
            lvl = max(a[1] for a in args)
            names = [a[0] for a in args]
            fast_ok = getattr(self, "fma_ok", False) and FAST_DIV and n.loop[0] is DType.f32
            if code is ElemCode.select:
                T = n.dtype.ctype
                expr = f"gr::select<{T}>({names[0]}, {names[1]}, {names[2]})"
            elif code is ElemCode.div and fast_ok:
                expr = f"gr::div_full({names[0]}, {names[1]})"
            elif code is ElemCode.sqrt and fast_ok:
                expr = f"gr::sqrt_approx({names[0]})"
            elif code is ElemCode.div and n.loop[0].is_float and args[1][1] < args[0][1]:
                # divisor hoisted out of the dividend's scope: one reciprocal per
                # divisor, exact Markstein correction per element
                T = n.loop[0].ctype
                rk = ("rcp", names[1])
                r = self.const_memo.get(rk)
                if r is None or args[1][1] > 0:
                    r = self.emit(args[1][1], f"gr::DivShared<{T}>", f"gr::div_prep<{T}>({names[1]})")
                    if args[1][1] == 0:
                        self.const_memo[rk] = r
                if self.div_fast and args[1][1] == 1 and args[0][1] > 1 and hasattr(self, "stmt"):
                    # row-level divisor, per-element dividends: track the
                    # dividends' range, test the window once per row
                    w = self.const_memo.get(("divrange", r))
                    if w is None:
                        w = self.fresh("w")
                        self.stmt(1, f"gr::DivRange<{T}> {w} = gr::div_range_init<{T}>();")
                        self.const_memo[("divrange", r)] = w
                        self.div_finalize.append(f"bad |= gr::div_range_bad<{T}>({w}, {r});")
                    expr = f"gr::div_shr<FAST, {T}>({names[0]}, {r}, {w})"
                    self.used_div_fast = True
                elif self.div_fast:
                    expr = f"gr::div_sh<FAST, {T}>({names[0]}, {r}, bad)"
                    self.used_div_fast = True
                else:
                    expr = f"gr::div_shared<{T}>({names[0]}, {r})"
            elif code in _BIN:
                T = n.loop[0].ctype
                expr = _BIN[code].format(T=T) + f"({names[0]}, {names[1]})"
            else:
                T = n.loop[0].ctype
                expr = _UN[code].format(T=T) + f"({names[0]})"
            return self.emit(lvl, n.dtype.ctype, expr), lvl
        if k is OpKind.CAST:
            (p,) = n.preds
            return self.cast(self.value(p, coords), p.dtype, n.dtype)
        if k is OpKind.TRANSPOSE:
            (perm,) = n.op.attrs
            (p,) = n.preds
            pc = [None] * len(perm)
            for i, ax in enumerate(perm):
                pc[ax] = coords[i]
            return self.value(p, pc)
        if k is OpKind.BROADCAST:
            (p,) = n.preds
            return self.value(p, bcast_coords(coords, n.shape, p.shape))
        if k is OpKind.SLICE:
            (sl,) = n.op.attrs
            (p,) = n.preds
            pc = [c.scale(step) + start for c, (start, step, _l) in zip(coords, sl)]
            return self.value(p, pc)
        if k is OpKind.RESHAPE:
            (p,) = n.preds
            return self.value(p, self.reshape_coords(coords, n.shape, p.shape))
        if k is OpKind.SLICE_ASSIGN:
            return self.slice_assign(n, coords)
        raise UnsupportedNodeInFusedStep(f"{n.op!r} cannot appear inside this fused step")

    def _fma(self, n: Node, coords):
        """add/sub with a single-use product operand as one fused multiply-add
        (inexact regions only: ``fma_ok``, set by the map family)."""
        code = n.op.code
        if code not in (ElemCode.add, ElemCode.sub) or not n.dtype.is_float or n.loop[0] is not n.dtype:
            return None
        fusable = getattr(self, "_fusable", None)
        if fusable is None:
            # products every consumer of which is an add/sub of the same type
            # (and that are not roots): each consumer fuses its own copy
            users = {}
            for m in self.region.nodes:
                for q in m.preds:
                    users.setdefault(q.id, []).append(m)
            roots = {r.id for r in self.region.roots}
            fusable = self._fusable = set()
            for m in self.region.nodes:
                if (m.kind is OpKind.MAP and m.op.code in (ElemCode.mul, ElemCode.square) and m.id not in roots
                        and m.id not in self.leaf_index and all(lt is m.dtype for lt in m.loop)):
                    us = users.get(m.id, [])
                    adds = [u.kind is OpKind.MAP and u.op.code in (ElemCode.add, ElemCode.sub) and u.dtype is m.dtype
                            for u in us]
                    if us and ((FMA_MULTI == "any" and any(adds)) or (FMA_MULTI == "all" and all(adds))
                               or (len(us) == 1 and all(adds))):
                        fusable.add(m.id)
        order = list(enumerate(n.preds))
        if FMA_PICK == "last":
            order.reverse()
        for k, prod in order:
            if prod.id in fusable and prod.dtype is n.dtype:
                other = n.preds[1 - k]
                pc = bcast_coords(coords, n.shape, prod.shape)
                a = self.cast(self.value(prod.preds[0], bcast_coords(pc, prod.shape, prod.preds[0].shape)),
                              prod.preds[0].dtype, n.dtype)
                b = a if prod.op.code is ElemCode.square else self.cast(
                    self.value(prod.preds[1], bcast_coords(pc, prod.shape, prod.preds[1].shape)),
                    prod.preds[1].dtype, n.dtype)
                c = self.cast(self.value(other, bcast_coords(coords, n.shape, other.shape)), other.dtype, n.dtype)
                return self._fma_emit(n, a, b, c, k)
        return None

    def _fma_emit(self, n: Node, a, b, c, k):
        T = n.dtype.ctype
        lvl = max(a[1], b[1], c[1])
        if n.op.code is ElemCode.add:
            expr = f"gr::fma_({a[0]}, {b[0]}, {c[0]})"
        elif k == 0:            # a*b - c
            expr = f"gr::fma_({a[0]}, {b[0]}, gr::neg<{T}>({c[0]}))"
        else:                   # c - a*b
            expr = f"gr::fma_(gr::neg<{T}>({a[0]}), {b[0]}, {c[0]})"
        return self.emit(lvl, T, expr), lvl

    def reshape_coords(self, coords, out_shape, in_shape) -> List[Aff]:
        """Index map through Reshape: linearize over the
        output shape, delinearize over the input shape; stays affine when the
        dims regroup without merging (splits, unit dims)."""
        out_shape = list(out_shape)
        in_shape = list(in_shape)
        res: List[Optional[Aff]] = [None] * len(in_shape)
        i = j = 0
        while i < len(out_shape) or j < len(in_shape):
            # grow blocks until products match
            bi, bj = [i], [j]
            po = out_shape[i] if i < len(out_shape) else 1
            pi = in_shape[j] if j < len(in_shape) else 1
            i += 1
            j += 1
            while po != pi:
                if po < pi:
                    bi.append(i)
                    po *= out_shape[i]
                    i += 1
                else:
                    bj.append(j)
                    pi *= in_shape[j]
                    j += 1
            bi = [x for x in bi if x < len(out_shape)]
            bj = [x for x in bj if x < len(in_shape)]
            # linear index within the block over the output dims
            lin = Aff.of(0)
            acc = 1
            for x in reversed(bi):
                lin = lin + coords[x].scale(acc)
                acc *= out_shape[x]
            nonunit = [x for x in bj if in_shape[x] != 1]
            for x in bj:
                res[x] = Aff.of(0)
            if len(nonunit) <= 1:
                if nonunit:
                    res[nonunit[0]] = lin
                continue
            # merge: delinearize with div/mod (derived variables)
            lvl = lin.level
            rest = lin
            for x in reversed(nonunit):
                ext = in_shape[x]
                if x == nonunit[0]:
                    res[x] = rest
                else:
                    q = self.derived_var(lvl, f"{rest.c()} % {ext}")
                    res[x] = Aff.of(q)
                    rest = Aff.of(self.derived_var(lvl, f"{rest.c()} / {ext}"))
        return [r if r is not None else Aff.of(0) for r in res]

    def derived_var(self, level, expr) -> Var:
        name = self.emit(level, "long long", expr)
        return Var(name, level)

    def slice_assign(self, n: Node, coords):
        """SliceAssign lowers to select(in-region, value-branch, target-branch)
        (SPEC.md:304, 336).  Value-branch coordinates are clamped so the load
        stays in bounds when the predicate is false."""
        if self.fast:
            v = self._slice_assign_interior(n, coords)
            if v is not None:
                return v
        (region,) = n.op.attrs
        target, val = n.preds
        conds = []
        vcoords = []
        lvl = 0
        for c, (start, step, length) in zip(coords, region):
            rel = (c + (-start))
            lvl = max(lvl, c.level)
            if step == 1:
                conds.append(f"({rel.c()} >= 0 && {rel.c()} < {length})")
                q = self.derived_var(c.level, f"gr::clampll({rel.c()}, {max(length - 1, 0)}LL)")
            else:
                conds.append(f"({rel.c()} % {step} == 0 && {rel.c()} / {step} >= 0 && {rel.c()} / {step} < {length})")
                q = self.derived_var(c.level, f"gr::clampll({rel.c()} / {step}, {max(length - 1, 0)}LL)")
            vcoords.append(Aff.of(q))
        pred = self.emit(lvl, "bool", " && ".join(conds) if conds else "true")
        vv = self.cast(self.value(val, bcast_coords(vcoords, tuple(r[2] for r in region), val.shape)),
                       val.dtype, n.dtype)
        tv = self.value(target, coords)
        lv = max(lvl, vv[1], tv[1])
        return self.emit(lv, n.dtype.ctype, f"gr::select<{n.dtype.ctype}>({pred}, {vv[0]}, {tv[0]})"), lv


    def _slice_assign_interior(self, n: Node, coords):
        """Fast-mode SliceAssign: the lane group lies inside the region, so the
        result is the value branch at coordinates (c - start) — affine, which
        keeps its loads vectorised.  The group-level guard is recorded."""
        (region,) = n.op.attrs
        target, val = n.preds
        lane = getattr(self, "lane_var", None)
        vec = getattr(self, "vec", 1)
        conds, vcoords = [], []
        for c, (start, step, length) in zip(coords, region):
            if step != 1:
                return None
            rel = c + (-start)
            cl = rel.coef(lane) if lane is not None else 0
            base = rel.without(lane) if lane is not None else rel
            if cl not in (0, 1) or base.level >= LEVEL_LANE:
                return None
            hi = vec - 1 if cl else 0
            conds.append(f"({base.c()}) >= 0 && ({base.c()}) + {hi} < {length}")
            vcoords.append(rel)
        self.guards.extend(conds)
        vv = self.cast(self.value(val, bcast_coords(vcoords, tuple(r[2] for r in region), val.shape)),
                       val.dtype, n.dtype)
        return vv


# ---------------------------------------------------------------------------
# Family K1: flat map
# ---------------------------------------------------------------------------

HEADER = '#include "gr_ops.cuh"\n#include "gr_mem.cuh"\n#include "gr_pair.cuh"\n'

LEVEL_KERNEL, LEVEL_GROUP, LEVEL_LANE = 0, 1, 2


class MapEmitter(ValueEmitter):
    """Three scopes: kernel constants, per-group (arrays indexed by u), per-lane."""

    def __init__(self, region, vec, vars_group, lane_var):
        super().__init__(region)
        self.vec = vec
        self.group_lines: List[str] = []   # executed for each u, values stored in [u] arrays
        self.group_decls: List[str] = []   # array declarations
        self.lane_lines: List[str] = []
        self.lane_var = lane_var

    def emit(self, level, ctype, expr):
        name = self.fresh()
        if level <= LEVEL_KERNEL:
            self.consts.append(f"const {ctype} {name} = {expr};")
            return name
        if level == LEVEL_GROUP:
            self.group_decls.append(f"{ctype} {name}[N];")
            self.group_lines.append(f"{name}[u] = {expr};")
            return f"{name}[u]"
        self.lane_lines.append(f"const {ctype} {name} = {expr};")
        return name

    def derived_var(self, level, expr):
        name = self.emit(level, "long long", expr)
        return Var(name, level)

    def _addr(self, leaf: Node, off: Aff, width: int = 1) -> str:
        """Element offset of a load; fast-mode loads run before the group's
        guard is known, so their addresses are clamped into the leaf."""
        if not self.fast:
            return off.c()
        hi = max(element_count(leaf.shape) - width, 0) // width * width   # keeps vectors aligned
        return f"gr::clampll({off.c()}, {hi}LL)"

    def group_vector(self, leaf: Node, base: Aff) -> str:
        """An aligned VEC-element vector of ``leaf`` at ``base`` (group level),
        shared by every access that needs it."""
        key = ("gvec", leaf.id, base.key())
        hit = self.const_memo.get(key)
        if hit is None:
            T = leaf.dtype.ctype
            hit = self.fresh("L")
            self.group_decls.append(f"{T} {hit}[N][{self.vec}];")
            self.group_lines.append(f"gr::ldv<{T}, {self.vec}>({hit}[u], p.in{self.leaf_index[leaf.id]} + "
                                    f"{self._addr(leaf, base, self.vec)});")
            self.const_memo[key] = hit
        return hit

    def shifted(self, leaf: Node, rest: Aff):
        """(V0, V1, s): ``rest`` = aligned base + s (0 < s < VEC), the lanes'
        elements are window[v + s] of the two aligned vectors V0 ++ V1."""
        s = rest.const % self.vec
        base = rest + (-s)
        if (s == 0 or base.alignment() % self.vec or element_count(leaf.shape) % self.vec
                or leaf.dtype.itemsize * self.vec != 16):
            return None
        return self.group_vector(leaf, base), self.group_vector(leaf, base + self.vec), s

    def load_leaf(self, leaf: Node, off: Aff):
        idx = self.leaf_index[leaf.id]
        T = leaf.dtype.ctype
        ptr = f"p.in{idx}"
        lvl = off.level
        lane = self.lane_var
        if lvl < LEVEL_LANE:
            return self.emit(lvl, T, f"gr::ld<{T}>({ptr} + {self._addr(leaf, off)})"), lvl
        cv = off.coef(lane)
        rest = off.without(lane)
        if cv == 1 and self.vec > 1 and rest.level < LEVEL_LANE and (rest.alignment() % self.vec == 0):
            name = self.group_vector(leaf, rest)
            return f"{name}[u][v]", LEVEL_LANE
        if cv == 1 and self.vec > 1 and rest.level < LEVEL_LANE:
            sh = self.shifted(leaf, rest)
            if sh is not None:
                a, b, s_ = sh
                return f"gr::pick<{T}, {self.vec}>({a}[u], {b}[u], v + {s_})", LEVEL_LANE
        return self.emit(LEVEL_LANE, T, f"gr::ld<{T}>({ptr} + {self._addr(leaf, off)})"), LEVEL_LANE


class NotPairable(Exception):
    pass


_PAIR_BIN = {
    ElemCode.add: "gr::p2::add", ElemCode.sub: "gr::p2::sub", ElemCode.mul: "gr::p2::mul",
    ElemCode.div: "gr::p2::div", ElemCode.maximum: "gr::p2::maximum", ElemCode.minimum: "gr::p2::minimum",
    ElemCode.cmp_lt: "gr::p2::lt", ElemCode.cmp_gt: "gr::p2::gt", ElemCode.cmp_le: "gr::p2::le",
    ElemCode.cmp_ge: "gr::p2::ge", ElemCode.cmp_eq: "gr::p2::eq", ElemCode.cmp_ne: "gr::p2::ne",
}
_PAIR_UN = {
    ElemCode.neg: "gr::p2::neg", ElemCode.abs: "gr::p2::abs_", ElemCode.exp: "gr::p2::exp_",
    ElemCode.log: "gr::p2::log_", ElemCode.sqrt: "gr::p2::sqrt_", ElemCode.square: "gr::p2::square",
    ElemCode.erf: "gr::p2::erf_",
}
_PAIR_BOOL = {ElemCode.logical_and: "gr::p2::land", ElemCode.logical_or: "gr::p2::lor"}


_TRANSCENDENTAL = {ElemCode.exp, ElemCode.log, ElemCode.erf, ElemCode.tanh, ElemCode.sin, ElemCode.cos,
                   ElemCode.pow}
_DISCONTINUOUS = {ElemCode.cmp_lt, ElemCode.cmp_gt, ElemCode.cmp_le, ElemCode.cmp_ge, ElemCode.cmp_eq,
                  ElemCode.cmp_ne, ElemCode.select, ElemCode.floor, ElemCode.ceil, ElemCode.mod,
                  ElemCode.floordiv, ElemCode.isnan, ElemCode.maximum, ElemCode.minimum}


def inexact_region(region: Region) -> bool:
    """Every root is a float carrying libm error (a transcendental upstream),
    and nothing in the region branches on a value (compares, selects,
    rounding to integers, max/min).  Such results are checked to a
    tolerance, never bit for bit, so a product may fuse with the add that
    consumes it (one rounding instead of NumPy's two: FFMA2)."""
    by_id = {n.id: n for n in region.nodes}
    for n in region.nodes:
        if n.kind is OpKind.MAP and n.op.code in _DISCONTINUOUS:
            return False
        if n.kind is OpKind.CAST and not n.dtype.is_float:
            return False
        if n.kind not in (OpKind.MAP, OpKind.CAST, OpKind.BROADCAST, OpKind.TRANSPOSE, OpKind.SLICE, OpKind.RESHAPE):
            return False
    memo = {}

    def trans(n):
        if n.id not in by_id:
            return False
        if n.id not in memo:
            memo[n.id] = (n.kind is OpKind.MAP and n.op.code in _TRANSCENDENTAL) or any(trans(p) for p in n.preds)
        return memo[n.id]
    return all(r.dtype.is_float and trans(r) for r in region.roots)


CONTRACT = os.environ.get("GRUMPY_CONTRACT", "1") == "1"
# fuse a product into every add/sub that consumes it (the product itself is
# then never formed) rather than only into a sole consumer
# inexact f32 regions also divide with div.full.f32 (2 ulp) and take square
# roots with sqrt.approx.f32 (the same choice in the packed body and the tail)
FAST_DIV = os.environ.get("GRUMPY_FAST_DIV", "1") == "1"
# debug runs: bounds-check every leaf read in generated kernels
DEBUG_BOUNDS = os.environ.get("GRUMPY_DEBUG_BOUNDS", "0") == "1"
# ptxas's own FFMA2 contraction of the packed body (with the tail run through
# the same body): measured 1.054 vs 1.078 ms on Black-Scholes f32, but which
# product ptxas fuses in a*b - c*d follows the emission order, which differs
# between recordings of the same program (streamed chunks vs a plain force
# disagreed in the last bit) — off; explicit, DAG-determined fusion instead
PTXAS_CONTRACT = os.environ.get("GRUMPY_PTXAS_CONTRACT", "0") == "1"
# "one": only a product with a single (add/sub) consumer; "all": a product all
# of whose consumers are adds/subs; "any": every add/sub consumer fuses its own
# copy of the product (the product is still formed for other consumers) — the
# choice ptxas makes when it contracts
FMA_MULTI = os.environ.get("GRUMPY_FMA_MULTI", "one")
# which product an add/sub of two fusable products fuses: its "first" or
# "last" operand (fixed by the DAG, never by emission order)
FMA_PICK = os.environ.get("GRUMPY_FMA_PICK", "last")


class PairMapEmitter(MapEmitter):
    """Map emitter whose lane loop walks lane PAIRS (v = 0 .. VEC/2-1) and
    evaluates f32 lane values as packed ``gr::f2`` (FADD2/FMUL2/FFMA2), bools
    as ``gr::b2``.  Values hoisted out of the lane loop stay scalar and are
    splatted once where a lane pair consumes them.  In an inexact region
    (``inexact_region``) a single-use product feeding an add/sub becomes an
    explicit FFMA2 (the same products the scalar tail fuses); every other
    product stays uncontractable (``mul_nc``)."""

    def __init__(self, *a, **k):
        super().__init__(*a, **k)
        self.contract = CONTRACT and inexact_region(self.region)
        # "explicit": the single-use products fused as explicit FFMA2 (the
        # same ones the scalar tail fuses); "ptxas": products feeding adds
        # are plain FMUL2 that ptxas contracts itself — used only when every
        # point of the space runs this packed body (no scalar tail)
        self.contract_mode = "explicit"

    def emit(self, level, ctype, expr):
        if level >= LEVEL_LANE:
            ctype = {"float": "gr::f2", "bool": "gr::b2"}.get(ctype)
            if ctype is None:
                raise NotPairable("non-f32 lane value")
        return super().emit(level, ctype, expr)

    def splat(self, val, dtype: DType):
        expr, lvl = val
        if lvl >= LEVEL_LANE:
            return val
        if dtype is DType.f32:
            key = ("splat", expr)
            hit = self.const_memo.get(key)
            if hit is None:
                hit = MapEmitter.emit(self, lvl, "gr::f2", f"gr::splat({expr})")
                if lvl == 0:
                    self.const_memo[key] = hit
            return hit, LEVEL_LANE
        if dtype is DType.bool8:
            return f"gr::b2{{{expr}, {expr}}}", LEVEL_LANE
        raise NotPairable("splat of non-f32")

    def cast(self, val, frm: DType, to: DType):
        if frm is to:
            return val
        if val[1] >= LEVEL_LANE:
            raise NotPairable("cast inside the lane loop")
        return super().cast(val, frm, to)

    def _fma_emit(self, n: Node, a, b, c, k):
        """The packed form of ``ValueEmitter._fma``: exactly the products the
        scalar (tail) body fuses are fused here, so a lane's result does not
        depend on whether it ran packed or scalar (chunking, sharding)."""
        if max(a[1], b[1], c[1]) < LEVEL_LANE:
            return super()._fma_emit(n, a, b, c, k)
        if n.dtype is not DType.f32:
            raise NotPairable("fused multiply-add on non-f32 lanes")
        if n.op.code is ElemCode.sub:
            # negate the operand that is hoisted out of the lane loop when there
            # is one (free), else per lane
            tgt = 2 if k == 0 else 0
            v = (a, b, c)[tgt]
            if v[1] < LEVEL_LANE:
                v = (MapEmitter.emit(self, v[1], "float", f"gr::neg<float>({v[0]})"), v[1])
            else:
                v = (self.emit(LEVEL_LANE, "float", f"gr::p2::neg({v[0]})"), LEVEL_LANE)
            a, b, c = [v if i == tgt else x for i, x in enumerate((a, b, c))]
        names = [self.splat(x, DType.f32)[0] for x in (a, b, c)]
        return self.emit(LEVEL_LANE, "float", f"gr::p2::fma({names[0]}, {names[1]}, {names[2]})"), LEVEL_LANE

    def _value(self, n: Node, coords):
        if n.id not in self.leaf_index and n.op.kind is OpKind.MAP and n.op.code is not ElemCode.const_splat:
            if self.contract and self.contract_mode == "explicit":
                fused = self._fma(n, coords)
                if fused is not None:
                    return fused
            code = n.op.code
            args = []
            for p, lt in zip(n.preds, n.loop):
                v = self.value(p, bcast_coords(coords, n.shape, p.shape))
                args.append((self.cast(v, p.dtype, lt), lt))
            lvl = max(a[0][1] for a in args)
            if lvl < LEVEL_LANE:
                return super()._value(n, coords)
            if any(lt not in (DType.f32, DType.bool8) for _, lt in args) or n.dtype not in (DType.f32, DType.bool8):
                raise NotPairable(f"{code} on {n.loop}")
            names = [self.splat(a, lt)[0] for a, lt in args]
            if code in (ElemCode.mul, ElemCode.square) and self._feeds_add(n) and not (
                    self.contract and self.contract_mode == "ptxas"):
                # keep ptxas from contracting the product into its add (gr_pair.cuh)
                fn = "gr::p2::mul_nc" if code is ElemCode.mul else "gr::p2::square_nc"
                return self.emit(LEVEL_LANE, n.dtype.ctype, f"{fn}({', '.join(names)})"), LEVEL_LANE
            fast_ok = self.contract and FAST_DIV and n.loop[0] is DType.f32
            if code is ElemCode.select:
                expr = f"gr::p2::select({names[0]}, {names[1]}, {names[2]})"
            elif code is ElemCode.div and fast_ok:
                expr = f"gr::p2::div_full({names[0]}, {names[1]})"
            elif code is ElemCode.sqrt and fast_ok:
                expr = f"gr::p2::sqrt_approx({names[0]})"
            elif code in _PAIR_BIN and n.loop[0] is DType.f32:
                expr = f"{_PAIR_BIN[code]}({names[0]}, {names[1]})"
            elif code in _PAIR_UN and n.loop[0] is DType.f32:
                expr = f"{_PAIR_UN[code]}({names[0]})"
            elif code in _PAIR_BOOL and n.loop[0] is DType.bool8:
                expr = f"{_PAIR_BOOL[code]}({names[0]}, {names[1]})"
            elif code is ElemCode.logical_not and n.loop[0] is DType.bool8:
                expr = f"gr::p2::lnot({names[0]})"
            else:
                raise NotPairable(f"no packed form for {code}")
            return self.emit(LEVEL_LANE, n.dtype.ctype, expr), LEVEL_LANE
        ok = (OpKind.MAP, OpKind.TRANSPOSE, OpKind.BROADCAST, OpKind.SLICE, OpKind.RESHAPE, OpKind.CAST)
        if self.fast:
            ok += (OpKind.SLICE_ASSIGN,)    # the interior form is the value branch alone
        if n.id not in self.leaf_index and n.op.kind not in ok:
            raise NotPairable(f"{n.op!r}")
        return super()._value(n, coords)

    def derived_var(self, level, expr):
        if level >= LEVEL_LANE:
            raise NotPairable("per-lane index arithmetic")
        return super().derived_var(level, expr)

    def load_leaf(self, leaf: Node, off: Aff):
        idx = self.leaf_index[leaf.id]
        T = leaf.dtype.ctype
        lvl = off.level
        if lvl < LEVEL_LANE:
            return super().load_leaf(leaf, off)
        if leaf.dtype not in (DType.f32, DType.bool8):
            raise NotPairable("non-f32 leaf in the lane loop")
        lane = self.lane_var
        cv = off.coef(lane)
        rest = off.without(lane)
        if cv == 1 and rest.level < LEVEL_LANE and rest.alignment() % self.vec == 0:
            name = self.group_vector(leaf, rest)
            if leaf.dtype is DType.f32:
                return f"gr::pk({name}[u][2 * v], {name}[u][2 * v + 1])", LEVEL_LANE
            return f"gr::b2{{{name}[u][2 * v], {name}[u][2 * v + 1]}}", LEVEL_LANE
        if cv == 1 and rest.level < LEVEL_LANE:
            sh = self.shifted(leaf, rest)
            if sh is not None:
                a, b, s_ = sh
                lo = f"gr::pick<{T}, {self.vec}>({a}[u], {b}[u], 2 * v + {s_})"
                hi = f"gr::pick<{T}, {self.vec}>({a}[u], {b}[u], 2 * v + {s_ + 1})"
                if leaf.dtype is DType.f32:
                    return f"gr::pk({lo}, {hi})", LEVEL_LANE
                return f"gr::b2{{{lo}, {hi}}}", LEVEL_LANE
        # gather: lane 2v and 2v+1 (the lane variable counts pairs)
        o0 = rest + Aff.of(lane).scale(2 * cv)
        o1 = o0 + cv
        a = f"gr::ld<{T}>(p.in{idx} + {self._addr(leaf, o0)})"
        b = f"gr::ld<{T}>(p.in{idx} + {self._addr(leaf, o1)})"
        if leaf.dtype is DType.f32:
            return self.emit(LEVEL_LANE, T, f"gr::pk({a}, {b})"), LEVEL_LANE
        return self.emit(LEVEL_LANE, T, f"gr::b2{{{a}, {b}}}"), LEVEL_LANE


def _index_ctype(region: Region) -> str:
    big = max([element_count(r.shape) for r in region.roots] + [element_count(l.shape) for l in region.leaves])
    return "long long" if big >= 2**31 - 64 else "int"


def choose_vec(region: Region, shape) -> int:
    sizes = [r.dtype.itemsize for r in region.roots] + [l.dtype.itemsize for l in region.leaves]
    vec = max(1, 16 // max(sizes))
    n = element_count(shape)
    if not shape or n == 0:
        return 1
    if len(shape) > 1 and shape[-1] % vec != 0:
        # fall back to the largest power of two dividing the innermost extent
        v = vec
        while v > 1 and shape[-1] % v != 0:
            v //= 2
        vec = v
    return vec


def gen_map(region: Region, kname="gr_region", unroll=None, block=256) -> KernelSource:
    """Family K1: every root has the same shape S; out[p] = point(p)."""
    shape = tuple(region.roots[0].shape)
    for r in region.roots:
        if tuple(r.shape) != shape:
            raise UnsupportedNodeInFusedStep("map roots must share one shape")
    n = element_count(shape)
    vec = choose_vec(region, shape)
    ngroups = n // vec
    tail = n - ngroups * vec
    ictype = _index_ctype(region)
    # one 16-byte group per leaf per thread per trip: measured best for f32 and
    # f64 (BS f64 U=2: 80 regs, 4.13 ms; U=1: 46 regs, 4.02 ms)
    if unroll is None:
        unroll = int(os.environ.get("GRUMPY_MAP_UNROLL", "1"))
    rank = len(shape)

    def build(mode, pair=False, fast=False, contract_mode="explicit"):
        lane = Var("v", LEVEL_LANE)
        cls = PairMapEmitter if pair else MapEmitter
        em = cls(region, vec if mode == "group" else 1, None, lane)
        em.fma_ok = CONTRACT and inexact_region(region) and contract_mode == "explicit"
        if pair:
            em.contract_mode = contract_mode
        if fast:
            em.fast, em.ns = True, "f"
        coords: List[Aff] = []
        if rank == 0:
            lin0 = Aff.of(0)
        else:
            # group-level coordinates from the linear start of the group
            pass
            inner = shape[-1]
            if rank == 1:
                cin = Var("lin", LEVEL_GROUP if mode == "group" else LEVEL_LANE, align=vec if mode == "group" else 1)
                coords = [Aff.of(cin) + (Aff.of(lane) if mode == "group" else Aff.of(0))]
            else:
                base = em.emit(LEVEL_GROUP if mode == "group" else LEVEL_LANE, ictype, f"lin % {inner}")
                cin = Var(base, LEVEL_GROUP if mode == "group" else LEVEL_LANE,
                          align=vec if mode == "group" else 1)
                outer: List[Aff] = []
                rest = em.emit(LEVEL_GROUP if mode == "group" else LEVEL_LANE, ictype, f"lin / {inner}")
                for d in range(rank - 2, -1, -1):
                    ext = shape[d]
                    lvl = LEVEL_GROUP if mode == "group" else LEVEL_LANE
                    if ext == 1:
                        outer.append(Aff.of(0))
                        continue
                    if d == 0:
                        outer.append(Aff.of(Var(rest, lvl)))
                    else:
                        c = em.emit(lvl, ictype, f"{rest} % {ext}")
                        outer.append(Aff.of(Var(c, lvl)))
                        rest = em.emit(lvl, ictype, f"{rest} / {ext}")
                outer.reverse()
                coords = outer + [Aff.of(cin) + (Aff.of(lane) if mode == "group" else Aff.of(0))]
        outs = []
        for ri, r in enumerate(region.roots):
            val = em.value(r, coords)
            outs.append(val)
        return em, outs

    # ---- group body (vectorised); f32 regions evaluate lane pairs packed
    pair = False
    packed_tail = False
    if vec % 2 == 0 and os.environ.get("GRUMPY_PAIR", "1") != "0" and not DEBUG_BOUNDS:
        try:
            if PTXAS_CONTRACT and CONTRACT and inexact_region(region) and (tail == 0 or rank == 1):
                # ptxas contraction, provided the tail (if any) can run this
                # same packed body (every point then gets the same contractions)
                em, outs = build("group", pair=True, contract_mode="ptxas")
                packed_tail = tail == 0 or _packable_tail(em)
                if not packed_tail:
                    em, outs = build("group", pair=True)
            else:
                em, outs = build("group", pair=True)
            pair = True
        except NotPairable:
            pair = False
    if not pair:
        em, outs = build("group")
    def lane_loop(em, outs, pair, ind):
        nl = vec // 2 if pair else vec
        out = []
        for ri, r in enumerate(region.roots):
            out.append(f"{ind}{r.dtype.ctype} o{ri}[{vec}];")
        out.append("#pragma unroll")
        out.append(f"{ind}for (int v = 0; v < {nl}; ++v) {{")
        for l in em.lane_lines:
            out.append(f"{ind}  " + l)
        for ri, (r, (expr, _lvl)) in enumerate(zip(region.roots, outs)):
            if not pair:
                out.append(f"{ind}  o{ri}[v] = {expr};")
            elif _lvl < LEVEL_LANE:
                out.append(f"{ind}  o{ri}[2 * v] = {expr}; o{ri}[2 * v + 1] = {expr};")
            elif r.dtype is DType.f32:
                out.append(f"{ind}  o{ri}[2 * v] = gr::lo({expr}); o{ri}[2 * v + 1] = gr::hi({expr});")
            else:
                out.append(f"{ind}  o{ri}[2 * v] = ({expr}).lo; o{ri}[2 * v + 1] = ({expr}).hi;")
        out.append(f"{ind}}}")
        for ri, r in enumerate(region.roots):
            T = r.dtype.ctype
            if vec > 1:
                out.append(f"{ind}gr::stv<{T}, {vec}>(p.out{ri} + lin, o{ri});")
            else:
                out.append(f"{ind}gr::st<{T}>(p.out{ri} + lin, o{ri}[0]);")
        return out

    # ---- fast group (slice-assign regions): the lane group inside every
    # assigned region, value branches at affine coordinates (vector and
    # shifted-vector loads); taken when its guard holds, else the general body
    fast_fn = []
    if unroll == 1 and vec > 1 and any(n_.kind is OpKind.SLICE_ASSIGN for n_ in region.nodes):
        fem = fouts = None
        for fpair in ((True, False) if vec % 2 == 0 and os.environ.get("GRUMPY_PAIR", "1") != "0" and not DEBUG_BOUNDS else (False,)):
            try:
                fem, fouts = build("group", pair=fpair, fast=True)
                fp = fpair
                break
            except NotPairable:
                continue
        if fem is not None and fem.guards:
            fast_fn.append("static __device__ __forceinline__ bool fast_group(const Params& p, long long g0) {")
            fast_fn += ["  " + c for c in fem.consts]
            fast_fn.append("  const int u = 0; (void)u;")
            fast_fn.append(f"  const {ictype} lin = ({ictype})g0 * {vec}; (void)lin;")
            fast_fn += ["  " + d.replace("[N]", "[1]") for d in fem.group_decls]
            fast_fn += ["  " + l for l in fem.group_lines]
            fast_fn.append(f"  if (!({' && '.join('(' + g + ')' for g in dict.fromkeys(fem.guards))})) return false;")
            fast_fn += lane_loop(fem, fouts, fp, "  ")
            fast_fn.append("  return true;")
            fast_fn.append("}")

    lines = []
    lines.append("template <int N> static __device__ __forceinline__ void group(const Params& p, long long g0, long long stride) {")
    if fast_fn:
        lines.append("  if constexpr (N == 1) { if (fast_group(p, g0)) return; }")
    for d in em.group_decls:
        lines.append("  " + d)
    lines.append("#pragma unroll")
    lines.append("  for (int u = 0; u < N; ++u) {")
    lines.append(f"    const {ictype} lin = ({ictype})(g0 + u * stride) * {vec}; (void)lin;")
    for l in em.group_lines:
        lines.append("    " + l)
    lines.append("  }")
    lines.append("#pragma unroll")
    lines.append("  for (int u = 0; u < N; ++u) {")
    lines.append(f"    const {ictype} lin = ({ictype})(g0 + u * stride) * {vec}; (void)lin;")
    lines += lane_loop(em, outs, pair, "    ")
    lines.append("  }")
    lines.append("}")
    consts = list(em.consts)

    # ---- scalar tail (rank-1 spaces whose length is not a multiple of VEC)
    tail_lines = ["static __device__ __forceinline__ void tail(const Params& p) {"]
    if tail and packed_tail and pair:
        # the last partial group through the packed body: masked vector loads
        # and stores, lanes beyond the end computed on a copy of element 0
        tail_lines.append("  const int u = 0; (void)u;")
        tail_lines.append(f"  const {ictype} lin = ({ictype}){ngroups * vec}; (void)lin;")
        for l in consts:
            tail_lines.append("  " + l)
        for d in em.group_decls:
            tail_lines.append("  " + d.replace("[N]", "[1]"))
        for l in em.group_lines:
            tail_lines.append("  " + _TAIL_LD.sub(rf"gr::ldv_part<\1, \2>(\3, \4 + (lin), {tail});", l))
        for l in lane_loop(em, outs, pair, "  "):
            tail_lines.append(_TAIL_ST.sub(rf"gr::stv_part<\1, \2>(\3 + lin, \4, {tail});", l))
    elif tail:
        em2, outs2 = build("tail")
        consts2 = em2.consts
        tail_lines.append(f"  for (int v = 0; v < {tail}; ++v) {{")
        tail_lines.append("    const int u = 0; (void)u;")
        tail_lines.append(f"    const {ictype} lin = ({ictype}){ngroups * vec} + v; (void)lin;")
        for l in consts2:
            tail_lines.append("    " + l)
        for d in em2.group_decls:
            tail_lines.append("    " + d.replace("[N]", "[1]"))
        for l in em2.group_lines:
            tail_lines.append("    " + l)
        for l in em2.lane_lines:
            tail_lines.append("    " + l)
        for ri, (r, (expr, _)) in enumerate(zip(region.roots, outs2)):
            tail_lines.append(f"    gr::st<{r.dtype.ctype}>(p.out{ri} + lin, {expr});")
        tail_lines.append("  }")
    tail_lines.append("}")

    params = _params_struct(region)
    src = [HEADER, '#include "gr_map.cuh"\n', "struct K {", params,
           f"  static constexpr long long NGROUPS = {ngroups}LL;",
           f"  static constexpr int U = {unroll};",
           f"  static constexpr bool TAIL = {'true' if tail else 'false'};"]
    if fast_fn:
        src.append("  " + "\n  ".join(fast_fn))
    src.append("  " + "\n  ".join(_wrap_consts(lines, consts)))
    src.append("  " + "\n  ".join(tail_lines))
    src.append("};")
    src.append(f'extern "C" __global__ void __launch_bounds__({block}) {kname}(const K::Params p) {{ gr::map_kernel<K>(p); }}')
    return KernelSource("map", "\n".join(src) + "\n", kname,
                        leaf_slots=list(range(len(region.leaves))),
                        root_slots=list(range(len(region.roots))),
                        block=block, groups=ngroups, vec=vec, unroll=unroll,
                        meta={"shape": shape, "tail": tail, "fast_group": bool(fast_fn)})


_TAIL_LD = re.compile(r"gr::ldv<([^,]+), (\d+)>\(([^,]+), (p\.in\d+) \+ \(lin\)\);")
_TAIL_ST = re.compile(r"gr::stv<([^,]+), (\d+)>\((p\.out\d+) \+ lin, (o\d+)\);")


def _packable_tail(em) -> bool:
    """Every global access of the packed group body is a whole vector at the
    group's start (rank-1 contiguous leaves), so the last partial group can
    run the same body with masked loads and stores."""
    for l in em.group_lines:
        if "p.in" in l and not _TAIL_LD.fullmatch(l.strip()):
            return False
    return not any("p.in" in l for l in em.lane_lines)


def _wrap_consts(fn_lines, consts):
    """Insert kernel-level constants at the top of a generated function body."""
    out = [fn_lines[0]]
    out += ["  " + c for c in consts]
    out += fn_lines[1:]
    return out


def _params_struct(region: Region) -> str:
    fields = []
    for i, l in enumerate(region.leaves):
        fields.append(f"const {l.dtype.ctype}* __restrict__ in{i};")
    for i, r in enumerate(region.roots):
        fields.append(f"{r.dtype.ctype}* __restrict__ out{i};")
    fields.append("void* __restrict__ scratch;")
    return "  struct Params {\n    " + "\n    ".join(fields) + "\n  };"


# ---------------------------------------------------------------------------
# Region canonicalisation, signatures, dispatch
# ---------------------------------------------------------------------------


def canonicalize(region: Region) -> Region:
    """Order leaves by first visit in a DFS from the roots so structurally equal
    regions produce identical kernels and parameter layouts."""
    leaf_ids = {l.id: l for l in region.leaves}
    order: List[Node] = []
    seen = set()
    stack = list(reversed(region.roots))
    while stack:
        n = stack.pop()
        if n.id in seen:
            continue
        seen.add(n.id)
        if n.id in leaf_ids:
            order.append(n)
            continue
        for p in reversed(n.preds):
            stack.append(p)
    for l in region.leaves:  # leaves only reachable through pruned paths
        if l.id not in seen:
            order.append(l)
    return Region(region.roots, order, region.nodes)


def signature(region: Region) -> tuple:
    """Structural key: equal keys ⇒ identical generated source."""
    local: Dict[int, int] = {}
    items = []
    leaf_pos = {l.id: i for i, l in enumerate(region.leaves)}

    def visit(n: Node) -> int:
        if n.id in local:
            return local[n.id]
        if n.id in leaf_pos:
            idx = len(items)
            items.append(("leaf", leaf_pos[n.id], n.shape, n.dtype.value))
        else:
            ps = tuple(visit(p) for p in n.preds)
            idx = len(items)
            items.append((repr(n.op), n.shape, n.dtype.value, ps,
                          tuple(d.value for d in n.loop) if n.loop else None))
        local[n.id] = idx
        return idx

    roots = tuple(visit(r) for r in region.roots)
    return (tuple(items), roots)


def needs_launch_when_empty(region: Region) -> bool:
    return False


def row_fusable(reduction: Node, consumer: Node) -> bool:
    """Planner hook (optimistic): may ``reduction`` stay inside ``consumer``'s
    kernel?  Row-local reductions (leading axis kept) are proposed; the code
    generator has the last word and raises NotFusable otherwise."""
    if reduction.kind is OpKind.REDUCE:
        axes = reduction.op.attrs[1]
        return bool(axes) and min(axes) > 0
    if reduction.kind is OpKind.ARGREDUCE:
        ax = reduction.op.attrs[1]
        return ax is not None and ax > 0
    return False


def generate(region: Region) -> KernelSource:
    """Pick the kernel family for a region and emit its source."""
    from . import codegen_rows
    kinds = {n.op.kind for n in region.nodes}
    if OpKind.MATMUL in kinds:
        # a skinny product as the prologue of its consumers' row kernel
        return codegen_rows.gen_rows(region)
    if OpKind.SCAN in kinds:
        from . import codegen_scan
        return codegen_scan.generate(region)
    if OpKind.KEYED_SUM in kinds:
        return codegen_rows.gen_rows(region)
    if kinds & {OpKind.REDUCE, OpKind.ARGREDUCE}:
        from . import codegen_coop, codegen_wrow
        order = (codegen_wrow, codegen_coop) if ROW_FAMILY == "wrow" else (codegen_coop, codegen_wrow)
        for fam in order:
            ks = fam.try_generate(region)
            if ks is not None:
                return ks
        return codegen_rows.gen_rows(region)
    from . import codegen_tile
    ks = codegen_tile.try_generate(region)
    if ks is not None:
        return ks
    return gen_map(region)


# long-row reduction regions: the cooperative register-staged family first
# ("coop", default) or the warp-per-row shared-memory ring ("wrow")
ROW_FAMILY = os.environ.get("GRUMPY_ROW_FAMILY", "coop")

_GEN_CACHE: Dict[tuple, KernelSource] = {}


def cached_generate(region: Region) -> KernelSource:
    """generate() memoised by structural signature (region must be canonical)."""
    sig = signature(region)
    ks = _GEN_CACHE.get(sig)
    if ks is None:
        ks = generate(region)
        if len(_GEN_CACHE) > 4096:
            _GEN_CACHE.clear()
        _GEN_CACHE[sig] = ks
    return ks


def check_step(step) -> None:
    """Planner feedback: raise NotFusable if the step's region cannot be generated."""
    cached_generate(canonicalize(Region(step.roots, step.leaves, step.nodes)))


def grid_for(ks: KernelSource, sm_count: int, blocks_per_sm: int) -> int:
    """Persistent grid: enough CTAs to cover the work, capped at one full wave
    (SM count × resident CTAs per SM)."""
    per_cta = ks.block * max(ks.unroll, 1)
    need = max(1, -(-ks.groups // per_cta))
    g = min(need, sm_count * max(blocks_per_sm, 1))
    if ks.meta.get("max_grid"):
        g = min(g, ks.meta["max_grid"])
    return int(max(1, g))
