"""kernel-lowering: the reference's IterSpace / IndexMap / PointProgram /
FusedKernel view of a fused step, and ``lower`` / ``compile``.

Reference module ``kernel-lowering`` (
PAPER.md:463-483, 519-528).  On the B200 path the executable form of a step is
the generated sm_100a kernel (codegen.py → NVRTC); this module exposes the
reference-facing description of the same step so callers and tests written
against the reference's interface keep working:

* ``lower(step, g)``: iteration space = root shape (Map) or
  the root operand's shape (MapReduce, MapScan); a point program
  built by walking root → leaves composing index maps — Transpose permutes,
  Slice gives ``coord·step + offset``, broadcast dims give constant 0, Reshape
  linearizes over the output and delinearizes over the input, SliceAssign
  becomes ``select(in-region, value, target)``.  Row-fused
  interior reductions of a B200 region appear as ``fold``
  lines over their reduced coordinates.
* ``PointProgram.dump()``: the readable pseudo-C debug dump:
  one load per line with its index map, then the body in SSA form.
* ``compile(point)``: the per-point function compiled to a
  map kernel on the device (the strategy is free); calling it
  evaluates every point of the space on the GPU and returns the values at the
  requested coordinates.  The contract — value-identical to ``eval_point``
  (the oracle's per-point evaluator, oracle/eager.py) at every coordinate — is
  the dual-execution test in tests/test_gpu_executor_api.py.
"""

from __future__ import annotations

import dataclasses
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from .dag import ElemCode, Node, Op, OpKind, ReduceOp
from .errors import ShapeMismatch, UnsupportedNodeInFusedStep
from .planner import PlanStep
from .tensor import DType, TensorBuffer, element_count


# ---------------------------------------------------------------------------
# Domain types
# ---------------------------------------------------------------------------


@dataclasses.dataclass(frozen=True)
class IterSpace:
    """Ordered positive extents, one per root dimension; rank 0 → one point
    (SPEC.md:279-282)."""

    extents: Tuple[int, ...]

    @property
    def points(self) -> int:
        return element_count(self.extents)


@dataclasses.dataclass(frozen=True)
class IndexMap:
    """Per-target-dimension expression over the point coordinates i0..in-1
    (SPEC.md:283-286): ``ik``, ``ik*step+offset``, ``0`` (broadcast dim) or a
    linearize/delinearize expression (reshape)."""

    terms: Tuple[str, ...]

    def __str__(self):
        return "[" + ", ".join(self.terms) + "]"


@dataclasses.dataclass
class PointProgram:
    """Point function of a fused step.

    ``params`` are the n iteration coordinates; ``loads`` the (leaf node id,
    IndexMap) list; ``body`` the SSA lines; ``results`` one value name per
    output (the reference has one; B200 multi-root regions have several)."""

    params: Tuple[str, ...]
    loads: List[Tuple[int, IndexMap]]
    body: List[str]
    results: List[str]
    dtype: DType
    step: PlanStep
    value_nodes: List[Node]           # the nodes whose values the point function returns

    @property
    def result(self) -> str:
        return self.results[0]

    def dump(self) -> str:
        head = f"point({', '.join(self.params)}) -> {self.dtype.value}"
        lines = [head]
        lines += ["  " + b for b in self.body]
        lines.append("  return " + ", ".join(self.results))
        return "\n".join(lines) + "\n"


@dataclasses.dataclass
class FusedKernel:
    """kind Map | MapReduce | MapScan, space, point program, combine op and
    axes."""

    kind: str
    space: IterSpace
    point: PointProgram
    combine: Optional[ReduceOp] = None
    reduce_axes: Optional[Tuple[int, ...]] = None
    scan_axis: Optional[int] = None
    step: Optional[PlanStep] = None

    def __post_init__(self):
        if (self.kind == "Map") != (self.combine is None):
            raise ValueError("kind=Map ⇔ no combine op (SPEC.md:297)")


# ---------------------------------------------------------------------------
# Index-map text composition
# ---------------------------------------------------------------------------


import re

_TERM = re.compile(r"^(?:(?P<var>[A-Za-z_]\w*)(?:\*(?P<k>-?\d+))?|(?P<c>-?\d+))$")


def _affine(s: str):
    """Parse 'i0*2 + i1 - 3' style text into ({var: coef}, const), or None."""
    coefs, const = {}, 0
    for tok in re.split(r"\s+(?=[+-]\s)", s.strip()):
        sign = 1
        tok = tok.strip()
        if tok.startswith("+ "):
            tok = tok[2:]
        elif tok.startswith("- "):
            sign, tok = -1, tok[2:]
        if tok.startswith("-") and not tok[1:].isdigit():
            sign, tok = -sign, tok[1:]
        m = _TERM.match(tok)
        if m is None:
            return None
        if m.group("c") is not None:
            const += sign * int(m.group("c"))
        else:
            v = m.group("var")
            coefs[v] = coefs.get(v, 0) + sign * int(m.group("k") or 1)
    return coefs, const


def _render(coefs, const) -> str:
    parts = []
    for v, k in coefs.items():
        if k == 0:
            continue
        t = v if abs(k) == 1 else f"{v}*{abs(k)}"
        parts.append(("- " if k < 0 else "+ ") + t)
    if const:
        parts.append(("- " if const < 0 else "+ ") + str(abs(const)))
    if not parts:
        return "0"
    s = " ".join(parts)
    return s[2:] if s.startswith("+ ") else "-" + s[2:]


def _scale(c: str, k: int) -> str:
    if c == "0" or k == 0:
        return "0"
    if k == 1:
        return c
    a = _affine(c)
    if a is not None:
        return _render({v: x * k for v, x in a[0].items()}, a[1] * k)
    return f"({c})*{k}"


def _plus(a: str, b: str) -> str:
    if a == "0":
        return b
    if b == "0":
        return a
    x, y = _affine(a), _affine(b)
    if x is not None and y is not None:
        coefs = dict(x[0])
        for v, k in y[0].items():
            coefs[v] = coefs.get(v, 0) + k
        return _render(coefs, x[1] + y[1])
    return f"{a} + {b}"


def _atomic(c: str) -> bool:
    return all(ch.isalnum() or ch == "_" for ch in c)


def _bcast(cs: Sequence[str], out_shape, in_shape) -> List[str]:
    off = len(out_shape) - len(in_shape)
    return ["0" if in_shape[d] == 1 else cs[off + d] for d in range(len(in_shape))]


def _reshape(cs: Sequence[str], out_shape, in_shape) -> List[str]:
    """linearize over the output shape, delinearize over the input shape,
    per block of dims whose extents multiply to the same count."""
    out_shape, in_shape = list(out_shape), list(in_shape)
    res: List[Optional[str]] = [None] * len(in_shape)
    i = j = 0
    while i < len(out_shape) or j < len(in_shape):
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
        lin, acc = "0", 1
        for x in reversed(bi):
            if out_shape[x] != 1:
                lin = _plus(_scale(cs[x], acc), lin)
            acc *= out_shape[x]
        nonunit = [x for x in bj if in_shape[x] != 1]
        for x in bj:
            res[x] = "0"
        if len(nonunit) == 1:
            res[nonunit[0]] = lin
        elif nonunit:
            inner = 1
            lin_p = lin if _atomic(lin) else f"({lin})"
            for x in reversed(nonunit):
                ext = in_shape[x]
                if x == nonunit[0]:
                    res[x] = lin_p if inner == 1 else f"{lin_p}/{inner}"
                else:
                    res[x] = f"{lin_p}%{ext}" if inner == 1 else f"{lin_p}/{inner}%{ext}"
                inner *= ext
    return [r if r is not None else "0" for r in res]


class _PointBuilder:
    def __init__(self, step: PlanStep):
        self.leaf_ids = {l.id for l in step.leaves}
        self.loads: List[Tuple[int, IndexMap]] = []
        self.body: List[str] = []
        self.memo: Dict[tuple, str] = {}
        self.count = 0
        self.rvars = 0

    def fresh(self, p="t"):
        self.count += 1
        return f"{p}{self.count}"

    def value(self, n: Node, cs: Sequence[str], indent=0) -> str:
        key = (n.id, tuple(cs))
        hit = self.memo.get(key)
        if hit is not None:
            return hit
        v = self._value(n, list(cs), indent)
        self.memo[key] = v
        return v

    def line(self, indent, text):
        self.body.append("  " * indent + text)

    def _value(self, n: Node, cs: List[str], ind: int) -> str:
        if n.id in self.leaf_ids:
            im = IndexMap(tuple(cs))
            name = f"ld{len(self.loads)}"
            self.loads.append((n.id, im))
            self.line(ind, f"{name} = load L{n.id}{im}")
            return name
        k = n.kind
        if k is OpKind.MAP:
            if n.op.code is ElemCode.const_splat:
                return repr(n.op.attrs[0])
            args = [self.value(p, _bcast(cs, n.shape, p.shape), ind) for p in n.preds]
            args = [a if p.dtype is lt else f"{lt.value}({a})" for a, p, lt in zip(args, n.preds, n.loop)]
            name = self.fresh()
            self.line(ind, f"{name} = {n.op.code.value}({', '.join(args)})")
            return name
        if k is OpKind.CAST:
            a = self.value(n.preds[0], cs, ind)
            name = self.fresh()
            self.line(ind, f"{name} = {n.dtype.value}({a})")
            return name
        if k is OpKind.TRANSPOSE:
            (perm,) = n.op.attrs
            pc = [None] * len(perm)
            for i, ax in enumerate(perm):
                pc[ax] = cs[i]
            return self.value(n.preds[0], pc, ind)
        if k is OpKind.BROADCAST:
            return self.value(n.preds[0], _bcast(cs, n.shape, n.preds[0].shape), ind)
        if k is OpKind.SLICE:
            (sl,) = n.op.attrs
            pc = [_plus(_scale(c, step), str(start)) for c, (start, step, _l) in zip(cs, sl)]
            return self.value(n.preds[0], pc, ind)
        if k is OpKind.RESHAPE:
            return self.value(n.preds[0], _reshape(cs, n.shape, n.preds[0].shape), ind)
        if k is OpKind.SLICE_ASSIGN:
            (reg,) = n.op.attrs
            target, val = n.preds
            conds, vc = [], []
            for c, (start, step, length) in zip(cs, reg):
                rel = _plus(c, str(-start)) if start else c
                if step == 1:
                    conds.append(f"{start} <= {c} < {start + length}")
                    vc.append(rel)
                else:
                    conds.append(f"({rel}) % {step} == 0 && 0 <= ({rel})/{step} < {length}")
                    vc.append(f"({rel})/{step}")
            pred = self.fresh("p")
            self.line(ind, f"{pred} = {' && '.join(conds) if conds else 'true'}")
            vv = self.value(val, _bcast(vc, tuple(r[2] for r in reg), val.shape), ind)
            tv = self.value(target, cs, ind)
            name = self.fresh()
            self.line(ind, f"{name} = select({pred}, {vv}, {tv})")
            return name
        if k in (OpKind.REDUCE, OpKind.ARGREDUCE):
            p = n.preds[0]
            if k is OpKind.REDUCE:
                rop, axes, keepdims, _odt = n.op.attrs
                what = rop.value
            else:
                what, axis, keepdims = n.op.attrs
                axes = tuple(range(len(p.shape))) if axis is None else (axis,)
                what = "arg" + what
            pc, it, rv = [], iter(cs), []
            for d in range(len(p.shape)):
                if d in axes:
                    self.rvars += 1
                    r = f"r{self.rvars}"
                    rv.append(f"{r} < {p.shape[d]}")
                    pc.append(r)
                    if keepdims:
                        next(it)
                else:
                    pc.append(next(it))
            name = self.fresh()
            self.line(ind, f"{name} = fold {what} over ({', '.join(rv)}):")
            inner = self.value(p, pc, ind + 1)
            self.line(ind + 1, f"yield {inner}")
            return name
        raise UnsupportedNodeInFusedStep(f"{n.op!r} cannot appear inside a fused step (SPEC.md:306)")


def _map_values(step: PlanStep) -> Tuple[str, List[Node], tuple]:
    """(kernel kind, nodes the point function evaluates, space extents)."""
    roots = step.roots
    kinds = {r.kind for r in roots}
    if kinds & {OpKind.MATMUL, OpKind.MATVEC}:
        raise UnsupportedNodeInFusedStep("library calls are steps of their own (SPEC.md:306)")
    r0 = roots[0]
    if r0.kind is OpKind.SCAN:
        return "MapScan", [r0.preds[0]], tuple(r0.preds[0].shape)
    if r0.kind in (OpKind.REDUCE, OpKind.ARGREDUCE, OpKind.KEYED_SUM):
        return "MapReduce", [r0.preds[0]], tuple(r0.preds[0].shape)
    return "Map", list(roots), tuple(r0.shape)


def lower(step: PlanStep, g=None) -> FusedKernel:
    """SPEC.md:301-309."""
    if step.kind != "Fused":
        raise ValueError("lower() takes a Fused step; library steps go to run_library")
    for n in step.nodes:
        if n.kind in (OpKind.MATMUL, OpKind.MATVEC):
            raise UnsupportedNodeInFusedStep(f"{n.op!r} in the interior of a fused step (SPEC.md:306)")
        if n.kind is OpKind.SCAN and n not in step.roots:
            raise UnsupportedNodeInFusedStep("a scan is only ever a step root (SPEC.md:306)")
        if n.kind is OpKind.SCAN and len(n.preds) > 1:
            raise UnsupportedNodeInFusedStep("a seeded scan (streamed carry) has no reference point program")
    kind, vals, extents = _map_values(step)
    b = _PointBuilder(step)
    params = tuple(f"i{k}" for k in range(len(extents)))
    results = [b.value(v, params) if len(v.shape) == len(extents) else b.value(v, _bcast(params, extents, v.shape))
               for v in vals]
    point = PointProgram(params, b.loads, b.body, results, vals[0].dtype, step, vals)
    r0 = step.roots[0]
    combine = axes = scan_axis = None
    if kind == "MapReduce":
        if r0.kind is OpKind.REDUCE:
            combine, axes = r0.op.attrs[0], tuple(r0.op.attrs[1])
        elif r0.kind is OpKind.ARGREDUCE:
            combine = ReduceOp.max if r0.op.attrs[0] == "max" else ReduceOp.min
            axes = tuple(range(len(extents))) if r0.op.attrs[1] is None else (r0.op.attrs[1],)
        else:
            combine, axes = ReduceOp.sum, (0,)
    elif kind == "MapScan":
        combine = r0.op.attrs[0]
        scan_axis = r0.op.attrs[1]
    return FusedKernel(kind, IterSpace(extents), point, combine, axes, scan_axis, step)


# ---------------------------------------------------------------------------
# compile
# ---------------------------------------------------------------------------


class CompiledPoint:
    """Executable form of a point program: a generated map kernel evaluating
    the point function over the whole iteration space on the device."""

    def __init__(self, point: PointProgram):
        from . import session as _session
        self.point = point
        self.session = _session.default_session()
        ex = self.session.executor
        leaves = list(point.step.leaves)
        roots = []
        nodes = {n.id: n for n in point.step.nodes if n.id not in {r.id for r in point.step.roots}
                 or n in point.value_nodes}
        for v in point.value_nodes:
            if v.id in {l.id for l in leaves}:
                # the point function is a bare load: an identity reshape root
                # keeps it a (trivial) device map
                v2 = Node(Op(OpKind.RESHAPE, attrs=(tuple(v.shape),)), (v,), tuple(v.shape), v.dtype)
                nodes[v2.id] = v2
                roots.append(v2)
            else:
                roots.append(v)
        self._step = PlanStep("Fused", roots, sorted(nodes.values(), key=lambda n: n.id), leaves, "Map")
        self._ex = ex
        self._last = None

    def run(self, leaves: Dict[int, TensorBuffer]) -> List[TensorBuffer]:
        """Evaluate the point function at every point (one kernel launch)."""
        return self._ex.run_fused(self._step, bind=leaves)

    def __call__(self, coords, leaves: Dict[int, TensorBuffer]):
        key = tuple(sorted((k, id(v)) for k, v in leaves.items()))
        if self._last is None or self._last[0] != key:
            self._last = (key, [b.to_numpy() for b in self.run(leaves)])
        return self._last[1][0][tuple(coords)]


def compile(point: PointProgram) -> CompiledPoint:  # noqa: A001 - the reference's name
    return CompiledPoint(point)


__all__ = ["IterSpace", "IndexMap", "PointProgram", "FusedKernel", "lower", "compile", "CompiledPoint"]
