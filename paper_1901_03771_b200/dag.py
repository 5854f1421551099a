"""expr-dag: the deferred-operation DAG recorded by the array proxies.

Follows the reference spec module ``expr-dag``:

* ``OpKind``, ``ElemCode`` and ``ReduceOp``
   name the operation vocabulary.  The B200 build adds
  ``ARGREDUCE`` (first-index argmax/argmin), ``CAST``,
  ``BROADCAST`` and ``KEYED_SUM`` (bincount) because the north-star configs need
  them and the spec's "reduce + select" formulation costs three passes.
* ``Node`` carries the paper's three attributes — operation, data,
  is_materialized — plus inferred shape and
  dtype.
* ``Graph`` is append-only; edges point from later to earlier ids, so creation
  order is a topological order.

Memory policy differs from SPEC.md:471 ("retained for the session") on purpose:
a 2^28-element Black-Scholes step allocates gigabytes, so the graph store holds
nodes weakly and a node drops its strong references to predecessors once it is
materialized (their ids are kept for audits/DOT).  Dead proxies therefore
return device memory to the pool exactly like NumPy temporaries.
"""

from __future__ import annotations

import dataclasses
import enum
import itertools
import weakref
from typing import Any, List, Optional, Sequence, Tuple

import numpy as np

from .errors import (
    AlreadyMaterializedWithDifferentData,
    BadAxis,
    DTypeMismatch,
    ShapeMismatch,
    UnsupportedDType,
)
from .tensor import (
    DType,
    Shape,
    TensorBuffer,
    broadcast_many,
    dtype_of,
    element_count,
    normalize_axes,
    normalize_axis,
)


class OpKind(enum.Enum):
    __hash__ = object.__hash__   # members are singletons: identity hash (recording hot path)

    INPUT = "Input"
    MAP = "MapElementwise"
    CAST = "Cast"
    MATMUL = "MatMul"
    MATVEC = "MatVec"
    TRANSPOSE = "Transpose"
    RESHAPE = "Reshape"
    SLICE = "Slice"
    SLICE_ASSIGN = "SliceAssign"
    BROADCAST = "Broadcast"
    REDUCE = "Reduce"
    ARGREDUCE = "ArgReduce"
    SCAN = "Scan"
    KEYED_SUM = "KeyedSum"


class ElemCode(enum.Enum):
    """Elementwise codes (SPEC.md:109-112 plus the NumPy ufuncs the drop-in needs)."""

    __hash__ = object.__hash__   # members are singletons: identity hash (recording hot path)


    add = "add"
    sub = "sub"
    mul = "mul"
    div = "div"
    floordiv = "floordiv"
    mod = "mod"
    pow = "pow"
    neg = "neg"
    abs = "abs"
    exp = "exp"
    log = "log"
    sqrt = "sqrt"
    square = "square"
    sin = "sin"
    cos = "cos"
    tanh = "tanh"
    erf = "erf"
    floor = "floor"
    ceil = "ceil"
    isnan = "isnan"
    maximum = "maximum"
    minimum = "minimum"
    cmp_lt = "cmp_lt"
    cmp_gt = "cmp_gt"
    cmp_le = "cmp_le"
    cmp_ge = "cmp_ge"
    cmp_eq = "cmp_eq"
    cmp_ne = "cmp_ne"
    logical_and = "logical_and"
    logical_or = "logical_or"
    logical_xor = "logical_xor"
    logical_not = "logical_not"
    select = "select"
    const_splat = "const_splat"


UNARY = {
    ElemCode.neg, ElemCode.abs, ElemCode.exp, ElemCode.log, ElemCode.sqrt,
    ElemCode.square, ElemCode.sin, ElemCode.cos, ElemCode.tanh, ElemCode.erf,
    ElemCode.floor, ElemCode.ceil, ElemCode.isnan, ElemCode.logical_not,
}
BINARY = {
    ElemCode.add, ElemCode.sub, ElemCode.mul, ElemCode.div, ElemCode.floordiv,
    ElemCode.mod, ElemCode.pow, ElemCode.maximum, ElemCode.minimum,
    ElemCode.cmp_lt, ElemCode.cmp_gt, ElemCode.cmp_le, ElemCode.cmp_ge,
    ElemCode.cmp_eq, ElemCode.cmp_ne, ElemCode.logical_and, ElemCode.logical_or,
    ElemCode.logical_xor,
}


def arity(code: ElemCode) -> int:
    if code is ElemCode.const_splat:
        return 0
    if code is ElemCode.select:
        return 3
    return 1 if code in UNARY else 2


# NumPy ufunc whose type resolution defines each code's loop dtypes.
UFUNC_OF = {
    ElemCode.add: np.add, ElemCode.sub: np.subtract, ElemCode.mul: np.multiply,
    ElemCode.div: np.true_divide, ElemCode.floordiv: np.floor_divide,
    ElemCode.mod: np.remainder, ElemCode.pow: np.power, ElemCode.neg: np.negative,
    ElemCode.abs: np.absolute, ElemCode.exp: np.exp, ElemCode.log: np.log,
    ElemCode.sqrt: np.sqrt, ElemCode.square: np.square, ElemCode.sin: np.sin,
    ElemCode.cos: np.cos, ElemCode.tanh: np.tanh, ElemCode.floor: np.floor,
    ElemCode.ceil: np.ceil, ElemCode.isnan: np.isnan, ElemCode.maximum: np.maximum,
    ElemCode.minimum: np.minimum, ElemCode.cmp_lt: np.less, ElemCode.cmp_gt: np.greater,
    ElemCode.cmp_le: np.less_equal, ElemCode.cmp_ge: np.greater_equal,
    ElemCode.cmp_eq: np.equal, ElemCode.cmp_ne: np.not_equal,
    ElemCode.logical_and: np.logical_and, ElemCode.logical_or: np.logical_or,
    ElemCode.logical_xor: np.logical_xor, ElemCode.logical_not: np.logical_not,
}
CODE_OF_UFUNC = {v.__name__: k for k, v in UFUNC_OF.items()}
CODE_OF_UFUNC["divide"] = ElemCode.div
CODE_OF_UFUNC["erf"] = ElemCode.erf  # scipy.special.erf


class ReduceOp(enum.Enum):
    """Associative-commutative combine ops with identities."""

    __hash__ = object.__hash__   # members are singletons: identity hash (recording hot path)


    sum = "sum"
    prod = "prod"
    max = "max"
    min = "min"


@dataclasses.dataclass(frozen=True, eq=False)
class Op:
    """An operation: kind plus immutable attributes.

    attrs by kind
      MAP          code: ElemCode; attrs = (value,) for const_splat
      CAST         attrs = (DType,)
      TRANSPOSE    attrs = (perm,)
      RESHAPE      attrs = (new_shape,)
      BROADCAST    attrs = (new_shape,)
      SLICE        attrs = (((start, step, length), ...),)   per dim, step != 0
      SLICE_ASSIGN attrs = (((start, step, length), ...),)   region in target
      REDUCE       attrs = (ReduceOp, axes, keepdims, out DType or None)
      ARGREDUCE    attrs = ("max"|"min", axis or None, keepdims)
      SCAN         attrs = (ReduceOp, axis or None, out DType or None)
      MATMUL       attrs = ()
      MATVEC       attrs = (transposed,)   transposed: y = x @ M instead of M @ x
      KEYED_SUM    attrs = (nbins,)        preds (keys[, weights])
    """

    kind: OpKind
    code: Optional[ElemCode] = None
    attrs: Tuple[Any, ...] = ()

    # structural equality with the hash computed once (plan-cache keys hash
    # every op of a DAG signature on every force)
    def __post_init__(self):
        object.__setattr__(self, "_h", hash((self.kind, self.code, self.attrs)))

    def __hash__(self):
        return self._h

    def __eq__(self, other):
        if self is other:
            return True
        if other.__class__ is not Op:
            return NotImplemented
        return self._h == other._h and self.kind is other.kind and self.code is other.code and self.attrs == other.attrs

    def __repr__(self):
        if self.kind is OpKind.MAP:
            if self.code is ElemCode.const_splat:
                return f"const({self.attrs[0]!r})"
            return self.code.value
        if self.attrs:
            return f"{self.kind.value}{self.attrs!r}"
        return self.kind.value


INPUT_OP = Op(OpKind.INPUT)


def const_op(value) -> Op:
    return Op(OpKind.MAP, ElemCode.const_splat, (value,))


_ids = itertools.count()
_MAP_INFER: dict = {}


class Node:
    """One recorded operation.

    ``loop`` holds the input dtypes of the resolved NumPy ufunc loop for MAP
    nodes (operands are cast to these before the op, as NumPy does).
    """

    __slots__ = ("id", "op", "preds", "pred_ids", "shape", "dtype", "data", "loop", "dist", "__weakref__")

    def __init__(self, op: Op, preds: Sequence["Node"], shape: Shape, dtype: DType, loop=None, data=None):
        self.dist = None   # distribution tag after a sharded force (distributed.py)
        self.id = next(_ids)
        self.op = op
        self.preds: Tuple[Node, ...] = tuple(preds)
        self.pred_ids = tuple([p.id for p in self.preds])
        self.shape = shape
        self.dtype = dtype
        self.loop = loop
        self.data: Optional[TensorBuffer] = data

    @property
    def is_materialized(self) -> bool:
        return self.data is not None

    @property
    def kind(self) -> OpKind:
        return self.op.kind

    @property
    def size(self) -> int:
        return element_count(self.shape)

    def __repr__(self):
        m = " [M]" if self.is_materialized else ""
        return f"{self.id}: {self.op!r} {self.shape} {self.dtype.value}{m}"


# ----------------------------------------------------------------------------
# Inference
# ----------------------------------------------------------------------------

_SUPPORTED_NP = {d.np for d in DType}


def _resolve_loop(code: ElemCode, in_dtypes: Sequence[Any]):
    """NumPy loop resolution for ``code``.

    ``in_dtypes`` entries are DType (strong) or the Python types ``int``/``float``
    (weak scalars, NEP 50).  Returns (loop input DTypes, output DType).
    """
    if code is ElemCode.erf:
        # scipy.special.erf has loops f->f, d->d: the first loop the input
        # casts to safely (bool, f32 -> f; ints, f64 -> d).
        d = in_dtypes[0]
        if d is DType.f32 or d is DType.bool8:
            return (DType.f32,), DType.f32
        return (DType.f64,), DType.f64
    uf = UFUNC_OF[code]
    args = tuple(d.np if isinstance(d, DType) else d for d in in_dtypes) + (None,)
    try:
        res = uf.resolve_dtypes(args)
    except Exception as e:  # numpy raises _UFuncNoLoopError / TypeError
        raise DTypeMismatch(f"{uf.__name__} does not support dtypes {in_dtypes}: {e}") from None
    for r in res:
        if r not in _SUPPORTED_NP:
            raise UnsupportedDType(f"{uf.__name__}{tuple(in_dtypes)} resolves to {r}")
    return tuple(dtype_of(r) for r in res[:-1]), dtype_of(res[-1])


_LOOP_CACHE: dict = {}


def resolve_map(code: ElemCode, in_dtypes: Sequence[Any]):
    """Public wrapper used by the session (weak Python scalars allowed).

    Memoised: NumPy's resolution is a pure function of (ufunc, dtypes)."""
    key = (code, tuple(in_dtypes))
    hit = _LOOP_CACHE.get(key)
    if hit is None:
        hit = _resolve_map(code, key[1])
        _LOOP_CACHE[key] = hit
    return hit


def _resolve_map(code: ElemCode, in_dtypes: Sequence[Any]):
    if code is ElemCode.select:
        cond, a, b = in_dtypes
        args = [x.np if isinstance(x, DType) else x for x in (a, b)]
        try:
            r = np.result_type(*args)
        except Exception as e:
            raise DTypeMismatch(str(e)) from None
        if r not in _SUPPORTED_NP:
            raise UnsupportedDType(f"where resolves to {r}")
        out = dtype_of(r)
        return (DType.bool8, out, out), out
    return _resolve_loop(code, in_dtypes)


def _reduce_dtype(op: ReduceOp, d: DType) -> DType:
    # NumPy: add/multiply reductions upcast bool and small ints to the default int.
    if op in (ReduceOp.sum, ReduceOp.prod) and d in (DType.bool8, DType.i32):
        return DType.i64
    return d


def infer(op: Op, pred_shapes: Sequence[Shape], pred_dtypes: Sequence[DType]) -> Tuple[Shape, DType, Any]:
    """Shape/dtype inference.  Returns (shape, dtype, loop)."""
    k = op.kind
    if k is OpKind.INPUT:
        raise ShapeMismatch("Input nodes are created with add_input")
    if k is OpKind.MAP:
        code = op.code
        if len(pred_shapes) != arity(code):
            raise ShapeMismatch(f"{code.value} takes {arity(code)} operands, got {len(pred_shapes)}")
        if code is ElemCode.const_splat:
            raise ShapeMismatch("const_splat nodes are created with add_const")
        s0 = pred_shapes[0]
        shape = s0 if all(s == s0 for s in pred_shapes) else broadcast_many(pred_shapes)
        loop, out = resolve_map(code, pred_dtypes)
        return shape, out, loop
    if k is OpKind.CAST:
        return tuple(pred_shapes[0]), op.attrs[0], None
    if k is OpKind.TRANSPOSE:
        (perm,) = op.attrs
        s = pred_shapes[0]
        if sorted(perm) != list(range(len(s))):
            raise BadAxis(f"{perm} is not a permutation of 0..{len(s) - 1}")
        return tuple(s[p] for p in perm), pred_dtypes[0], None
    if k is OpKind.RESHAPE:
        (ns,) = op.attrs
        if element_count(ns) != element_count(pred_shapes[0]):
            raise ShapeMismatch(f"cannot reshape {pred_shapes[0]} into {ns}")
        return tuple(ns), pred_dtypes[0], None
    if k is OpKind.BROADCAST:
        (ns,) = op.attrs
        if broadcast_many([ns, pred_shapes[0]]) != tuple(ns):
            raise ShapeMismatch(f"cannot broadcast {pred_shapes[0]} to {ns}")
        return tuple(ns), pred_dtypes[0], None
    if k is OpKind.SLICE:
        (sl,) = op.attrs
        s = pred_shapes[0]
        if len(sl) != len(s):
            raise ShapeMismatch("slice rank mismatch")
        out = []
        for (start, step, length), ext in zip(sl, s):
            if length < 0 or step == 0:
                raise ShapeMismatch("bad slice")
            if length and not (0 <= start < ext and 0 <= start + (length - 1) * step < ext):
                raise ShapeMismatch(f"slice ({start},{step},{length}) outside extent {ext}")
            out.append(length)
        return tuple(out), pred_dtypes[0], None
    if k is OpKind.SLICE_ASSIGN:
        (region,) = op.attrs
        ts, vs = pred_shapes
        if len(region) != len(ts):
            raise ShapeMismatch("slice-assign rank mismatch")
        rshape = tuple(r[2] for r in region)
        for (start, step, length), ext in zip(region, ts):
            if length and not (0 <= start < ext and 0 <= start + (length - 1) * step < ext):
                raise ShapeMismatch("slice-assign region outside target")
        if broadcast_many([rshape, vs]) != rshape:
            raise ShapeMismatch(f"value of shape {vs} does not broadcast to region {rshape}")
        return tuple(ts), pred_dtypes[0], None
    if k is OpKind.REDUCE:
        rop, axes, keepdims, odt = op.attrs
        s = pred_shapes[0]
        for a in axes:
            if not 0 <= a < len(s):
                raise BadAxis(f"axis {a} out of range for rank {len(s)}")
        if keepdims:
            shape = tuple(1 if i in axes else d for i, d in enumerate(s))
        else:
            shape = tuple(d for i, d in enumerate(s) if i not in axes)
        if rop in (ReduceOp.max, ReduceOp.min):
            if any(s[a] == 0 for a in axes):
                raise ShapeMismatch(f"zero-size reduction of {rop.value} has no identity")
        return shape, odt or _reduce_dtype(rop, pred_dtypes[0]), None
    if k is OpKind.ARGREDUCE:
        which, axis, keepdims = op.attrs
        s = pred_shapes[0]
        if axis is None:
            if element_count(s) == 0:
                raise ShapeMismatch("attempt to get arg%s of an empty sequence" % which)
            shape = (1,) * len(s) if keepdims else ()
        else:
            if not 0 <= axis < len(s):
                raise BadAxis(f"axis {axis} out of range")
            if s[axis] == 0:
                raise ShapeMismatch("attempt to get arg%s of an empty sequence" % which)
            shape = tuple(1 if i == axis else d for i, d in enumerate(s)) if keepdims else \
                tuple(d for i, d in enumerate(s) if i != axis)
        return shape, DType.i64, None
    if k is OpKind.SCAN:
        # an optional second operand seeds the fold: out[k] = init (+) x[0]
        # (+) ... (+) x[k], init shaped like one line of the scan (the kept
        # axes; (1,) for 1-D) — the streamed chunks' carry (streaming.py)
        rop, axis, odt = op.attrs
        s = pred_shapes[0]
        if axis is None:
            shape = (element_count(s),)
        else:
            if not 0 <= axis < len(s):
                raise BadAxis(f"axis {axis} out of range")
            shape = tuple(s)
        if len(pred_shapes) > 1:
            kept = (1,) if axis is None or len(s) == 1 else tuple(d for i, d in enumerate(s) if i != axis)
            if tuple(pred_shapes[1]) != kept:
                raise ShapeMismatch(f"scan seed of shape {tuple(pred_shapes[1])}, expected {kept}")
        return shape, odt or _reduce_dtype(rop, pred_dtypes[0]), None
    if k is OpKind.MATMUL:
        a, b = pred_shapes
        if len(a) != 2 or len(b) != 2 or a[1] != b[0]:
            raise ShapeMismatch(f"matmul shapes {a} and {b} not aligned")
        return (a[0], b[1]), _matmul_dtype(pred_dtypes), None
    if k is OpKind.MATVEC:
        (trans,) = op.attrs
        a, b = pred_shapes
        if not trans:
            if len(a) != 2 or len(b) != 1 or a[1] != b[0]:
                raise ShapeMismatch(f"matvec shapes {a} and {b} not aligned")
            return (a[0],), _matmul_dtype(pred_dtypes), None
        # x @ M: preds (M, x) with M [k, n], x [k]
        if len(a) != 2 or len(b) != 1 or a[0] != b[0]:
            raise ShapeMismatch(f"vecmat shapes {b} and {a} not aligned")
        return (a[1],), _matmul_dtype(pred_dtypes), None
    if k is OpKind.KEYED_SUM:
        (nbins,) = op.attrs
        ks = pred_shapes[0]
        if len(ks) != 1:
            raise ShapeMismatch("bincount keys must be 1-D")
        if pred_dtypes[0] not in (DType.i32, DType.i64, DType.bool8):
            raise DTypeMismatch("bincount keys must be integers")
        if len(pred_shapes) == 2:
            if tuple(pred_shapes[1]) != tuple(ks):
                raise ShapeMismatch("bincount weights must match keys")
            return (nbins,), DType.f64, None
        return (nbins,), DType.i64, None
    raise ShapeMismatch(f"unknown op {op}")  # pragma: no cover


def _matmul_dtype(dts):
    r = np.result_type(*[d.np for d in dts])
    if r not in (np.float32, np.float64):
        raise UnsupportedDType(f"np.dot on {dts}: only f32/f64 go to the library path")
    return dtype_of(r)


# ----------------------------------------------------------------------------
# Graph
# ----------------------------------------------------------------------------


class Graph:
    """Append-only DAG with a weak node store (see module docstring)."""

    # The store maps id -> weakref.ref(node) in a plain dict (a
    # WeakValueDictionary's per-insert callback costs as much as building the
    # node); dead entries are swept every _SWEEP appends.
    _SWEEP = 4096

    def __init__(self):
        self._nodes: Dict[int, "weakref.ref[Node]"] = {}
        self._since_sweep = 0

    def _sweep(self):
        self._nodes = {k: r for k, r in self._nodes.items() if r() is not None}
        self._since_sweep = 0

    def __len__(self):
        self._sweep()
        return len(self._nodes)

    def get(self, nid: int) -> Optional[Node]:
        r = self._nodes.get(nid)
        return r() if r is not None else None

    def live_nodes(self) -> List[Node]:
        self._sweep()
        out = [self._nodes[k]() for k in sorted(self._nodes)]
        return [n for n in out if n is not None]

    def _append(self, n: Node) -> Node:
        self._nodes[n.id] = weakref.ref(n)
        self._since_sweep += 1
        if self._since_sweep >= self._SWEEP:
            self._sweep()
        return n

    def add_input(self, buf: TensorBuffer) -> Node:
        """New materialized Input node; no interning."""
        return self._append(Node(INPUT_OP, (), buf.shape, buf.dtype, data=buf))

    def add_const(self, value, dtype: DType, shape: Shape = ()) -> Node:
        """const_splat(value) of ``dtype``: value splatted into the body."""
        value = dtype.np.type(value).item()
        return self._append(Node(const_op(value), (), tuple(shape), dtype))

    def add_op(self, op: Op, preds: Sequence[Node]) -> Node:
        """Append an unmaterialized node with inferred shape/dtype.

        Inference is a pure function of (op, operand shapes, operand dtypes),
        so elementwise results are memoised: re-recording a loop body costs a
        dictionary hit per op instead of broadcasting and loop resolution."""
        if op.kind is OpKind.MAP:
            if len(preds) == 2:
                a, b = preds
                key = (op, a.shape, a.dtype, b.shape, b.dtype)
            else:
                key = (op,) + tuple([x for p in preds for x in (p.shape, p.dtype)])
            hit = _MAP_INFER.get(key)
            if hit is None:
                hit = infer(op, [p.shape for p in preds], [p.dtype for p in preds])
                if len(_MAP_INFER) > 65536:
                    _MAP_INFER.clear()
                _MAP_INFER[key] = hit
            shape, dtype, loop = hit
        else:
            shape, dtype, loop = infer(op, [p.shape for p in preds], [p.dtype for p in preds])
        return self._append(Node(op, preds, shape, dtype, loop=loop))

    @staticmethod
    def infer(op: Op, pred_shapes, pred_dtypes):
        return infer(op, pred_shapes, pred_dtypes)[:2]

    def mark_materialized(self, n: Node, buf: TensorBuffer) -> None:
        """Attach data.

        Idempotent for the same buffer; ShapeMismatch on shape/dtype mismatch;
        AlreadyMaterializedWithDifferentData when a different value arrives.
        Once materialized the node drops strong references to its predecessors.
        """
        if tuple(buf.shape) != tuple(n.shape) or buf.dtype is not n.dtype:
            raise ShapeMismatch(
                f"buffer {buf.dtype.value}{buf.shape} does not match node {n.dtype.value}{n.shape}"
            )
        if n.data is not None:
            if n.data is buf:
                return
            a, b = n.data.host, buf.host
            if a is not None and b is not None and np.array_equal(a, b, equal_nan=n.dtype.is_float):
                return
            raise AlreadyMaterializedWithDifferentData(f"node {n.id} already materialized")
        n.data = buf
        n.preds = ()

    def audit(self) -> None:
        """Re-infer every live unmaterialized node; check acyclicity."""
        for n in self.live_nodes():
            if n.kind is OpKind.INPUT:
                assert n.is_materialized
                continue
            if n.op.code is ElemCode.const_splat or not n.preds:
                continue
            for p in n.preds:
                assert p.id < n.id, "edge from an earlier to a later node"
            s, d, _ = infer(n.op, [p.shape for p in n.preds], [p.dtype for p in n.preds])
            assert s == n.shape and d is n.dtype, f"node {n} re-infers to {s} {d}"

    def dot(self) -> str:
        """DOT emission of the live DAG."""
        lines = ["digraph dag {"]
        for n in self.live_nodes():
            m = " [M]" if n.is_materialized else ""
            lines.append(f'  n{n.id} [shape=record,label="{n.id}: {n.op!r} {list(n.shape)} {n.dtype.value}{m}"];')
        for n in self.live_nodes():
            for pid in n.pred_ids:
                lines.append(f"  n{pid} -> n{n.id};")
        lines.append("}")
        return "\n".join(lines) + "\n"


def normalize_reduce_axes(axis, ndim):
    return normalize_axes(axis, ndim)


__all__ = [
    "OpKind", "ElemCode", "ReduceOp", "Op", "Node", "Graph", "infer", "arity",
    "resolve_map", "const_op", "UFUNC_OF", "CODE_OF_UFUNC", "normalize_axis",
]
