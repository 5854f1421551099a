"""session: the lazy array API, materialization triggers and fusion statistics.

Reference module ``session`` and the paper's
drop-in ``grumpy`` module:

* ``ndarray`` — "an instance of the grumpy.ndarray object represents a node in
  the DAG".  Operators, NumPy ufuncs
  (``__array_ufunc__``) and NumPy functions (``__array_function__``) record
  nodes; nothing executes at call time.  Shape and dtype
  errors surface eagerly.
* ``force`` — plan + execute the demanded region(s), cache the result
  (SPEC.md:437-445).  Triggers: ``print``/``repr``, ``tolist``, ``__array__``,
  ``item``/``float``, iteration, and storing into a NumPy array.
* unsupported operations materialize their operands and forward to NumPy
  (materialize-before-fallback); array
  results come back as grumpy arrays so the rest of the program stays lazy.
* ``SessionStats`` — kernels_executed, library_calls, nodes_materialized,
  plan/exec time.
"""

from __future__ import annotations

import builtins
import dataclasses
import numbers
import os
import time
from typing import Any, List, Optional, Sequence

import numpy as np

from . import planner as _planner
from .dag import CODE_OF_UFUNC, ElemCode, Graph, Node, Op, OpKind, ReduceOp, resolve_map
from .errors import BadAxis, DTypeMismatch, ShapeMismatch, UnsupportedDType
from .tensor import DType, TensorBuffer, dtype_of, element_count, normalize_axes, normalize_axis


# np.dot boundary (tools/gemm_probe.py): f32 GEMMs run
# as FP32 emulated with BF16x9 tensor-core products (GRUMPY_GEMM_MATH=bf16x9,
# the default: 2.4x faster than SIMT SGEMM and closer to the float64 product),
# and a GEMM feeding one `+ bias[N]` (then one `maximum(., 0)`) is planned as a
# single cuBLASLt call with a BIAS / RELU_BIAS epilogue (GRUMPY_GEMM_EPILOGUE).
GEMM_MATH = os.environ.get("GRUMPY_GEMM_MATH", "bf16x9")
GEMM_EPILOGUES = os.environ.get("GRUMPY_GEMM_EPILOGUE", "1") == "1" and GEMM_MATH == "bf16x9"


@dataclasses.dataclass
class SessionStats:
    """Fusion counters plus B200 transfer/compile counters."""

    kernels_executed: int = 0
    library_calls: int = 0
    nodes_materialized: int = 0
    collectives: int = 0
    plan_time: float = 0.0
    exec_time: float = 0.0
    compile_ms: float = 0.0
    h2d_bytes: int = 0
    d2h_bytes: int = 0
    streamed_chunks: int = 0   # chunks of streamed to_external forces (streaming.py)

    def snapshot(self):
        return dataclasses.replace(self)


class Session:
    """A deferred-evaluation session.

    planner: "region" (B200 region pass, default) or "algorithm1" (the
    reference's Algorithm 1) — both execute on the GPU.
    """

    def __init__(self, planner: str = "region", limits: Optional[_planner.PlannerLimits] = None):
        if planner not in ("region", "algorithm1"):
            raise ValueError("planner must be 'region' or 'algorithm1'")
        self.graph = Graph()
        self.stats = SessionStats()
        self.planner = planner
        self.limits = limits or _planner.PlannerLimits()
        self._executor = None
        self._consts = {}
        self._plan_cache = {}
        self._arg_operand_shape = {}
        self._shard_cache = {}
        self.comm = None  # distributed.Comm when sharded

    @property
    def executor(self):
        if self._executor is None:
            from .executor import Executor
            self._executor = Executor(self)
        return self._executor

    # -- planning ------------------------------------------------------------
    def plan(self, roots: Sequence[Node]):
        if self.planner == "algorithm1":
            steps = []
            done = set()
            for r in roots:
                for st in _planner.plan(r, self.graph, self.limits):
                    if st.root.id not in done:
                        steps.append(st)
                        done.add(st.root.id)
            return steps
        from . import codegen, codegen_rows
        return _planner.plan_regions(roots, row_fusion=codegen.row_fusable, check=codegen.check_step,
                                     epilogues=GEMM_EPILOGUES, skinny=codegen_rows.skinny_ok)

    def const(self, value, dtype: DType) -> Node:
        """Interned rank-0 const_splat node (constants are immutable)."""
        key = (type(value), value, dtype)
        n = self._consts.get(key)
        if n is None:
            if len(self._consts) > 4096:
                self._consts.clear()
            n = self.graph.add_const(value, dtype, ())
            self._consts[key] = n
        return n

    # -- materialization -----------------------------------------------------
    def force_nodes(self, nodes: Sequence[Node]):
        """Plan (or reuse a cached plan for a structurally identical DAG) and
        execute.  The plan cache turns the per-force host cost into one DAG
        traversal for iterative programs (SPEC.md:521 warm vs cold)."""
        pending = [n for n in nodes if not n.is_materialized]
        if not pending:
            return
        if self.comm is not None:
            return self._force_sharded(pending)
        t0 = time.perf_counter()
        key, order = _planner.dag_signature(pending)
        tmpl = self._plan_cache.get(key)
        if tmpl is None:
            steps = self.plan(pending)
            tmpl = _planner.make_template(steps, order)
            if len(self._plan_cache) > 1024:
                self._plan_cache.clear()
            self._plan_cache[key] = tmpl
        else:
            steps = _planner.instantiate(tmpl, order)
        t1 = time.perf_counter()
        self.stats.plan_time += t1 - t0
        self.executor.run(steps)
        self.stats.exec_time += time.perf_counter() - t1

    def _force_sharded(self, pending):
        """Leading-axis sharded execution (distributed.py): partial nodes become
        step roots and are allreduced after their kernel; arg-reductions over
        the sharded axis are combined from (value, global index) pairs.

        Plans are cached like unsharded ones, keyed by the DAG signature plus
        the distribution of its materialized leaves, so an iterative sharded
        program pays one classification and one region pass per structure."""
        from . import distributed as D
        t0 = time.perf_counter()
        key, order = _planner.dag_signature(pending)
        leafdist = tuple(D.leaf_dist(n) for n in order if n.is_materialized)
        ckey = (key, leafdist)
        hit = self._shard_cache.get(ckey)
        if hit is None:
            dist = D.classify(pending)
            partial = [n for n in order if not n.is_materialized and dist.get(n.id, "R")[0] in "PA"]
        else:
            tmpl, partial_idx, tags = hit
            partial = [order[i] for i in partial_idx]
        aux = {}
        for n in partial:
            if n.op.kind is OpKind.ARGREDUCE:
                info = D.shard_of(n.preds[0])
                self._arg_operand_shape[n.id] = (n.preds[0].shape, info[1] if info else 0)
                which, axis, keepdims = n.op.attrs
                x = n.preds[0]
                axes = tuple(range(len(x.shape))) if axis is None else (axis,)
                rop = ReduceOp.max if which == "max" else ReduceOp.min
                aux[n.id] = self.graph.add_op(Op(OpKind.REDUCE, None, (rop, axes, bool(keepdims), None)), [x])
        roots = list(dict((n.id, n) for n in list(pending) + partial + list(aux.values())).values())
        _k2, order2 = _planner.dag_signature(roots)
        if hit is None:
            steps = self.plan(roots)
            idx = {n.id: i for i, n in enumerate(order)}
            tags = tuple(dist.get(n.id, "R") for n in order2)
            if len(self._shard_cache) > 256:
                self._shard_cache.clear()
            self._shard_cache[ckey] = (_planner.make_template(steps, order2), [idx[n.id] for n in partial], tags)
        else:
            steps = _planner.instantiate(tmpl, order2)
            dist = {n.id: t for n, t in zip(order2, tags)}
        self.stats.plan_time += time.perf_counter() - t0
        t1 = time.perf_counter()
        self.executor.run(steps, dist=dist, comm=self.comm)
        for n in partial:
            if n.op.kind is OpKind.ARGREDUCE:
                self._combine_arg(n, aux[n.id], "max" if n.op.attrs[0] == "max" else "min")
            n.dist = "R"
        self.stats.exec_time += time.perf_counter() - t1

    def _combine_arg(self, n, aux, which):
        """Global first-index arg-reduction from every rank's (best value,
        local index), on the device: the local index is offset to a global
        one, both are gathered over the ranks (ncclAllGather), and an
        arg-reduction over the rank axis picks the winning rank per element —
        ranks hold consecutive rows, so the lowest rank among equal values
        (and the first NaN) is NumPy's first index."""
        from .tensor import TensorBuffer as _TB
        src_shape, off_rows = self._arg_operand_shape[n.id]
        offset = off_rows * int(np.prod(src_shape[1:])) if n.op.attrs[1] is None else off_rows
        comm = self.comm
        world = comm.world
        count = int(np.prod(n.shape)) if n.shape else 1
        gidx = ndarray(n, self) + np.int64(offset)
        self.force_nodes([gidx._node])
        rt = self.executor.rt
        gv = comm.allgather_device(rt, aux.data.device, count, aux.dtype)
        gi = comm.allgather_device(rt, gidx._node.data.device, count, DType.i64)
        self.stats.collectives += 2
        V = ndarray(self.graph.add_input(_TB(aux.dtype, (world,) + tuple(n.shape), device=gv)), self)
        I = ndarray(self.graph.add_input(_TB(DType.i64, (world,) + tuple(n.shape), device=gi)), self)
        win = V.argmax(axis=0) if which == "max" else V.argmin(axis=0)
        res = I[0] * (win == 0)
        for k in range(1, world):
            res = res + I[k] * (win == k)
        self.force_nodes([res._node])
        n.data.device = res._node.data.device
        n.data.host = None

    def to_numpy(self, node: Node) -> np.ndarray:
        self.force_nodes([node])
        buf = node.data
        if buf.host is None:
            buf.host = buf.device.to_numpy(buf.dtype, buf.shape)
            self.stats.d2h_bytes += buf.host.nbytes
        return buf.host


_default = Session()


def default_session() -> Session:
    return _default


def set_default_session(s: Session) -> Session:
    global _default
    old = _default
    _default = s
    return old


# ---------------------------------------------------------------------------
# Operand conversion
# ---------------------------------------------------------------------------


def _is_weak_scalar(x):
    return isinstance(x, (bool, int, float)) and not isinstance(x, np.generic)


def _input_node(arr: np.ndarray, sess: Session) -> Node:
    return sess.graph.add_input(TensorBuffer.from_numpy(arr))


def _as_node(x, sess: Session) -> Node:
    if isinstance(x, ndarray):
        return x._node
    if isinstance(x, np.ndarray) and x.ndim > 0:
        return _input_node(x, sess)
    if isinstance(x, (np.ndarray, np.generic)):
        a = np.asarray(x)
        return sess.graph.add_const(a.item(), dtype_of(a.dtype), ())
    if _is_weak_scalar(x):
        dt = DType.bool8 if isinstance(x, bool) else DType.i64 if isinstance(x, int) else DType.f64
        return sess.graph.add_const(x, dt, ())
    return _input_node(np.asarray(x), sess)


def _wrap(node: Node, sess: Session) -> "ndarray":
    return ndarray(node, sess)


def _dt_arg(x):
    """dtype argument for loop resolution: DType for arrays/strong scalars,
    the Python type for weak scalars (NEP 50)."""
    if isinstance(x, ndarray):
        return x._node.dtype
    if _is_weak_scalar(x):
        return bool if isinstance(x, bool) else int if isinstance(x, int) else float
    a = np.asarray(x)
    return dtype_of(a.dtype)


def _check_int_range(v, dt: DType):
    if isinstance(v, int) and not isinstance(v, bool) and dt.is_int:
        info = np.iinfo(dt.np)
        if v < info.min or v > info.max:
            raise OverflowError(f"Python integer {v} out of bounds for {dt.np}")


_MAP_OPS = {c: Op(OpKind.MAP, c) for c in ElemCode}
_WEAK = {float: float, int: int, bool: DType.bool8}


def elementwise(code: ElemCode, *args, sess: Optional[Session] = None) -> "ndarray":
    """Record MapElementwise(code) with NumPy's ufunc type resolution.

    Hot path of recording: weak Python scalars (NEP 50) resolve with their
    Python type and become const_splat nodes of the loop dtype."""
    if sess is None:
        sess = _session_of(args)
    dts = []
    for a in args:
        t = type(a)
        if t is ndarray:
            dts.append(a._node.dtype)
        elif t in _WEAK:
            dts.append(_WEAK[t])
        else:
            d = _dt_arg(a)
            dts.append(DType.bool8 if d is bool else d)
    loop, out = resolve_map(code, dts)
    preds = []
    g = sess.graph
    for a, lt in zip(args, loop):
        t = type(a)
        if t is ndarray:
            preds.append(a._node)
        elif t in _WEAK:
            if t is int:
                _check_int_range(a, lt)
            preds.append(sess.const(a, lt))
        else:
            preds.append(_as_node(a, sess))
    return ndarray(g.add_op(_MAP_OPS[code], preds), sess)


def _session_of(args) -> Session:
    for a in args:
        if isinstance(a, ndarray):
            return a._session
    return _default


# ---------------------------------------------------------------------------
# The lazy array proxy
# ---------------------------------------------------------------------------


def _binop(code, swap=False):
    op = _MAP_OPS[code]

    def f(self, other):
        t = type(other)
        if t is ndarray and other._session is self._session:
            # hot path: two lazy arrays of one session
            a, b = (other._node, self._node) if swap else (self._node, other._node)
            return ndarray(self._session.graph.add_op(op, (a, b)), self._session)
        if t is float and self._node.dtype.is_float:
            # float scalar with a float array: NEP 50 keeps the array's dtype
            sess = self._session
            c = sess.const(other, self._node.dtype)
            a, b = (c, self._node) if swap else (self._node, c)
            return ndarray(sess.graph.add_op(op, (a, b)), sess)
        if isinstance(other, (list, tuple)):
            other = np.asarray(other)
        if not isinstance(other, (ndarray, np.ndarray, np.generic, numbers.Number)):
            return NotImplemented
        return elementwise(code, other, self) if swap else elementwise(code, self, other)
    return f


class ndarray:
    """grumpy.ndarray — a lazy proxy for one DAG node."""

    __slots__ = ("_node", "_session", "__weakref__")
    __array_priority__ = 1000

    def __init__(self, node: Node, session: Optional[Session] = None):
        self._node = node
        self._session = session or _default

    # -- metadata (no forcing) -------------------------------------------------
    @property
    def shape(self):
        return self._node.shape

    @property
    def dtype(self):
        return self._node.dtype.np

    @property
    def ndim(self):
        return len(self._node.shape)

    @property
    def size(self):
        return element_count(self._node.shape)

    @property
    def nbytes(self):
        return self.size * self._node.dtype.itemsize

    @property
    def node(self) -> Node:
        return self._node

    @property
    def is_materialized(self) -> bool:
        return self._node.is_materialized

    def __len__(self):
        if not self._node.shape:
            raise TypeError("len() of unsized object")
        return self._node.shape[0]

    # -- materialization triggers ------------------------------------------------
    def force(self) -> "ndarray":
        self._session.force_nodes([self._node])
        return self

    def numpy(self, out: Optional[np.ndarray] = None) -> np.ndarray:
        """Materialize and return host data; with ``out`` (e.g. a page-locked
        array) the device->host copy lands there directly."""
        if out is None:
            return self._session.to_numpy(self._node)
        self._session.force_nodes([self._node])
        buf = self._node.data
        if out.shape != self.shape or out.dtype != self.dtype or not out.flags.c_contiguous:
            raise ShapeMismatch("out must be a C-contiguous array of the same shape and dtype")
        if buf.host is not None:
            out[...] = buf.host
        else:
            buf.device.copy_to_host(out)
            self._session.stats.d2h_bytes += out.nbytes
        return out

    def __array__(self, dtype=None, copy=None):
        a = self.numpy()
        if dtype is not None and np.dtype(dtype) != a.dtype:
            return a.astype(dtype)
        if copy:
            return a.copy()
        return a

    def tolist(self):
        return self.numpy().tolist()

    def item(self, *args):
        return self.numpy().item(*args)

    def __float__(self):
        return float(self.numpy())

    def __int__(self):
        return int(self.numpy())

    def __index__(self):
        return int(self.numpy().__index__())

    def __bool__(self):
        return bool(self.numpy())

    def __complex__(self):
        return complex(self.numpy())

    def __iter__(self):
        if not self.shape:
            raise TypeError("iteration over a 0-d array")
        for i in range(self.shape[0]):
            yield self[i]

    def __repr__(self):
        return "grumpy." + repr(self.numpy())

    def __str__(self):
        return str(self.numpy())

    def __format__(self, spec):
        return format(self.numpy(), spec)

    # -- arithmetic ----------------------------------------------------------------
    __add__ = _binop(ElemCode.add)
    __radd__ = _binop(ElemCode.add, swap=True)
    __sub__ = _binop(ElemCode.sub)
    __rsub__ = _binop(ElemCode.sub, swap=True)
    __mul__ = _binop(ElemCode.mul)
    __rmul__ = _binop(ElemCode.mul, swap=True)
    __truediv__ = _binop(ElemCode.div)
    __rtruediv__ = _binop(ElemCode.div, swap=True)
    __floordiv__ = _binop(ElemCode.floordiv)
    __rfloordiv__ = _binop(ElemCode.floordiv, swap=True)
    __mod__ = _binop(ElemCode.mod)
    __rmod__ = _binop(ElemCode.mod, swap=True)
    __rpow__ = _binop(ElemCode.pow, swap=True)
    __lt__ = _binop(ElemCode.cmp_lt)
    __gt__ = _binop(ElemCode.cmp_gt)
    __le__ = _binop(ElemCode.cmp_le)
    __ge__ = _binop(ElemCode.cmp_ge)
    __eq__ = _binop(ElemCode.cmp_eq)
    __ne__ = _binop(ElemCode.cmp_ne)
    __and__ = _binop(ElemCode.logical_and)
    __rand__ = _binop(ElemCode.logical_and, swap=True)
    __or__ = _binop(ElemCode.logical_or)
    __ror__ = _binop(ElemCode.logical_or, swap=True)
    __xor__ = _binop(ElemCode.logical_xor)
    __rxor__ = _binop(ElemCode.logical_xor, swap=True)
    __hash__ = None

    def __pow__(self, other):
        # NumPy's array_power fast path: x**2 -> square, x**0.5 -> sqrt
        if _is_weak_scalar(other) and not isinstance(other, bool):
            if other == 2:
                return elementwise(ElemCode.square, self)
            if other == 0.5 and self._node.dtype.is_float:
                return elementwise(ElemCode.sqrt, self)
            if other == 1 and self._node.dtype.is_float:
                return self.copy()
        return elementwise(ElemCode.pow, self, other)

    def __neg__(self):
        return elementwise(ElemCode.neg, self)

    def __pos__(self):
        return self.copy()

    def __abs__(self):
        return elementwise(ElemCode.abs, self)

    def __invert__(self):
        if self._node.dtype is DType.bool8:
            return elementwise(ElemCode.logical_not, self)
        raise DTypeMismatch("bitwise invert is only supported for bool arrays")

    def __matmul__(self, other):
        return dot(self, other)

    def __rmatmul__(self, other):
        return dot(other, self)

    # -- views / shape ops --------------------------------------------------------
    def _view(self, op: Op) -> "ndarray":
        return _wrap(self._session.graph.add_op(op, [self._node]), self._session)

    def reshape(self, *shape, order="C"):
        if order != "C":
            return _fallback_method(self, "reshape", *shape, order=order)
        if len(shape) == 1 and isinstance(shape[0], (tuple, list)):
            shape = tuple(shape[0])
        shape = tuple(int(s) for s in shape)
        if shape.count(-1) > 1:
            raise ShapeMismatch("can only specify one unknown dimension")
        if -1 in shape:
            known = element_count([s for s in shape if s != -1])
            if known == 0 or self.size % known:
                raise ShapeMismatch(f"cannot reshape {self.shape} into {shape}")
            shape = tuple(self.size // known if s == -1 else s for s in shape)
        if shape == self.shape:
            return self
        return self._view(Op(OpKind.RESHAPE, None, (shape,)))

    def ravel(self):
        return self.reshape(-1)

    flatten = ravel

    def transpose(self, *axes):
        if not axes or axes == (None,):
            perm = tuple(reversed(range(self.ndim)))
        else:
            if len(axes) == 1 and isinstance(axes[0], (tuple, list)):
                axes = tuple(axes[0])
            perm = tuple(normalize_axis(a, self.ndim) for a in axes)
        if perm == tuple(range(self.ndim)):
            return self
        return self._view(Op(OpKind.TRANSPOSE, None, (perm,)))

    @property
    def T(self):
        return self.transpose()

    def astype(self, dtype, copy=True):
        dt = dtype_of(dtype)
        if dt is self._node.dtype and not copy:
            return self
        return self._view(Op(OpKind.CAST, None, (dt,)))

    def copy(self):
        return self._view(Op(OpKind.CAST, None, (self._node.dtype,)))

    def squeeze(self, axis=None):
        if axis is None:
            shape = tuple(s for s in self.shape if s != 1)
        else:
            axes = normalize_axes(axis, self.ndim)
            for a in axes:
                if self.shape[a] != 1:
                    raise ShapeMismatch("cannot select an axis to squeeze out which has size not equal to one")
            shape = tuple(s for i, s in enumerate(self.shape) if i not in axes)
        return self.reshape(shape)

    def __getitem__(self, key):
        return _getitem(self, key)

    def __setitem__(self, key, value):
        _setitem(self, key, value)

    # -- reductions ---------------------------------------------------------------
    def sum(self, axis=None, dtype=None, out=None, keepdims=False):
        return _reduce(self, ReduceOp.sum, axis, dtype, keepdims)

    def prod(self, axis=None, dtype=None, out=None, keepdims=False):
        return _reduce(self, ReduceOp.prod, axis, dtype, keepdims)

    def max(self, axis=None, out=None, keepdims=False):
        return _reduce(self, ReduceOp.max, axis, None, keepdims)

    def min(self, axis=None, out=None, keepdims=False):
        return _reduce(self, ReduceOp.min, axis, None, keepdims)

    def mean(self, axis=None, dtype=None, out=None, keepdims=False):
        return _mean(self, axis, dtype, keepdims)

    def var(self, axis=None, dtype=None, out=None, ddof=0, keepdims=False):
        return _var(self, axis, dtype, ddof, keepdims)

    def std(self, axis=None, dtype=None, out=None, ddof=0, keepdims=False):
        return elementwise(ElemCode.sqrt, _var(self, axis, dtype, ddof, keepdims))

    def argmax(self, axis=None, out=None, keepdims=False):
        return _argreduce(self, "max", axis, keepdims)

    def argmin(self, axis=None, out=None, keepdims=False):
        return _argreduce(self, "min", axis, keepdims)

    def cumsum(self, axis=None, dtype=None, out=None):
        return _scan(self, ReduceOp.sum, axis, dtype)

    def cumprod(self, axis=None, dtype=None, out=None):
        return _scan(self, ReduceOp.prod, axis, dtype)

    def any(self, axis=None, out=None, keepdims=False):
        b = self if self._node.dtype is DType.bool8 else self.astype(np.bool_)
        return _reduce(b, ReduceOp.max, axis, None, keepdims)

    def all(self, axis=None, out=None, keepdims=False):
        b = self if self._node.dtype is DType.bool8 else self.astype(np.bool_)
        return _reduce(b, ReduceOp.min, axis, None, keepdims)

    def clip(self, a_min=None, a_max=None):
        r = self
        if a_min is not None:
            r = elementwise(ElemCode.maximum, r, a_min)
        if a_max is not None:
            r = elementwise(ElemCode.minimum, r, a_max)
        return r

    def dot(self, other):
        return dot(self, other)

    # -- NumPy protocol hooks ----------------------------------------------------------
    def __array_ufunc__(self, ufunc, method, *inputs, **kwargs):
        name = ufunc.__name__
        if method == "__call__" and not kwargs:
            if name == "matmul":
                return dot(*inputs)
            if name in ("positive",):
                return _as_array(inputs[0]).copy()
            if name == "power" and len(inputs) == 2 and isinstance(inputs[0], ndarray):
                return inputs[0].__pow__(inputs[1])
            code = CODE_OF_UFUNC.get(name)
            if code is not None and len(inputs) == _nin(code):
                try:
                    return elementwise(code, *inputs)
                except (DTypeMismatch, UnsupportedDType):
                    pass
        if method == "reduce" and name in ("add", "multiply", "maximum", "minimum", "logical_or", "logical_and"):
            allowed = {"axis", "keepdims", "dtype"}
            if set(kwargs) <= allowed and len(inputs) == 1:
                rop = {"add": ReduceOp.sum, "multiply": ReduceOp.prod, "maximum": ReduceOp.max,
                       "minimum": ReduceOp.min, "logical_or": ReduceOp.max, "logical_and": ReduceOp.min}[name]
                x = _as_array(inputs[0])
                if name.startswith("logical") and x._node.dtype is not DType.bool8:
                    x = x.astype(np.bool_)
                return _reduce(x, rop, kwargs.get("axis", 0), kwargs.get("dtype"), kwargs.get("keepdims", False))
        if method == "accumulate" and name in ("add", "multiply", "maximum", "minimum") and set(kwargs) <= {"axis", "dtype"}:
            rop = {"add": ReduceOp.sum, "multiply": ReduceOp.prod, "maximum": ReduceOp.max,
                   "minimum": ReduceOp.min}[name]
            return _scan(_as_array(inputs[0]), rop, kwargs.get("axis", 0), kwargs.get("dtype"))
        return _fallback(getattr(ufunc, method), inputs, kwargs)

    def __array_function__(self, func, types, args, kwargs):
        impl = _FUNCS.get(func)
        if impl is not None:
            try:
                return impl(*args, **kwargs)
            except TypeError:
                pass
        return _fallback(func, args, kwargs)


def _nin(code):
    from .dag import arity
    return arity(code)


def _as_array(x, sess: Optional[Session] = None) -> ndarray:
    if isinstance(x, ndarray):
        return x
    sess = sess or _default
    return _wrap(_as_node(x, sess), sess)


# ---------------------------------------------------------------------------
# Fallback (materialize-before-fallback)
# ---------------------------------------------------------------------------


def _to_np(x):
    if isinstance(x, ndarray):
        return x.numpy()
    if isinstance(x, (list, tuple)):
        return type(x)(_to_np(y) for y in x)
    if isinstance(x, dict):
        return {k: _to_np(v) for k, v in x.items()}
    return x


def _from_np(x, sess):
    if isinstance(x, np.ndarray) and x.ndim > 0:
        try:
            dtype_of(x.dtype)
        except UnsupportedDType:
            return x
        return _wrap(_input_node(x, sess), sess)
    if isinstance(x, tuple):
        return tuple(_from_np(y, sess) for y in x)
    if isinstance(x, list):
        return [_from_np(y, sess) for y in x]
    return x


def _fallback(func, args, kwargs):
    sess = _session_of(list(args) + list(kwargs.values()))
    res = func(*_to_np(args), **_to_np(kwargs))
    return _from_np(res, sess)


def _fallback_method(a: ndarray, name, *args, **kwargs):
    res = getattr(a.numpy(), name)(*_to_np(args), **_to_np(kwargs))
    return _from_np(res, a._session)


# ---------------------------------------------------------------------------
# Reductions, scans, arg-reductions
# ---------------------------------------------------------------------------


def _reduce(a, rop: ReduceOp, axis, dtype, keepdims) -> ndarray:
    a = _as_array(a)
    axes = normalize_axes(axis, a.ndim)
    odt = None
    x = a
    if dtype is not None:
        odt = dtype_of(dtype)
        if odt is not a._node.dtype:
            x = a.astype(odt)
    g = a._session.graph
    return _wrap(g.add_op(Op(OpKind.REDUCE, None, (rop, axes, bool(keepdims), odt)), [x._node]), a._session)


def _count(a: ndarray, axes) -> int:
    """Number of reduced elements; the sharded leading axis counts globally."""
    n = 1
    glob = None
    if 0 in axes and a._session.comm is not None:
        from . import distributed as D
        if D.classify([a._node]).get(a._node.id) == "S":
            info = D.shard_of(a._node)
            glob = info[0] if info else None
    for ax in axes:
        n *= glob if (ax == 0 and glob is not None) else a.shape[ax]
    return n


def _acc_dtype(a: ndarray, dtype):
    if dtype is not None:
        return dtype_of(dtype)
    if a._node.dtype in (DType.i32, DType.i64, DType.bool8):
        return DType.f64
    return None


def _mean(a, axis, dtype, keepdims) -> ndarray:
    """NumPy _mean: add.reduce (dtype f64 for ints) then true_divide by count."""
    a = _as_array(a)
    axes = normalize_axes(axis, a.ndim)
    acc = _acc_dtype(a, dtype)
    s = _reduce(a, ReduceOp.sum, axes, acc, keepdims)
    return elementwise(ElemCode.div, s, _count(a, axes))


def _var(a, axis, dtype, ddof, keepdims) -> ndarray:
    """NumPy _var: mean with keepdims, x - mean, x*x, add.reduce, / (n - ddof)."""
    a = _as_array(a)
    axes = normalize_axes(axis, a.ndim)
    acc = _acc_dtype(a, dtype)
    n = _count(a, axes)
    m = elementwise(ElemCode.div, _reduce(a, ReduceOp.sum, axes, acc, True), n)
    d = a - m
    sq = elementwise(ElemCode.mul, d, d)
    s = _reduce(sq, ReduceOp.sum, axes, acc if acc is not None and acc is not sq._node.dtype else None, keepdims)
    return elementwise(ElemCode.div, s, builtins.max(n - ddof, 0))


def _argreduce(a, which, axis, keepdims) -> ndarray:
    a = _as_array(a)
    ax = None if axis is None else normalize_axis(axis, a.ndim)
    g = a._session.graph
    return _wrap(g.add_op(Op(OpKind.ARGREDUCE, None, (which, ax, bool(keepdims))), [a._node]), a._session)


def _scan(a, rop, axis, dtype) -> ndarray:
    a = _as_array(a)
    ax = None if axis is None else normalize_axis(axis, a.ndim)
    odt = dtype_of(dtype) if dtype is not None else None
    x = a if odt is None or odt is a._node.dtype else a.astype(odt)
    g = a._session.graph
    return _wrap(g.add_op(Op(OpKind.SCAN, None, (rop, ax, odt)), [x._node]), a._session)


# ---------------------------------------------------------------------------
# Indexing
# ---------------------------------------------------------------------------


def _parse_key(shape, key, allow_newaxis=True):
    """Basic indexing → (per-dim (start, step, length) , output shape, int dims).

    Returns None when the key needs advanced indexing (fallback)."""
    if not isinstance(key, tuple):
        key = (key,)
    n_ell = sum(1 for k in key if k is Ellipsis)
    if n_ell > 1:
        raise IndexError("an index can only have a single ellipsis")
    for k in key:
        if not (k is None or k is Ellipsis or isinstance(k, (slice, numbers.Integral))):
            return None
        if isinstance(k, (bool, np.bool_)):
            return None
    n_real = sum(1 for k in key if k is not None and k is not Ellipsis)
    if n_real > len(shape):
        raise IndexError(f"too many indices for array: array is {len(shape)}-dimensional, but {n_real} were indexed")
    if n_ell == 0:
        key = key + (Ellipsis,)
    spec = []
    out_shape = []
    d = 0
    for k in key:
        if k is Ellipsis:
            fill = len(shape) - n_real
            for _ in range(fill):
                spec.append((0, 1, shape[d]))
                out_shape.append(shape[d])
                d += 1
        elif k is None:
            if not allow_newaxis:
                return None
            out_shape.append(1)
        elif isinstance(k, slice):
            start, stop, step = k.indices(shape[d])
            length = len(range(start, stop, step))
            spec.append((start if length else 0, step, length))
            out_shape.append(length)
            d += 1
        else:
            i = int(k)
            if i < -shape[d] or i >= shape[d]:
                raise IndexError(f"index {i} is out of bounds for axis {d} with size {shape[d]}")
            if i < 0:
                i += shape[d]
            spec.append((i, 1, 1))
            d += 1
    return tuple(spec), tuple(out_shape)


def _getitem(a: ndarray, key):
    if isinstance(key, ndarray) or isinstance(key, (list, np.ndarray)):
        return _fallback_method(a, "__getitem__", key)
    parsed = _parse_key(a.shape, key)
    if parsed is None:
        return _fallback_method(a, "__getitem__", key)
    spec, out_shape = parsed
    x = a
    if any(s != (0, 1, ext) for s, ext in zip(spec, a.shape)):
        x = a._view(Op(OpKind.SLICE, None, (spec,)))
    if tuple(out_shape) != x.shape:
        x = x._view(Op(OpKind.RESHAPE, None, (tuple(out_shape),)))
    return x


def _setitem(a: ndarray, key, value):
    """Functional SliceAssign; the proxy is rebound to the new node."""
    parsed = _parse_key(a.shape, key, allow_newaxis=False)
    if parsed is None:
        raise IndexError("grumpy supports slice assignment with basic indices only")
    spec, _ = parsed
    v = value if isinstance(value, ndarray) else _as_array(value, a._session)
    if v._node.dtype is not a._node.dtype:
        v = v.astype(a.dtype)
    g = a._session.graph
    a._node = g.add_op(Op(OpKind.SLICE_ASSIGN, None, (spec,)), [a._node, v._node])


# ---------------------------------------------------------------------------
# Library ops
# ---------------------------------------------------------------------------


def dot(a, b) -> ndarray:
    """np.dot / matmul rank dispatch: (2,2) MatMul, (2,1) MatVec,
    (1,2) vector-matrix MatVec; (1,1) inner product as a map-reduce."""
    sess = _session_of([a, b])
    a = _as_array(a, sess)
    b = _as_array(b, sess)
    rt = np.result_type(a.dtype, b.dtype)
    if a.ndim == 1 and b.ndim == 1:
        if a.shape != b.shape:
            raise ShapeMismatch(f"shapes {a.shape} and {b.shape} not aligned")
        return _reduce(a * b, ReduceOp.sum, None, None, False)
    if rt not in (np.float32, np.float64):
        return _fallback(np.dot, (a, b), {})
    if a.dtype != rt:
        a = a.astype(rt)
    if b.dtype != rt:
        b = b.astype(rt)
    g = sess.graph
    if a.ndim == 2 and b.ndim == 2:
        return _wrap(g.add_op(Op(OpKind.MATMUL), [a._node, b._node]), sess)
    if a.ndim == 2 and b.ndim == 1:
        return _wrap(g.add_op(Op(OpKind.MATVEC, None, (False,)), [a._node, b._node]), sess)
    if a.ndim == 1 and b.ndim == 2:
        return _wrap(g.add_op(Op(OpKind.MATVEC, None, (True,)), [b._node, a._node]), sess)
    return _fallback(np.dot, (a, b), {})


def bincount(x, weights=None, minlength=0) -> ndarray:
    """np.bincount with a static length: keys must lie in [0, minlength)."""
    sess = _session_of([x, weights])
    x = _as_array(x, sess)
    if minlength <= 0:
        return _fallback(np.bincount, (x,), {"weights": weights, "minlength": minlength})
    preds = [x._node]
    if weights is not None:
        w = _as_array(weights, sess)
        if w._node.dtype is not DType.f64:
            w = w.astype(np.float64)
        preds.append(w._node)
    return _wrap(sess.graph.add_op(Op(OpKind.KEYED_SUM, None, (int(minlength),)), preds), sess)


def where(cond, x=None, y=None):
    if x is None and y is None:
        return _fallback(np.where, (cond,), {})
    sess = _session_of([cond, x, y])
    c = _as_array(cond, sess)
    if c._node.dtype is not DType.bool8:
        c = c.astype(np.bool_)
    return elementwise(ElemCode.select, c, x, y, sess=sess)


# ---------------------------------------------------------------------------
# NumPy function table for __array_function__
# ---------------------------------------------------------------------------


def _f_sum(a, axis=None, dtype=None, out=None, keepdims=False, **kw):
    if out is not None or kw:
        raise TypeError
    return _as_array(a).sum(axis=axis, dtype=dtype, keepdims=keepdims)


def _f_mean(a, axis=None, dtype=None, out=None, keepdims=False, **kw):
    if out is not None or kw:
        raise TypeError
    return _mean(a, axis, dtype, keepdims)


def _f_std(a, axis=None, dtype=None, out=None, ddof=0, keepdims=False, **kw):
    if out is not None or kw:
        raise TypeError
    return _as_array(a).std(axis=axis, dtype=dtype, ddof=ddof, keepdims=keepdims)


def _f_var(a, axis=None, dtype=None, out=None, ddof=0, keepdims=False, **kw):
    if out is not None or kw:
        raise TypeError
    return _var(a, axis, dtype, ddof, keepdims)


def _f_max(a, axis=None, out=None, keepdims=False, **kw):
    if out is not None or kw:
        raise TypeError
    return _reduce(a, ReduceOp.max, axis, None, keepdims)


def _f_min(a, axis=None, out=None, keepdims=False, **kw):
    if out is not None or kw:
        raise TypeError
    return _reduce(a, ReduceOp.min, axis, None, keepdims)


def _f_prod(a, axis=None, dtype=None, out=None, keepdims=False, **kw):
    if out is not None or kw:
        raise TypeError
    return _reduce(a, ReduceOp.prod, axis, dtype, keepdims)


def _f_argmax(a, axis=None, out=None, keepdims=False):
    if out is not None:
        raise TypeError
    return _argreduce(a, "max", axis, keepdims)


def _f_argmin(a, axis=None, out=None, keepdims=False):
    if out is not None:
        raise TypeError
    return _argreduce(a, "min", axis, keepdims)


def _f_cumsum(a, axis=None, dtype=None, out=None):
    if out is not None:
        raise TypeError
    return _scan(_as_array(a), ReduceOp.sum, axis, dtype)


def _f_transpose(a, axes=None):
    return _as_array(a).transpose(*(axes or ()))


def _f_reshape(a, shape=None, order="C", **kw):
    if "newshape" in kw:
        shape = kw.pop("newshape")
    if kw or order != "C":
        raise TypeError
    return _as_array(a).reshape(shape)


def _f_broadcast_to(a, shape, subok=False):
    a = _as_array(a)
    shape = tuple(shape)
    if shape == a.shape:
        return a
    return a._view(Op(OpKind.BROADCAST, None, (shape,)))


def _f_expand_dims(a, axis):
    a = _as_array(a)
    axes = axis if isinstance(axis, (tuple, list)) else (axis,)
    nd = a.ndim + len(axes)
    axes = sorted(normalize_axis(x, nd) for x in axes)
    shape = list(a.shape)
    for ax in axes:
        shape.insert(ax, 1)
    return a.reshape(tuple(shape))


def _f_squeeze(a, axis=None):
    return _as_array(a).squeeze(axis)


def _f_clip(a, a_min=None, a_max=None, out=None, **kw):
    if out is not None or kw:
        raise TypeError
    return _as_array(a).clip(a_min, a_max)


def _f_where(cond, x=None, y=None):
    return where(cond, x, y)


def _f_dot(a, b, out=None):
    if out is not None:
        raise TypeError
    return dot(a, b)


def _f_copy(a, order="K", subok=False):
    return _as_array(a).copy()


def _f_ravel(a, order="C"):
    if order != "C":
        raise TypeError
    return _as_array(a).ravel()


def _f_bincount(x, weights=None, minlength=0):
    return bincount(x, weights, minlength)


def _f_any(a, axis=None, out=None, keepdims=False, **kw):
    if out is not None or kw:
        raise TypeError
    return _as_array(a).any(axis=axis, keepdims=keepdims)


def _f_all(a, axis=None, out=None, keepdims=False, **kw):
    if out is not None or kw:
        raise TypeError
    return _as_array(a).all(axis=axis, keepdims=keepdims)


def _f_shape(a):
    return _as_array(a).shape


def _f_ndim(a):
    return _as_array(a).ndim


def _f_size(a, axis=None):
    a = _as_array(a)
    return a.size if axis is None else a.shape[axis]


def _f_astype(x, dtype, copy=True, **kw):
    return _as_array(x).astype(dtype)


_FUNCS = {
    np.sum: _f_sum, np.mean: _f_mean, np.std: _f_std, np.var: _f_var,
    np.max: _f_max, np.amax: _f_max, np.min: _f_min, np.amin: _f_min, np.prod: _f_prod,
    np.argmax: _f_argmax, np.argmin: _f_argmin, np.cumsum: _f_cumsum,
    np.transpose: _f_transpose, np.reshape: _f_reshape, np.broadcast_to: _f_broadcast_to,
    np.expand_dims: _f_expand_dims, np.squeeze: _f_squeeze, np.clip: _f_clip,
    np.where: _f_where, np.dot: _f_dot, np.copy: _f_copy, np.ravel: _f_ravel,
    np.bincount: _f_bincount, np.any: _f_any, np.all: _f_all, np.shape: _f_shape,
    np.ndim: _f_ndim, np.size: _f_size, np.astype: _f_astype,
}


# ---------------------------------------------------------------------------
# Module-level constructors and forcing
# ---------------------------------------------------------------------------


def asarray(x, dtype=None, session: Optional[Session] = None) -> ndarray:
    """Wrap host data as a materialized Input node; the H2D copy
    happens when a kernel first reads it."""
    sess = session or _default
    if isinstance(x, ndarray):
        return x if dtype is None else x.astype(dtype, copy=False)
    arr = np.asarray(x, dtype=dtype)
    if arr.dtype == np.float16:
        raise UnsupportedDType("float16")
    if arr.dtype.kind == "i" and arr.dtype not in (np.int32, np.int64):
        arr = arr.astype(np.int64)
    if arr.dtype.kind == "u":
        arr = arr.astype(np.int64)
    return _wrap(_input_node(arr, sess), sess)


def array(x, dtype=None, copy=True, session: Optional[Session] = None) -> ndarray:
    if isinstance(x, ndarray):
        return x.astype(dtype or x.dtype)
    arr = np.array(x, dtype=dtype, copy=copy)
    return asarray(arr, session=session)


def full(shape, fill_value, dtype=None, session: Optional[Session] = None) -> ndarray:
    sess = session or _default
    if isinstance(shape, numbers.Integral):
        shape = (int(shape),)
    shape = tuple(int(s) for s in shape)
    if dtype is None:
        dtype = np.asarray(fill_value).dtype
    dt = dtype_of(dtype)
    return _wrap(sess.graph.add_const(fill_value, dt, shape), sess)


def zeros(shape, dtype=np.float64, session=None) -> ndarray:
    return full(shape, 0, dtype, session)


def ones(shape, dtype=np.float64, session=None) -> ndarray:
    return full(shape, 1, dtype, session)


def empty(shape, dtype=np.float64, session=None) -> ndarray:
    return full(shape, 0, dtype, session)


def zeros_like(a, dtype=None):
    a = _as_array(a)
    return full(a.shape, 0, dtype or a.dtype, a._session)


def ones_like(a, dtype=None):
    a = _as_array(a)
    return full(a.shape, 1, dtype or a.dtype, a._session)


def full_like(a, fill_value, dtype=None):
    a = _as_array(a)
    return full(a.shape, fill_value, dtype or a.dtype, a._session)


def force(*arrays: ndarray):
    """Materialize several arrays together: their pending regions are planned at
    once, so arrays sharing inputs fuse into one multi-root kernel."""
    arrays = [a for a in arrays if isinstance(a, ndarray)]
    if not arrays:
        return
    sess = arrays[0]._session
    sess.force_nodes([a._node for a in arrays])


def materialize(*arrays, out=None) -> list:
    """to_external for several arrays at once: force them
    together and return host arrays (written into ``out`` when given).

    When the pending region reads host-resident inputs along the roots'
    leading axis and every root is row-local, the force is streamed
    (streaming.py): chunks of rows flow H2D -> fused kernel -> D2H on three
    streams so the PCIe copies overlap each other and the kernels.  Page-
    locked ``out`` arrays (``Runtime.pinned_empty``) let the D2H run async."""
    arrays = [a if isinstance(a, ndarray) else asarray(a) for a in arrays]
    if not arrays:
        return []
    outs = list(out) if out is not None else [None] * len(arrays)
    if len(outs) != len(arrays):
        raise ShapeMismatch("materialize: one out array per input array")
    for a, o in zip(arrays, outs):
        if o is not None and (o.shape != a.shape or o.dtype != a.dtype or not o.flags.c_contiguous):
            raise ShapeMismatch("out must be a C-contiguous array of the same shape and dtype")
    sess = arrays[0]._session
    nodes = [a._node for a in arrays]
    if (sess.comm is None and os.environ.get("GRUMPY_STREAM", "1") != "0"
            and len({n.id for n in nodes}) == len(nodes)):
        from . import streaming
        p = streaming.plan(nodes)
        if p is not None:
            outs = [o if o is not None else np.empty(a.shape, a.dtype) for a, o in zip(arrays, outs)]
            order = {n.id: i for i, n in enumerate(nodes)}
            streaming.run(sess, p, [outs[order[r.id]] for r in p.roots])
            return outs
    sess.force_nodes(nodes)
    return [a.numpy(out=o) if o is not None else a.numpy() for a, o in zip(arrays, outs)]


def asnumpy(a) -> np.ndarray:
    return a.numpy() if isinstance(a, ndarray) else np.asarray(a)

