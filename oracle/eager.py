"""ORACLE — test infrastructure only.  Never imported by the product package.

Eager reference evaluator: "a single-threaded per-node interpreter serving as
the correctness oracle, playing the role of the paper's baseline"
("speedup over Numpy").

Each DAG node is evaluated eagerly with the NumPy (and SciPy, for erf) call that
the NumPy program the node was recorded from would have made, so results are
NumPy's own — including NumPy's reduction association order (pairwise summation
along the contiguous axis, sequential along the others; restated and pinned in
``oracle/pairwise.py``).  Per-op semantics follow SPEC.md:93-116 (vocabulary),
SPEC.md:143 (inference), SPEC.md:304 (lowering of slices / SliceAssign),
SPEC.md:376/408 (reductions), SPEC.md:385 (scans), SPEC.md:394 (library calls).

Materialized nodes evaluate to their host data (the step-local check of
SURVEY.md §7 "check the region against its own leaves"); call ``evaluate``
before forcing to check a whole program from its inputs.

Parity pins: the spec's known-answer examples (tests/test_oracle_pins.py,
tests/golden/spec_kats.json) and NumPy itself (the reference's declared
arithmetic dependency, pkg/pyproject.toml:11, numpy 2.3.5 installed here).
No reference engine exists to run, so there is no oracle/_ref.
"""

from __future__ import annotations

from typing import Dict

import numpy as np

from paper_1901_03771_b200.dag import ElemCode, Node, OpKind, ReduceOp, UFUNC_OF
from paper_1901_03771_b200.errors import OutOfBounds

try:  # erf lives in SciPy (pkg/pyproject.toml:13), as NumPy has none
    from scipy.special import erf as _erf
except ImportError:  # pragma: no cover
    _erf = None


def _slices(spec):
    out = []
    for start, step, length in spec:
        if length == 0:
            out.append(slice(0, 0, 1))
            continue
        stop = start + length * step
        if step < 0 and stop < 0:
            stop = None
        out.append(slice(start, stop, step))
    return tuple(out)


def host_data(n: Node) -> np.ndarray:
    buf = n.data
    if buf.host is None:
        # Device-only buffer: copy back through the product's buffer API.
        return buf.device.to_numpy(buf.dtype, buf.shape)
    return buf.host


def evaluate(n: Node, cache: Dict[int, np.ndarray] | None = None) -> np.ndarray:
    """Eagerly evaluate ``n`` with NumPy; returns an ndarray (0-d for scalars)."""
    if cache is None:
        cache = {}
    return _eval(n, cache)


def eval_point(point, coords, leaves) -> np.generic:
    """Reference executor for a point program: the value of
    the point function at ``coords`` given leaf buffers (leaf node id →
    TensorBuffer or ndarray).  ``point`` is a ``lowering.PointProgram``; its
    value nodes are evaluated eagerly over the leaves, then indexed."""
    cache = {}
    for lid, b in leaves.items():
        cache[lid] = np.asarray(b.host if hasattr(b, "host") and b.host is not None else
                                (b.to_numpy() if hasattr(b, "to_numpy") else b))
    v = _eval(point.value_nodes[0], cache)
    return v[tuple(coords)]


def _eval(n: Node, cache) -> np.ndarray:
    hit = cache.get(n.id)
    if hit is not None:
        return hit
    if n.is_materialized:
        r = host_data(n)
    else:
        r = _compute(n, [_eval(p, cache) for p in n.preds])
    r = np.asarray(r)
    assert r.dtype == n.dtype.np, (n, r.dtype)
    assert r.shape == n.shape, (n, r.shape)
    cache[n.id] = r
    return r


def _compute(n: Node, a):
    op = n.op
    k = op.kind
    if k is OpKind.MAP:
        code = op.code
        if code is ElemCode.const_splat:
            return np.full(n.shape, op.attrs[0], dtype=n.dtype.np)
        if code is ElemCode.select:
            return np.where(a[0], a[1], a[2]).astype(n.dtype.np, copy=False)
        if code is ElemCode.erf:
            return _erf(a[0])
        with np.errstate(all="ignore"):
            if code is ElemCode.square:
                # NumPy's x**2 fast path (array_power) is np.square
                return np.square(a[0])
            return UFUNC_OF[code](*a)
    if k is OpKind.CAST:
        with np.errstate(all="ignore"):
            return a[0].astype(n.dtype.np)
    if k is OpKind.TRANSPOSE:
        return np.transpose(a[0], op.attrs[0])
    if k is OpKind.RESHAPE:
        return np.reshape(a[0], op.attrs[0])
    if k is OpKind.BROADCAST:
        return np.broadcast_to(a[0], op.attrs[0])
    if k is OpKind.SLICE:
        return a[0][_slices(op.attrs[0])]
    if k is OpKind.SLICE_ASSIGN:
        t = np.array(a[0], copy=True)
        t[_slices(op.attrs[0])] = a[1]
        return t
    if k is OpKind.REDUCE:
        rop, axes, keepdims, odt = op.attrs
        x = a[0]
        uf = {ReduceOp.sum: np.add, ReduceOp.prod: np.multiply,
              ReduceOp.max: np.maximum, ReduceOp.min: np.minimum}[rop]
        dt = n.dtype.np if n.dtype.np != x.dtype else None
        with np.errstate(all="ignore"):
            return uf.reduce(x, axis=axes, keepdims=keepdims, dtype=dt)
    if k is OpKind.ARGREDUCE:
        which, axis, keepdims = op.attrs
        f = np.argmax if which == "max" else np.argmin
        return f(a[0], axis=axis, keepdims=keepdims)
    if k is OpKind.SCAN:
        rop, axis, odt = op.attrs
        x = a[0]
        if axis is None:
            x = x.reshape(-1)
            axis = 0
        uf = {ReduceOp.sum: np.add, ReduceOp.prod: np.multiply,
              ReduceOp.max: np.maximum, ReduceOp.min: np.minimum}[rop]
        if len(a) > 1:
            # seeded: the fold starts from the seed (a line of the kept axes)
            seed = np.expand_dims(np.asarray(a[1]).reshape(
                tuple(d for i, d in enumerate(x.shape) if i != axis)), axis).astype(n.dtype.np)
            return uf.accumulate(np.concatenate([seed, x.astype(n.dtype.np)], axis=axis), axis=axis,
                                 dtype=n.dtype.np).take(range(1, x.shape[axis] + 1), axis=axis)
        return uf.accumulate(x, axis=axis, dtype=n.dtype.np)
    if k is OpKind.MATMUL:
        return np.matmul(a[0], a[1])
    if k is OpKind.MATVEC:
        (trans,) = op.attrs
        return a[1] @ a[0] if trans else a[0] @ a[1]
    if k is OpKind.KEYED_SUM:
        (nbins,) = op.attrs
        keys = a[0]
        if keys.size and (keys.min() < 0 or keys.max() >= nbins):
            raise OutOfBounds("bincount key outside [0, nbins)")
        w = a[1] if len(a) > 1 else None
        return np.bincount(keys, weights=w, minlength=nbins)
    raise NotImplementedError(k)
