"""CPU checks of the drop-in boundary and the host-side modules.

* libgrumpy_rt.so loads without a driver and exports every symbol
  include/grumpy_rt.h declares (no compute calls here);
* without a GPU the product path fails loudly (no CPU fallback);
* tensor-core / expr-dag properties and the session's
  laziness and eager shape errors."""
import ctypes
import os
import re

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

import paper_1901_03771_b200 as gp
from paper_1901_03771_b200 import errors, runtime, tensor
from paper_1901_03771_b200.dag import Graph, Op, OpKind

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(REPO, "include", "grumpy_rt.h")).read()
    return sorted(set(re.findall(r"\b(grumpy_rt_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_header_symbols():
    lib = runtime.load_library()
    syms = header_symbols()
    assert len(syms) >= 30
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(runtime.SIGNATURES), set(syms) ^ set(runtime.SIGNATURES)


def test_no_device_fails_loudly():
    lib = runtime.load_library()
    n = ctypes.c_int(-1)
    rc = lib.grumpy_rt_device_count(ctypes.byref(n))
    if rc == 0 and n.value > 0:
        pytest.skip("a GPU is present")
    s = gp.Session()
    x = gp.asarray(np.ones(4), session=s)
    with pytest.raises(errors.NativeLibraryMissing):
        np.asarray(x + 1)


def test_errors_mirror_reference():
    names = ["LazyFuseError", "IncompatibleShapes", "ShapeMismatch", "DTypeMismatch", "UnsupportedDType",
             "BadAxis", "OutOfBounds", "AlreadyMaterializedWithDifferentData", "UnsupportedNodeInFusedStep",
             "NpyFormatError", "VerificationFailed"]
    for nm in names:
        cls = getattr(errors, nm)
        assert issubclass(cls, errors.LazyFuseError)


shapes = st.lists(st.integers(1, 4), min_size=0, max_size=4).map(tuple)


@given(shapes, shapes, shapes)
@settings(max_examples=200, deadline=None)
def test_broadcast_commutative_associative(a, b, c):
    """SPEC.md:65-66."""
    def bs(x, y):
        try:
            return tensor.broadcast_shapes(x, y)
        except errors.IncompatibleShapes:
            return None
    assert bs(a, b) == bs(b, a)
    ab = bs(a, b)
    bc = bs(b, c)
    left = bs(ab, c) if ab is not None else None
    right = bs(a, bc) if bc is not None else None
    if left is not None and right is not None:
        assert left == right
    assert bs(a, (1,) * len(a)) == a and bs(a, ()) == a
    if ab is not None:
        assert ab == np.broadcast_shapes(a, b)


@given(st.lists(st.integers(1, 6), min_size=1, max_size=4))
@settings(max_examples=100, deadline=None)
def test_linearize_delinearize_roundtrip(shape):
    """SPEC.md:67."""
    n = int(np.prod(shape))
    for k in range(0, n, max(1, n // 17)):
        assert tensor.linearize(tensor.delinearize(k, shape), shape) == k


def test_graph_audit_and_materialize():
    """SPEC.md:156-169."""
    g = Graph()
    a = g.add_input(tensor.TensorBuffer.from_numpy(np.ones((2, 2))))
    s = g.add_op(Op(OpKind.REDUCE, None, (gp.dag.ReduceOp.sum, (0, 1), False, None)), [a])
    g.audit()
    buf = tensor.TensorBuffer.from_numpy(np.array(4.0))
    with pytest.raises(errors.ShapeMismatch):
        g.mark_materialized(s, tensor.TensorBuffer.from_numpy(np.ones(3)))
    g.mark_materialized(s, buf)
    g.mark_materialized(s, buf)          # idempotent
    with pytest.raises(errors.AlreadyMaterializedWithDifferentData):
        g.mark_materialized(s, tensor.TensorBuffer.from_numpy(np.array(5.0)))
    assert s.is_materialized
    dot = g.dot()
    assert "digraph" in dot and "[M]" in dot


def test_session_lazy_and_eager_errors():
    s = gp.Session()
    x = gp.asarray(np.ones((3, 4)), session=s)
    y = gp.asarray(np.ones((2, 4)), session=s)
    z = (x * 2 + 1).sum(1)                 # records only
    assert s.stats.kernels_executed == 0 and s._executor is None
    assert z.shape == (3,) and z.dtype == np.float64
    with pytest.raises(errors.IncompatibleShapes):
        x + y
    with pytest.raises(errors.BadAxis):
        x.sum(axis=2)
    with pytest.raises(errors.ShapeMismatch):
        x.reshape(5, 5)


def test_numpy_dtype_semantics():
    """NumPy (NEP 50) promotion, not SPEC.md:71's linear order."""
    s = gp.Session()
    f = gp.asarray(np.ones(3, np.float32), session=s)
    i = gp.asarray(np.ones(3, np.int32), session=s)
    L = gp.asarray(np.ones(3, np.int64), session=s)
    assert (f * 0.5).dtype == np.float32
    assert (f * np.float64(2)).dtype == np.float64
    assert (L + f).dtype == np.float64
    assert (i / i).dtype == np.float64
    assert (i + 3).dtype == np.int32
    assert gp.exp(i).dtype == np.float64
    assert (i ** 2).dtype == np.int32
    assert i.sum().dtype == np.int64 and i.mean().dtype == np.float64
    assert f.argmax().dtype == np.int64
    assert (f > 1).dtype == np.bool_
    with pytest.raises(OverflowError):
        i + 2 ** 40


def test_ufunc_and_function_protocol_record():
    s = gp.Session()
    old = gp.set_default_session(s)
    try:
        x = gp.asarray(np.ones((4, 4), np.float32))
        for r in (np.exp(x), np.maximum(x, 0), np.sum(x, axis=1), np.mean(x), np.argmax(x, axis=0),
                  np.where(x > 0, x, 0), np.dot(x, x), x @ x, np.transpose(x), np.add.reduce(x, axis=0)):
            assert isinstance(r, gp.ndarray)
        from scipy.special import erf
        assert isinstance(erf(x), gp.ndarray)
        assert s.stats.kernels_executed == 0
    finally:
        gp.set_default_session(old)
