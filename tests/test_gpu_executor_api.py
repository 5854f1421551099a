"""The reference's executor / lowering interface on the B200 path
(SPEC.md:301-420): lower → run_map / run_map_reduce / run_map_scan, compile
vs the oracle's eval_point (dual execution), run_library known answers."""
import numpy as np
import pytest

import paper_1901_03771_b200 as gp
from paper_1901_03771_b200 import lowering, planner
from paper_1901_03771_b200.dag import ElemCode, Graph, Op, OpKind, ReduceOp
from paper_1901_03771_b200.errors import ShapeMismatch
from paper_1901_03771_b200.executor import (ExecConfig, LibraryCall, run_library, run_map, run_map_reduce,
                                            run_map_scan)
from paper_1901_03771_b200.tensor import TensorBuffer

from oracle.eager import eval_point

pytestmark = pytest.mark.gpu

TB = TensorBuffer.from_numpy


def _kernel(root):
    steps = planner.plan(root)
    assert len(steps) == 1
    return lowering.lower(steps[0])


def test_run_map_identity():
    """identity map over [4] → [1,2,3,4]."""
    g = Graph()
    x = g.add_input(TB(np.array([1.0, 2, 3, 4])))
    r = g.add_op(Op(OpKind.RESHAPE, attrs=((4,),)), [x])
    k = _kernel(r)
    out = run_map(k, [TB(np.array([1.0, 2, 3, 4]))], ExecConfig(4))
    assert out.to_numpy().tolist() == [1, 2, 3, 4]


def test_run_map_fig1_bit_exact():
    """the Fig. 1 program on random 64×64 inputs equals the eager
    oracle bit-exactly; and for every num_threads."""
    rng = np.random.default_rng(3)
    W, a, b = rng.random((64, 64)), rng.random((64, 64)), rng.random((64, 64))
    s = gp.Session()
    gW, ga, gb = (gp.asarray(v, session=s) for v in (W, a, b))
    out = (ga * gW) * (gb * gW) * gW + ga + gb
    k = _kernel(out._node)
    leaves = {l.id: TB(l.data.host) for l in k.step.leaves}
    ref = (a * W) * (b * W) * W + a + b
    for nt in (1, 2, 4, 8):
        got = run_map(k, leaves, ExecConfig(nt)).to_numpy()
        assert np.array_equal(got, ref)


def test_run_map_empty_space():
    """empty space → empty buffer."""
    g = Graph()
    x = g.add_input(TB(np.zeros((0, 3))))
    y = g.add_op(Op(OpKind.MAP, ElemCode.neg), [x])
    k = _kernel(y)
    assert run_map(k, [TB(np.zeros((0, 3)))]).to_numpy().shape == (0, 3)


def test_run_map_reduce_kats():
    """SPEC.md:379-381."""
    g = Graph()
    x = g.add_input(TB(np.array([1.0, 2, 3, 4])))
    r = g.add_op(Op(OpKind.REDUCE, attrs=(ReduceOp.sum, (0,), False, None)), [x])
    # a pure sum's point program is a load: Algorithm 1 still plans one MapReduce
    k = _kernel(r)
    assert float(run_map_reduce(k, [TB(np.array([1.0, 2, 3, 4]))]).to_numpy()) == 10.0
    g = Graph()
    a = g.add_input(TB(np.array([1.0, 2, 3])))
    b = g.add_input(TB(np.array([4.0, 5, 6])))
    m = g.add_op(Op(OpKind.MAP, ElemCode.mul), [a, b])
    r = g.add_op(Op(OpKind.REDUCE, attrs=(ReduceOp.sum, (0,), False, None)), [m])
    k = _kernel(r)
    assert float(run_map_reduce(k, [TB(np.array([1.0, 2, 3])), TB(np.array([4.0, 5, 6]))]).to_numpy()) == 32.0
    v = np.random.default_rng(0).standard_normal(10**6)
    g = Graph()
    x = g.add_input(TB(v))
    r = g.add_op(Op(OpKind.REDUCE, attrs=(ReduceOp.max, (0,), False, None)), [x])
    assert float(run_map_reduce(_kernel(r), [TB(v)]).to_numpy()) == v.max()


def test_run_map_scan_kats():
    """SPEC.md:388-390."""
    for vals, op, exp in [([1, 2, 3], ReduceOp.sum, [1, 3, 6]), ([0.0, 0, 0, 0], ReduceOp.sum, [0, 0, 0, 0]),
                          ([3, 1, 4, 1, 5], ReduceOp.max, [3, 3, 4, 4, 5])]:
        g = Graph()
        arr = np.array(vals)
        x = g.add_input(TB(arr))
        s = g.add_op(Op(OpKind.SCAN, attrs=(op, None, None)), [x])
        k = _kernel(s)
        assert k.kind == "MapScan"
        assert run_map_scan(k, [TB(arr)]).to_numpy().tolist() == exp


def test_run_checks_leaves():
    g = Graph()
    x = g.add_input(TB(np.zeros(4)))
    y = g.add_op(Op(OpKind.MAP, ElemCode.neg), [x])
    k = _kernel(y)
    with pytest.raises(ShapeMismatch):
        run_map(k, [TB(np.zeros(5))])
    with pytest.raises(ValueError):
        run_map_reduce(k, [TB(np.zeros(4))])


def test_compile_equals_eval_point_1000_coords():
    """compiled(coords) == eval_point(coords) at 1000 random
    coordinates — Black-Scholes body, f64, ≤1e-12 rel (bit-exact for the
    pure +,* parts)."""
    from paper_1901_03771_b200 import workloads as wl
    rng = np.random.default_rng(11)
    n = 4096
    S, X, T = rng.uniform(5, 30, n), rng.uniform(1, 100, n), rng.uniform(0.25, 10, n)
    s = gp.Session()
    call, put = wl.blackscholes(gp, gp.asarray(S, session=s), gp.asarray(X, session=s), gp.asarray(T, session=s))
    steps = planner.plan(call._node)
    st = steps[-1]
    k = lowering.lower(st)
    fn = lowering.compile(k.point)
    leaves = {l.id: TB(l.data.host) for l in st.leaves}
    coords = rng.integers(0, n, 1000)
    for c in coords:
        got = fn((int(c),), leaves)
        ref = eval_point(k.point, (int(c),), leaves)
        assert abs(got - ref) <= 1e-12 * max(abs(ref), 1e-300) + 1e-10, (c, got, ref)


def test_compile_map_reduce_point_is_the_operand():
    rng = np.random.default_rng(12)
    x = rng.standard_normal((16, 32)).astype(np.float32)
    s = gp.Session()
    r = (gp.asarray(x, session=s) * 3 - 1).sum(1)
    k = _kernel(r._node)
    fn = lowering.compile(k.point)
    leaves = {l.id: TB(l.data.host) for l in k.step.leaves}
    for c in [(0, 0), (5, 17), (15, 31)]:
        assert fn(c, leaves) == eval_point(k.point, c, leaves) == np.float32(x[c] * np.float32(3) - np.float32(1))


def test_run_library_kats():
    """SPEC.md:397-399."""
    y = run_library(LibraryCall("Gemv", (False,)), [TB(np.eye(3)), TB(np.array([7.0, 8, 9]))])
    assert y.to_numpy().tolist() == [7, 8, 9]
    y = run_library(LibraryCall("Gemv", (True,)), [TB(np.array([[1.0, 2], [3, 4]])), TB(np.array([1.0, 1]))])
    assert y.to_numpy().tolist() == [4, 6]
    rng = np.random.default_rng(13)
    A, B = rng.standard_normal((2, 3)), rng.standard_normal((3, 2))
    C = run_library(LibraryCall("Gemm", (False, False)), [TB(A), TB(B)]).to_numpy()
    naive = np.array([[sum(A[i, q] * B[q, j] for q in range(3)) for j in range(2)] for i in range(2)])
    np.testing.assert_allclose(C, naive, rtol=1e-12)
    for ta in (False, True):
        for tb in (False, True):
            A2 = rng.standard_normal((5, 7) if not ta else (7, 5))
            B2 = rng.standard_normal((7, 4) if not tb else (4, 7))
            got = run_library(LibraryCall("Gemm", (ta, tb)), [TB(A2), TB(B2)]).to_numpy()
            np.testing.assert_allclose(got, (A2.T if ta else A2) @ (B2.T if tb else B2), rtol=1e-12)
    with pytest.raises(ShapeMismatch):
        run_library(LibraryCall("Gemv"), [TB(np.eye(3)), TB(np.ones(4))])


def test_run_library_random_128_f64():
    """equals the naive triple loop within 1e-12 rel up to 128×128."""
    rng = np.random.default_rng(14)
    for m, kk, n in [(1, 1, 1), (17, 33, 9), (128, 128, 128)]:
        A, B = rng.standard_normal((m, kk)), rng.standard_normal((kk, n))
        got = run_library(LibraryCall("Gemm"), [TB(A), TB(B)]).to_numpy()
        ref = np.einsum("ik,kj->ij", A.astype(np.longdouble), B.astype(np.longdouble)).astype(np.float64)
        np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-12 * np.abs(A).sum() * np.abs(B).max())
