"""Pin the oracle before trusting it (CPU only).

1. the spec's known-answer examples (tests/golden/spec_kats.json, each citing
   /root/reference/SPEC.md) through the eager oracle and the host modules;
2. the pairwise-summation restatement (oracle/pairwise.py) against NumPy's
   own add.reduce for many lengths, dtypes and axes;
3. the eager DAG evaluator against the same programs run on plain NumPy;
4. the committed config fixtures against a fresh NumPy/SciPy evaluation.
"""
import json
import os

import numpy as np
import pytest

import paper_1901_03771_b200 as gp
from paper_1901_03771_b200 import errors, tensor, workloads as wl
from paper_1901_03771_b200.dag import Graph, Op, OpKind, ReduceOp, ElemCode
from oracle import eager, pairwise

GOLD = os.path.join(os.path.dirname(__file__), "golden")
KATS = json.load(open(os.path.join(GOLD, "spec_kats.json")))


@pytest.fixture
def sess():
    s = gp.Session()
    old = gp.set_default_session(s)
    yield s
    gp.set_default_session(old)


@pytest.mark.parametrize("kat", KATS, ids=[k["name"] for k in KATS])
def test_spec_kat(kat, sess):
    op = kat["op"]
    if "raises" in kat:
        exc = getattr(errors, kat["raises"])
        with pytest.raises(exc):
            if op == "broadcast_shapes":
                tensor.broadcast_shapes(kat["a"], kat["b"])
            else:
                tensor.delinearize(kat["linear"], kat["shape"])
        return
    g = Graph()
    if op == "broadcast_shapes":
        got = list(tensor.broadcast_shapes(kat["a"], kat["b"]))
    elif op == "delinearize":
        got = list(tensor.delinearize(kat["linear"], kat["shape"]))
        assert tensor.linearize(got, kat["shape"]) == kat["linear"]
    elif op.startswith("infer"):
        ins = [g.add_input(tensor.TensorBuffer.from_numpy(np.zeros(s))) for s in kat["shapes"]]
        if op == "infer_map_mul":
            n = g.add_op(Op(OpKind.MAP, ElemCode.mul), ins)
        elif op == "infer_matvec":
            n = g.add_op(Op(OpKind.MATVEC, None, (False,)), ins)
        elif op == "infer_reduce_all":
            n = g.add_op(Op(OpKind.REDUCE, None, (ReduceOp.sum, (0, 1), False, None)), ins)
        elif op == "infer_transpose":
            n = g.add_op(Op(OpKind.TRANSPOSE, None, (tuple(kat["perm"]),)), ins)
        elif op == "infer_slice":
            n = g.add_op(Op(OpKind.SLICE, None, (((1, 1, 64), (1, 1, 64)),)), ins)
        else:
            n = g.add_op(Op(OpKind.SCAN, None, (ReduceOp.sum, 0, None)), ins)
        got = list(n.shape)
    else:
        if op == "map_identity":
            r = gp.asarray(np.array(kat["x"])).copy()
        elif op == "sum":
            r = gp.asarray(np.array(kat["x"])).sum()
        elif op == "inner":
            r = gp.dot(gp.asarray(np.array(kat["a"])), gp.asarray(np.array(kat["b"])))
        elif op == "cumsum":
            r = gp.asarray(np.array(kat["x"])).cumsum()
        elif op == "cummax":
            r = np.maximum.accumulate(gp.asarray(np.array(kat["x"])))
        elif op == "gemv":
            A = gp.asarray(np.array(kat["A"], dtype=np.float64))
            x = gp.asarray(np.array(kat["x"], dtype=np.float64))
            r = (A.T if kat["trans"] else A) @ x
        elif op == "const3":
            r = gp.full(tuple(kat["shape"]), 3.0)
        elif op == "inner_point":
            r = (gp.asarray(np.array(kat["a"])) * gp.asarray(np.array(kat["b"])))[kat["i"]]
        got = eager.evaluate(r.node).tolist()
    assert got == kat["expect"], (kat, got)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_pairwise_restatement_matches_numpy(dtype):
    rng = np.random.default_rng(0)
    for n in [0, 1, 5, 7, 8, 9, 15, 16, 100, 127, 128, 129, 255, 256, 1000, 4096, 12345, 65536, 100003]:
        a = rng.standard_normal(n).astype(dtype)
        assert pairwise.add_reduce_1d(a) == np.add.reduce(a), n


def test_numpy_reduction_order_rules():
    """Row sums are per-row pairwise; axis-0 sums are sequential from 0.0."""
    rng = np.random.default_rng(1)
    x = rng.standard_normal((33, 300)).astype(np.float32)
    rows = np.array([pairwise.add_reduce_1d(r) for r in x], dtype=np.float32)
    assert np.array_equal(rows, x.sum(1))
    col = np.zeros(300, np.float32)
    for r in x:
        col = col + r
    assert np.array_equal(np.float32(0) + col, x.sum(0))
    assert pairwise.add_reduce_1d(x.ravel()) == x.sum()


def test_executor_oracles():
    """blocked folds, three-phase scans and naive library ops."""
    rng = np.random.default_rng(2)
    a = rng.integers(-50, 50, 997)
    for T in (1, 2, 4, 8):
        assert pairwise.blocked_fold(a, lambda x, y: x + y, 0, T) == a.sum()
        assert pairwise.blocked_fold(a, max, -10**9, T) == a.max()
    for block in (1, 7, 997, 2000):
        assert np.array_equal(pairwise.scan_three_phase(a, lambda x, y: x + y, block), np.cumsum(a))
    A = rng.standard_normal((5, 7))
    B = rng.standard_normal((7, 3))
    np.testing.assert_allclose(pairwise.naive_gemm(A, B), A @ B, rtol=1e-12)
    np.testing.assert_allclose(pairwise.naive_gemm(A.T, B, trans_a=True), A @ B, rtol=1e-12)
    x7 = rng.standard_normal(7)
    x5 = rng.standard_normal(5)
    np.testing.assert_allclose(pairwise.naive_gemv(A, x7), A @ x7, rtol=1e-12)
    np.testing.assert_allclose(pairwise.naive_gemv(A, x5, trans_a=True), A.T @ x5, rtol=1e-12)


def test_eager_oracle_equals_numpy_programs(sess):
    W, a, b = wl.listing1_inputs(n=1000)
    r = wl.listing1(gp, gp.asarray(W), gp.asarray(a), gp.asarray(b))
    assert np.array_equal(eager.evaluate(r.node), wl.listing1(np, W, a, b))
    S, X, T = wl.blackscholes_inputs(n=1000, dtype=np.float32)
    c, p = wl.blackscholes(gp, gp.asarray(S), gp.asarray(X), gp.asarray(T))
    ec, ep = wl.blackscholes(np, S, X, T)
    assert np.array_equal(eager.evaluate(c.node), ec)
    assert np.array_equal(eager.evaluate(p.node), ep)
    (x,) = wl.rownorm_inputs(rows=16, cols=256)
    y, t = wl.rownorm(gp, gp.asarray(x))
    ey, et = wl.rownorm(np, x)
    assert np.array_equal(eager.evaluate(y.node), ey)
    assert eager.evaluate(t.node) == et
    P, C = wl.kmeans_inputs(n=512, k=8, d=4)
    lab, sums, counts = wl.kmeans_partials(gp, gp.asarray(P), gp.asarray(C))
    elab, esums, ecounts = wl.kmeans_partials(np, P, C)
    assert np.array_equal(eager.evaluate(lab.node), elab)
    assert np.array_equal(eager.evaluate(counts.node), ecounts)
    for s, e in zip(sums, esums):
        assert np.array_equal(eager.evaluate(s.node), e)


def test_config_fixtures_reproduce():
    f = np.load(os.path.join(GOLD, "configs_small.npz"))
    assert np.array_equal(wl.listing1(np, f["l1_W"], f["l1_a"], f["l1_b"]), f["l1_out"])
    for tag in ("f32", "f64"):
        c, p = wl.blackscholes(np, f[f"bs{tag}_S"], f[f"bs{tag}_X"], f[f"bs{tag}_T"])
        assert np.array_equal(c, f[f"bs{tag}_call"]) and np.array_equal(p, f[f"bs{tag}_put"])
    y, t = wl.rownorm(np, f["rn_x"])
    assert np.array_equal(y, f["rn_y"]) and t == f["rn_total"]
    lab, sums, counts = wl.kmeans_partials(np, f["km_P"], f["km_C"])
    assert np.array_equal(lab, f["km_lab"]) and np.array_equal(counts, f["km_counts"])
