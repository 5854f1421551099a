"""fusion-planner: Algorithm 1 golden plans and region-pass
invariants checked with a plan simulator (CPU only)."""
import numpy as np
import pytest

import paper_1901_03771_b200 as gp
from paper_1901_03771_b200 import codegen, planner, workloads as wl
from paper_1901_03771_b200.dag import OpKind
from paper_1901_03771_b200.planner import PlannerLimits, demand_set, materialize_node, materialize_pred_of_node, plan


@pytest.fixture
def sess():
    s = gp.Session()
    old = gp.set_default_session(s)
    yield s
    gp.set_default_session(old)


def describe(steps):
    out = []
    for s in steps:
        if s.kind == "Library":
            out.append(("Library", s.call, s.trans_flags, s.root.id, frozenset(l.id for l in s.leaves)))
        else:
            out.append(("Fused", s.kernel_kind, s.root.id, frozenset(l.id for l in s.leaves)))
    return out


def simulate(steps, roots):
    """Plan simulator: at each step, the leaves and only the
    leaves are materialized; every root ends materialized."""
    done = set()
    for st in steps:
        for l in st.leaves:
            # const_splat nodes carry their value in the op: a
            # leaf that is always ready
            const = l.kind is OpKind.MAP and l.op.code is not None and l.op.code.name == "const_splat"
            assert l.is_materialized or l.id in done or const, f"leaf {l.id} not ready before step {st.describe()}"
        interior = {n.id for n in st.nodes}
        for l in st.leaves:
            assert l.id not in interior
        for r in st.roots:
            done.add(r.id)
    for r in roots:
        assert r.is_materialized or r.id in done


def test_golden_mnist_pattern(sess):
    """3 steps — Fused(Map) max, Library(Gemv, transA), Fused(Map) output."""
    W = gp.asarray(np.ones((784, 10)))
    x = gp.asarray(np.ones(784))
    b = gp.asarray(np.ones(10))
    m = gp.maximum(x, 0.0)
    mv = W.T @ m
    out = mv + b
    steps = plan(out.node)
    d = describe(steps)
    assert d == [
        ("Fused", "Map", m.node.id, frozenset({x.node.id})),
        ("Library", "Gemv", (True, False), mv.node.id, frozenset({W.node.id, m.node.id})),
        ("Fused", "Map", out.node.id, frozenset({mv.node.id, b.node.id})),
    ]
    simulate(steps, [out.node])


def test_golden_listing1_one_step(sess):
    """the pointwise DAG of Fig. 1 is one Fused(Map) step."""
    W, a, b = (gp.asarray(np.ones(16)) for _ in range(3))
    out = wl.listing1(gp, W, a, b)
    steps = plan(out.node)
    assert describe(steps) == [("Fused", "Map", out.node.id, frozenset({W.node.id, a.node.id, b.node.id}))]


def test_golden_shared_exp_sum_add(sess):
    """v=exp(x); s=sum(v); out=s+v → 3 steps (multiple-use rule)."""
    x = gp.asarray(np.ones(8))
    v = gp.exp(x)
    s = v.sum()
    out = s + v
    steps = plan(out.node)
    assert describe(steps) == [
        ("Fused", "Map", v.node.id, frozenset({x.node.id})),
        ("Fused", "MapReduce", s.node.id, frozenset({v.node.id})),
        ("Fused", "Map", out.node.id, frozenset({s.node.id, v.node.id})),
    ]
    simulate(steps, [out.node])


def test_plan_examples(sess):
    x = gp.asarray(np.ones(4))
    assert plan(x.node) == []
    y = x
    for _ in range(150):
        y = gp.exp(y)
    steps = plan(y.node, limits=PlannerLimits(100))
    assert [s.kind for s in steps] == ["Fused", "Fused"]
    assert all(len(s.nodes) <= 100 for s in steps)
    simulate(steps, [y.node])


def test_predicates(sess):
    """SPEC.md:220-231."""
    x = gp.asarray(np.ones((3, 3)))
    assert materialize_node(x.sum().node)
    assert not materialize_node((x + 1).node)
    assert materialize_node((x @ x).node)
    mv = x.T @ gp.asarray(np.ones(3))
    assert not materialize_pred_of_node(mv.node, mv.node.preds[0])    # absorbed transpose
    mm = gp.maximum(x, 0) @ x
    assert materialize_pred_of_node(mm.node, mm.node.preds[0])
    a = x + 1
    assert not materialize_pred_of_node(a.node, a.node.preds[0])


def test_demand_set(sess):
    """SPEC.md:211-213."""
    x = gp.asarray(np.ones(4))
    e = gp.exp(x)
    out = e + 1
    ids = {n.id for n in demand_set(out.node)}
    assert x.node.id in ids and e.node.id in ids and out.node.id in ids
    assert {n.id for n in demand_set(x.node)} == {x.node.id}


def region_plan(roots):
    return planner.plan_regions([r.node for r in roots], row_fusion=codegen.row_fusable, check=codegen.check_step)


def test_region_pass_fuses_configs(sess):
    S, X, T = (gp.asarray(v) for v in wl.blackscholes_inputs(n=64))
    c, p = wl.blackscholes(gp, S, X, T)
    steps = region_plan([c, p])
    assert len(steps) == 1 and len(steps[0].roots) == 2          # one multi-root kernel
    (x,) = (gp.asarray(v) for v in wl.rownorm_inputs(rows=8, cols=256))
    y, tot = wl.rownorm(gp, x)
    steps = region_plan([y, tot])
    assert len(steps) == 1                                      # Algorithm 1 would use 4
    assert len(plan(tot.node)) >= 4
    Xm, W1, b1, W2, b2 = (gp.asarray(v) for v in wl.mlp_inputs(batch=32, hidden=16))
    pr, lab = wl.mlp(gp, Xm, W1, b1, W2, b2)
    steps = region_plan([pr, lab])
    kinds = [s.kind for s in steps]
    assert kinds == ["Library", "Fused", "Library", "Fused"]    # GEMM, bias+ReLU, GEMM, softmax+argmax
    simulate(steps, [pr.node, lab.node])
    P, C = (gp.asarray(v) for v in wl.kmeans_inputs(n=256, k=8, d=4))
    l, sums, counts = wl.kmeans_partials(gp, P, C)
    steps = region_plan([l, *sums, counts])
    assert len(steps) == 1


def test_region_pass_cuts_nonlocal_reductions(sess):
    x = gp.asarray(np.ones((16, 8)))
    out = x - x.sum(0)               # column sums broadcast over rows: cut
    steps = region_plan([out])
    assert len(steps) == 2
    simulate(steps, [out.node])
    out2 = x - x.mean()              # full reduction consumed per element: cut
    steps = region_plan([out2])
    assert len(steps) == 2
    simulate(steps, [out2.node])


def test_plan_cache_reuses_structure(sess):
    from paper_1901_03771_b200.planner import dag_signature
    a = gp.asarray(np.ones(4))
    b = gp.asarray(np.ones(4))
    k1, _ = dag_signature([(a * b + 1).node])
    k2, _ = dag_signature([(a * b + 1).node])
    k3, _ = dag_signature([(a * a + 1).node])
    assert k1 == k2 and k1 != k3


def test_chained_jacobi_sweeps_one_step_each(sess):
    """10 lazily chained sweeps plan as 10 fused maps: a grid
    read through several slices is materialized, not recomputed per read."""
    a = gp.asarray(wl.jacobi_inputs(64)[0])
    for _ in range(10):
        a = wl.jacobi(gp, a)
    steps = sess.plan([a.node])
    assert [s.kernel_kind for s in steps] == ["Map"] * 10
    # a computed node read through one slice stays fused
    x = gp.asarray(np.arange(16.0))
    y = (x * 2.0)[1:] + 1.0
    assert len(sess.plan([y.node])) == 1


def test_gemm_epilogue_absorption(sess):
    """np.dot boundary: GEMM -> + bias[N] -> maximum(., 0) plans as one
    Library step with a RELU_BIAS epilogue; a GEMM with another consumer, a
    non-vector bias or a disabled flag keeps the separate fused map."""
    X, W1, b1, W2, b2 = wl.mlp_inputs(batch=64, hidden=32)
    args = [gp.asarray(a) for a in (X, W1, b1, W2, b2)]
    p, lab = wl.mlp(gp, *args)
    steps = planner.plan_regions([p.node, lab.node], row_fusion=codegen.row_fusable,
                                 check=codegen.check_step, epilogues=True)
    kinds = [(s.kind, s.epilogue[0] if s.epilogue else None) for s in steps]
    assert kinds == [("Library", "relu_bias"), ("Library", "bias"), ("Fused", None)]
    assert steps[0].library_node.kind is OpKind.MATMUL and steps[0].root.op.code.name == "maximum"
    off = planner.plan_regions([p.node, lab.node], row_fusion=codegen.row_fusable,
                               check=codegen.check_step, epilogues=False)
    assert [s.kind for s in off] == ["Library", "Fused", "Library", "Fused"]
    # the GEMM result also consumed elsewhere: no absorption
    h = args[0] @ args[1]
    y = gp.maximum(h + args[2], 0)
    t = h.sum()
    st = planner.plan_regions([y.node, t.node], row_fusion=codegen.row_fusable,
                              check=codegen.check_step, epilogues=True)
    assert all(s.epilogue is None for s in st)
    # a [M, N] addend is not a bias vector
    z = args[0] @ args[1] + gp.asarray(np.ones((64, 32), np.float32))
    st = planner.plan_regions([z.node], row_fusion=codegen.row_fusable, check=codegen.check_step, epilogues=True)
    assert all(s.epilogue is None for s in st)
    # plan-cache instantiation carries the epilogue
    key, order = planner.dag_signature([p.node, lab.node])
    tmpl = planner.make_template(steps, order)
    again = planner.instantiate(tmpl, order)
    assert again[0].epilogue[0] == "relu_bias" and again[0].epilogue[1] is steps[0].epilogue[1]


def test_skinny_product_plans_inside_the_row_region(sess):
    """C4 layer 2 at the config batch: h @ W2 (N = 10) + b2 + softmax + argmax
    is ONE fused row step after the layer-1 library call (gr_skinny.cuh
    prologue); below the row threshold it stays a library step."""
    from paper_1901_03771_b200 import codegen_rows
    X, W1, b1, W2, b2 = wl.mlp_inputs(batch=8192, hidden=256)
    args = [gp.asarray(a) for a in (X, W1, b1, W2, b2)]
    p, lab = wl.mlp(gp, *args)
    steps = planner.plan_regions([p.node, lab.node], row_fusion=codegen.row_fusable, check=codegen.check_step,
                                 epilogues=True, skinny=codegen_rows.skinny_ok)
    assert [(s.kind, s.epilogue[0] if s.epilogue else None) for s in steps] == [("Library", "relu_bias"),
                                                                                 ("Fused", None)]
    fused = steps[1]
    assert any(n.kind is OpKind.MATMUL for n in fused.nodes)
    region = codegen.canonicalize(codegen.Region(fused.roots, fused.leaves, fused.nodes))
    ks = codegen.generate(region)
    assert ks.meta["skinny"][:2] == (256, 10) and ks.meta["tmaps"] and ks.block == codegen_rows.SKINNY_BLOCK
    assert "gr::Skinny<" in ks.source and "__grid_constant__" in ks.source
    small = [gp.asarray(a) for a in wl.mlp_inputs(batch=1024, hidden=256)]
    p2, lab2 = wl.mlp(gp, *small)
    st2 = planner.plan_regions([p2.node, lab2.node], row_fusion=codegen.row_fusable, check=codegen.check_step,
                               epilogues=True, skinny=codegen_rows.skinny_ok)
    assert [s.kind for s in st2] == ["Library", "Library", "Fused"]


def test_skinny_ineligible_shapes(sess):
    from paper_1901_03771_b200 import codegen_rows
    A = gp.asarray(np.ones((8192, 100), np.float32))      # K not a multiple of 32
    B = gp.asarray(np.ones((100, 4), np.float32))
    assert not codegen_rows.skinny_ok((A @ B).node)
    A2 = gp.asarray(np.ones((8192, 64), np.float32))
    B2 = gp.asarray(np.ones((64, 17), np.float32))        # N > 16
    assert not codegen_rows.skinny_ok((A2 @ B2).node)
    B3 = gp.asarray(np.ones((64, 16), np.float64))        # f64
    assert not codegen_rows.skinny_ok((A2 @ B3).node)
    assert codegen_rows.skinny_ok((A2 @ gp.asarray(np.ones((64, 16), np.float32))).node)
