"""Randomised lazy programs vs the eager oracle on the GPU (SPEC.md:464-467,
534: ranks <= 3, extents <= 16, depth <= 12, all op kinds; exact for integer
and bool results, 1e-5 rel for f32, 1e-12 rel for f64 — with an absolute floor
scaled by the operands for cancelling sums) and the committed config fixtures.

GRUMPY_RANDOM_PROGRAMS (default 120) sets the number of programs; the
acceptance run uses 1000 (each program compiles its own kernels with NVRTC)."""
import os

import numpy as np
import pytest

import paper_1901_03771_b200 as gp
from paper_1901_03771_b200 import workloads as wl
from oracle import eager
from random_programs import GP, check_outputs, make_program

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
NPROG = int(os.environ.get("GRUMPY_RANDOM_PROGRAMS", "120"))


@pytest.mark.parametrize("seed", range(NPROG))
def test_random_program(sess, seed):
    outs, transcendental, depth = make_program(seed, GP())
    expect = [eager.evaluate(o.node) for o in outs]
    gp.force(*outs)
    got = [np.asarray(o) for o in outs]
    bad = check_outputs(seed, got, expect)
    assert not bad, (seed, [o.node for o in outs], bad)
    for o, g, e in zip(outs, got, expect):
        if not transcendental and e.dtype.kind == "f" and o.node.kind.value == "MapElementwise":
            # +,-,*,/,sqrt,max and casts are IEEE-exact: bit-identical to NumPy
            assert np.array_equal(g, e, equal_nan=True), (seed, "not bit-exact", o.node)


def test_config_fixtures(sess):
    f = np.load(os.path.join(GOLD, "configs_small.npz"))
    out = wl.listing1(gp, gp.asarray(f["l1_W"]), gp.asarray(f["l1_a"]), gp.asarray(f["l1_b"]))
    assert np.array_equal(np.asarray(out), f["l1_out"])
    for tag, tol in (("f32", 1e-5), ("f64", 1e-12)):
        S, X, T = f[f"bs{tag}_S"], f[f"bs{tag}_X"], f[f"bs{tag}_T"]
        c, p = wl.blackscholes(gp, gp.asarray(S), gp.asarray(X), gp.asarray(T))
        scale = np.maximum(S, X)
        assert np.all(np.abs(np.asarray(c) - f[f"bs{tag}_call"]) <= tol * scale)
        assert np.all(np.abs(np.asarray(p) - f[f"bs{tag}_put"]) <= tol * scale)
    y, t = wl.rownorm(gp, gp.asarray(f["rn_x"]))
    gp.force(y, t)
    assert np.array_equal(np.asarray(y), f["rn_y"]) and np.asarray(t) == f["rn_total"]
    pr, lab = wl.mlp(gp, *(gp.asarray(f[k]) for k in ("mlp_X", "mlp_W1", "mlp_b1", "mlp_W2", "mlp_b2")))
    gp.force(pr, lab)
    np.testing.assert_allclose(np.asarray(pr), f["mlp_p"], rtol=1e-4, atol=1e-6)
    assert np.mean(np.asarray(lab) == f["mlp_lab"]) >= 0.999   # GEMM order differs from OpenBLAS
    klab, ksums, kcounts = wl.kmeans_partials(gp, gp.asarray(f["km_P"]), gp.asarray(f["km_C"]))
    gp.force(klab, *ksums, kcounts)
    assert np.array_equal(np.asarray(klab), f["km_lab"])
    assert np.array_equal(np.asarray(kcounts), f["km_counts"])
    np.testing.assert_allclose(np.stack([np.asarray(s) for s in ksums], 1), f["km_sums"], rtol=1e-12, atol=1e-9)
