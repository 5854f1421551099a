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
from random_programs import GP, Numpy, make_program

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
NPROG = int(os.environ.get("GRUMPY_RANDOM_PROGRAMS", "120"))


def _within(got, wide, native, mag, eps, depth):
    """Per element: the device's error against an extended-precision run of
    the same program is at most 4x NumPy's own error plus
    64*(depth+2)*eps times the element's magnitude run (sum of |terms|)."""
    got = np.asarray(got)
    fin = np.isfinite(wide.astype(np.float64)) & np.isfinite(native)
    if not np.array_equal(np.isnan(got[~fin]), np.isnan(native[~fin])):
        return False, "nan positions"
    nn = ~fin & ~np.isnan(native)
    if not np.array_equal(got[nn], native[nn]):
        return False, "inf values"
    g = got[fin].astype(np.longdouble)
    w = wide[fin].astype(np.longdouble)
    n = native[fin].astype(np.longdouble)
    m = np.abs(mag[fin].astype(np.longdouble))
    bound = 4 * np.abs(n - w) + 64 * (depth + 2) * eps * m + np.longdouble(1e-300)
    err = np.abs(g - w)
    bad = int(np.count_nonzero(~(err <= bound)))
    return bad == 0, f"{bad} elements over the bound; worst err/bound {float(np.max(err / bound)) if err.size else 0:.3g}"


@pytest.mark.parametrize("seed", range(NPROG))
def test_random_program(sess, seed):
    outs, transcendental, depth = make_program(seed, GP())
    expect = [eager.evaluate(o.node) for o in outs]
    native, _t, _d = make_program(seed, Numpy())
    wide, _t, _d = make_program(seed, Numpy(wide=True))
    mag, _t, _d = make_program(seed, Numpy(absolute=True))
    f32_ancestry = any(getattr(n, "dtype", None) is not None and np.dtype(n.dtype.np) == np.float32
                       for n in _ancestry([o.node for o in outs]))
    gp.force(*outs)
    for o, e, nv, wv, mv in zip(outs, expect, native, wide, mag):
        got = np.asarray(o)
        nv = np.asarray(nv)
        assert got.shape == e.shape == nv.shape and got.dtype == e.dtype == nv.dtype
        if e.dtype.kind in "biu":
            assert np.array_equal(got, e) and np.array_equal(got, nv), (seed, o.node)
            continue
        eps = 2.0 ** -24 if (e.dtype == np.float32 or f32_ancestry) else 2.0 ** -53
        ok, why = _within(got, np.asarray(wv), nv, np.asarray(mv), eps, depth)
        assert ok, (seed, o.node, why)
        if not transcendental and o.node.kind.value == "MapElementwise":
            # +,-,*,/,sqrt,max and casts are IEEE-exact: bit-identical to NumPy
            assert np.array_equal(got, e, equal_nan=True), (seed, "not bit-exact", o.node)


def _ancestry(roots):
    seen, stack = {}, list(roots)
    while stack:
        n = stack.pop()
        if n.id in seen:
            continue
        seen[n.id] = n
        stack.extend(n.preds)
    return seen.values()


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
