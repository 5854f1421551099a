"""GPU parity for regions with reductions (K2-K5) against the NumPy oracle.

Float sums are generated in NumPy's pairwise order, so sums of IEEE-exact
terms are asserted bit-exact; transcendental terms use the stated tolerance.
"""
import numpy as np
import pytest

import paper_1901_03771_b200 as gp
from paper_1901_03771_b200 import workloads as wl
from oracle import eager

pytestmark = pytest.mark.gpu


def test_rownorm_exact(sess):
    (x,) = wl.rownorm_inputs(rows=512, cols=256)
    y, tot = wl.rownorm(gp, gp.asarray(x))
    gp.force(y, tot)
    assert sess.stats.kernels_executed == 1
    ey, et = wl.rownorm(np, x)
    assert np.array_equal(np.asarray(y), ey)
    assert np.asarray(tot) == et


@pytest.mark.parametrize("store_y", [False, True])
def test_rownorm_division_window_redo(sess, store_y):
    """Rows whose dividends leave the shared-divisor window (exact zeros,
    denormal-range values, a zero std, inf/nan) take the exact redo pass of
    the two-pass division; every row must still match NumPy bit for bit."""
    rng = np.random.default_rng(21)
    x = (rng.standard_normal((64, 4096)) * 2 + 5).astype(np.float32)
    x[3, :] = 7.0                        # std 0: 0/0 -> nan everywhere
    x[5, ::2] = 1.0
    x[5, 1::2] = -1.0                    # x - mean == ±1 exactly, mean 0
    x[9, :] = 0.0
    x[9, 17] = 1e-30                     # tiny dividends
    x[11, 100] = np.inf                  # inf / nan propagation
    x[12, 7] = np.nan
    x[20, :] = rng.standard_normal(4096).astype(np.float32) * np.float32(1e30)
    with np.errstate(all="ignore"):
        ey, et = wl.rownorm(np, x)
        y, tot = wl.rownorm(gp, gp.asarray(x))
        if store_y:
            gp.force(y, tot)
            assert np.array_equal(np.asarray(y), ey, equal_nan=True)
        got = np.asarray(tot)
    assert np.array_equal(got, et, equal_nan=True)
    # and without the pathological rows the fast pass alone is exact
    xs = np.delete(x, [3, 5, 9, 11, 12, 20], axis=0)
    ey, et = wl.rownorm(np, xs)
    y, tot = wl.rownorm(gp, gp.asarray(xs))
    gp.force(y, tot)
    assert np.array_equal(np.asarray(y), ey) and np.asarray(tot) == et


def test_softmax_argmax(sess):
    rng = np.random.default_rng(3)
    z = rng.standard_normal((1000, 10)).astype(np.float32)
    gz = gp.asarray(z)
    p = gp.exp(gz - gz.max(1)[:, None])
    p = p / p.sum(1)[:, None]
    lab = p.argmax(1)
    gp.force(p, lab)
    assert sess.stats.kernels_executed == 1
    ep = np.exp(z - z.max(1)[:, None])
    ep = ep / ep.sum(1)[:, None]
    np.testing.assert_allclose(np.asarray(p), ep, rtol=1e-5, atol=1e-7)
    assert np.array_equal(np.asarray(lab), ep.argmax(1))


def test_kmeans_labels_exact(sess):
    P, C = wl.kmeans_inputs(n=1 << 14, k=64, d=4)
    lab = wl.kmeans_assign(gp, gp.asarray(P), gp.asarray(C))
    assert np.array_equal(np.asarray(lab), wl.kmeans_assign(np, P, C))
    assert sess.stats.kernels_executed == 1


@pytest.mark.parametrize("shape,axis", [((300, 50), 0), ((300, 50), 1), ((7, 9, 11), (0, 2)),
                                        ((7, 9, 11), 1), ((1 << 16,), None), ((512, 256), None),
                                        ((1000, 3), None)])
def test_sum_axes_exact(sess, shape, axis):
    rng = np.random.default_rng(4)
    x = rng.standard_normal(shape).astype(np.float32)
    g = gp.asarray(x).sum(axis=axis)
    assert np.array_equal(np.asarray(g), x.sum(axis=axis))


@pytest.mark.parametrize("op", ["max", "min", "argmax", "argmin", "mean", "std", "prod"])
def test_reductions_misc(sess, op):
    rng = np.random.default_rng(5)
    x = rng.standard_normal((257, 33))
    x[3, 7] = np.nan
    for axis in (None, 0, 1):
        got = np.asarray(getattr(gp.asarray(x), op)(axis=axis))
        exp = getattr(x, op)(axis=axis)
        if op in ("argmax", "argmin", "max", "min"):
            assert np.array_equal(got, exp, equal_nan=True), (op, axis)
        else:
            np.testing.assert_allclose(got, exp, rtol=1e-12, equal_nan=True)


def test_int_and_bool_reductions(sess):
    rng = np.random.default_rng(6)
    a = rng.integers(-1000, 1000, (123, 45)).astype(np.int32)
    g = gp.asarray(a)
    assert np.array_equal(np.asarray(g.sum(1)), a.sum(1))
    assert np.asarray(g.sum()) == a.sum()
    assert np.array_equal(np.asarray((g > 0).any(0)), (a > 0).any(0))
    assert np.array_equal(np.asarray((g > -990).all(1)), (a > -990).all(1))
    assert np.array_equal(np.asarray(g.max(0)), a.max(0))


def test_kmeans_partials_one_kernel(sess):
    P, C = wl.kmeans_inputs(n=(1 << 15) + 17, k=64, d=4)
    lab, sums, counts = wl.kmeans_partials(gp, gp.asarray(P), gp.asarray(C))
    gp.force(lab, *sums, counts)
    assert sess.stats.kernels_executed == 1
    elab, esums, ecounts = wl.kmeans_partials(np, P, C)
    assert np.array_equal(np.asarray(lab), elab)
    assert np.array_equal(np.asarray(counts), ecounts)
    for s, e in zip(sums, esums):
        # fp64 sums of fp32 weights; order differs from NumPy's sequential loop
        np.testing.assert_allclose(np.asarray(s), e, rtol=1e-12, atol=1e-9)


def test_bincount_alone(sess):
    rng = np.random.default_rng(9)
    k = rng.integers(0, 100, 5000)
    w = rng.standard_normal(5000)
    g = gp.bincount(gp.asarray(k), weights=gp.asarray(w), minlength=100)
    np.testing.assert_allclose(np.asarray(g), np.bincount(k, weights=w, minlength=100), rtol=1e-12, atol=1e-12)
    c = gp.bincount(gp.asarray(k.astype(np.int32)), minlength=100)
    assert np.array_equal(np.asarray(c), np.bincount(k, minlength=100))


def test_region_against_eager_oracle(sess):
    rng = np.random.default_rng(7)
    x = gp.asarray(rng.standard_normal((64, 48)))
    y = gp.asarray(rng.standard_normal(48))
    r = (x * y - (x * y).mean(1, keepdims=True)).max(1) + x.sum() * 0.0
    expect = eager.evaluate(r.node)
    np.testing.assert_allclose(np.asarray(r), expect, rtol=1e-12)


def test_kmeans_nan_inf_ties_exact(sess):
    """Labels stay np.argmin-exact on the constant-bank / NaN-rescan path:
    NaN points (first NaN index = 0), a NaN centroid (its index wins for every
    point), +inf coordinates and duplicate centroids (first index wins)."""
    P, C = wl.kmeans_inputs(n=8192 + 5, k=64, d=4)
    P[10, 2] = np.nan
    P[11] = np.inf
    P[12, 0] = -np.inf
    C[7] = C[3]                       # exact ties: index 3 must win
    P[100:200] = C[3]                 # zero distance to 3 and 7
    lab = wl.kmeans_assign(gp, gp.asarray(P), gp.asarray(C))
    assert np.array_equal(np.asarray(lab), wl.kmeans_assign(np, P, C))
    C2 = C.copy()
    C2[40, 1] = np.nan
    lab2 = wl.kmeans_assign(gp, gp.asarray(P), gp.asarray(C2))
    assert np.array_equal(np.asarray(lab2), wl.kmeans_assign(np, P, C2))


@pytest.mark.parametrize("n", [64, 10])
def test_row_argmax_nan_rows(sess, n):
    rng = np.random.default_rng(11)
    x = rng.standard_normal((5000, n)).astype(np.float32)
    x[::7, n // 2] = np.nan
    x[::11, n - 1] = np.nan
    x[3] = np.nan
    x[4] = 1.0
    g = gp.asarray(x)
    for fn in ("argmax", "argmin"):
        assert np.array_equal(np.asarray(getattr(g * 2.0, fn)(1)), getattr(x * 2.0, fn)(1)), fn


@pytest.mark.parametrize("nkeys", [1, 3, 64])
def test_bincount_collisions(sess, nkeys):
    """Warp groups of equal keys (__match_any_sync) up to a whole warp."""
    rng = np.random.default_rng(12)
    k = rng.integers(0, nkeys, 10007)
    w = rng.standard_normal(10007)
    g = gp.bincount(gp.asarray(k), weights=gp.asarray(w), minlength=64)
    np.testing.assert_allclose(np.asarray(g), np.bincount(k, weights=w, minlength=64), rtol=1e-12, atol=1e-9)
    c = gp.bincount(gp.asarray(k), minlength=64)
    assert np.array_equal(np.asarray(c), np.bincount(k, minlength=64))


def test_kmeans_paired_loop_exact(sess, monkeypatch):
    """The paired argmin loop (the NumPy-order scan, here without the
    nearest-centre search in front of it) keeps np.argmin's answer."""
    from paper_1901_03771_b200 import codegen, codegen_rows
    monkeypatch.setattr(codegen_rows, "PAIR_LOOPS", True)
    monkeypatch.setattr(codegen_rows, "NEAREST", False)
    codegen._GEN_CACHE.clear()
    sess._plan_cache.clear()
    try:
        P, C = wl.kmeans_inputs(n=8192 + 5, k=64, d=4)
        P[10, 2] = np.nan
        C[7] = C[3]
        lab = wl.kmeans_assign(gp, gp.asarray(P), gp.asarray(C))
        got = np.asarray(lab)
        assert "gr::p2::" in sess.executor.last_steps[0].cache["ks"].source
        assert np.array_equal(got, wl.kmeans_assign(np, P, C))
    finally:
        codegen._GEN_CACHE.clear()


def test_kmeans_lloyd_iterations_exact(sess):
    """Several Lloyd iterations through one compiled kernel: the centroid
    leaf (constant bank + its pair-adjacent repacked copy) changes every
    launch and the labels must track NumPy's every time."""
    P, C = wl.kmeans_inputs(n=(1 << 14) + 3, k=64, d=4, seed=5)
    gP = gp.asarray(P)
    for _ in range(4):
        lab, sums, counts = wl.kmeans_partials(gp, gP, gp.asarray(C))
        gp.force(lab, *sums, counts)
        elab, esums, ecounts = wl.kmeans_partials(np, P, C)
        assert np.array_equal(np.asarray(lab), elab)
        assert np.array_equal(np.asarray(counts), ecounts)
        C = wl.kmeans_centroids(esums, ecounts, C)


@pytest.mark.parametrize("K,D,scale", [(64, 4, 1.0), (2, 1, 1e-3), (8, 3, 50.0), (256, 8, 1e4), (16, 2, 1e-20),
                                       (64, 4, 1e3)])
def test_nearest_centre_certified_exact(sess, K, D, scale):
    """The certified expanded-key search (gr_nearest.cuh) with its exact
    fallback: labels equal np.argmin on adversarial inputs — points on
    bisectors (exact ties), a few ulps off them, on centres, duplicated
    centres, far points, non-finite coordinates — and bincount partials of
    the same region stay right."""
    rng = np.random.default_rng([K, D])
    C = (rng.standard_normal((K, D)) * scale).astype(np.float32)
    if K >= 4:
        C[K // 2] = C[1]
    n = 40000
    P = (C[rng.integers(0, K, n)] + rng.standard_normal((n, D)).astype(np.float32) * np.float32(scale * 0.5)).astype(np.float32)
    i, j = rng.integers(0, K, 3000), rng.integers(0, K, 3000)
    P[:3000] = ((C[i].astype(np.float64) + C[j]) / 2).astype(np.float32)
    P[3000:6000] = (P[:3000] * (1 + rng.integers(-4, 5, (3000, 1)) * np.float32(2 ** -23))).astype(np.float32)
    P[6000:6100] = C[rng.integers(0, K, 100)]
    P[6100] *= np.float32(1e3)
    P[6101, 0] = np.nan
    P[6102] = np.inf
    P[6103, -1] = np.float32(3e19)
    lab = wl.kmeans_assign(gp, gp.asarray(P), gp.asarray(C))
    got = np.asarray(lab)
    assert "gr::nearest_centre" in sess.executor.last_steps[0].cache["ks"].source
    assert np.array_equal(got, wl.kmeans_assign(np, P, C))
    C2 = C.copy()
    C2[K - 1, 0] = np.nan                  # a NaN centre: every row takes the exact scan
    assert np.array_equal(np.asarray(wl.kmeans_assign(gp, gp.asarray(P), gp.asarray(C2))), wl.kmeans_assign(np, P, C2))


def test_nearest_centre_off_matches(sess, monkeypatch):
    """GRUMPY_NEAREST=0 (the NumPy-order scan alone) gives the same labels."""
    from paper_1901_03771_b200 import codegen, codegen_rows
    P, C = wl.kmeans_inputs(n=(1 << 15) + 3, k=64, d=4)
    on = np.asarray(wl.kmeans_assign(gp, gp.asarray(P), gp.asarray(C)))
    monkeypatch.setattr(codegen_rows, "NEAREST", False)
    codegen._GEN_CACHE.clear()
    sess._plan_cache.clear()
    try:
        off = wl.kmeans_assign(gp, gp.asarray(P), gp.asarray(C))
        got = np.asarray(off)
        assert "gr::nearest_centre" not in sess.executor.last_steps[0].cache["ks"].source
    finally:
        codegen._GEN_CACHE.clear()
    assert np.array_equal(on, got) and np.array_equal(on, wl.kmeans_assign(np, P, C))


@pytest.mark.parametrize("blocked", [False, True])
@pytest.mark.parametrize("rows", [8192, 16384])
@pytest.mark.parametrize("store_y", [False, True])
def test_rownorm_blocked_total_with_redo(sess, monkeypatch, blocked, rows, store_y):
    """Totals over many rows with rows redone exactly: the last CTA's batched
    fold (default) and the per-4096-row-block warp folds (codegen_coop
    TOT_BLOCK, GRUMPY_COOP_BLOCKED_TOTAL=1) are bit-identical to NumPy, also
    when rows of several blocks take the exact redo pass (counted only after
    their redo) and across repeated launches (counters reset)."""
    from paper_1901_03771_b200 import codegen, codegen_coop
    monkeypatch.setattr(codegen_coop, "COOP_BLOCKED_TOTAL", blocked)
    codegen._GEN_CACHE.clear()
    sess._plan_cache.clear()
    rng = np.random.default_rng([rows, store_y])
    x = (rng.standard_normal((rows, 4096)) * 2 + 5).astype(np.float32)
    # rows whose mean (exactly 2.0) equals two of their elements: a zero
    # dividend leaves the shared-divisor window, the row is redone exactly;
    # the std stays normal, so the total is finite
    pat = np.where(np.arange(4096) % 2 == 0, 1.0, 3.0).astype(np.float32)
    pat[0], pat[1] = 2.0, 2.0
    for r in (5, 4100, rows - 1):
        x[r, :] = pat
    x[4097, ::2] = 1.0
    x[4097, 1::2] = -1.0
    ey, et = wl.rownorm(np, x)
    gx = gp.asarray(x)
    for _ in range(3):
        y, tot = wl.rownorm(gp, gx)
        if store_y:
            gp.force(y, tot)
            assert np.array_equal(np.asarray(y), ey)
        assert np.isfinite(et) and np.asarray(tot) == et
    assert ("fold_block" in sess.executor.last_steps[0].cache["ks"].source) == blocked
    codegen._GEN_CACHE.clear()
