"""GPU parity for map-scan kernels and slice / slice-assign
regions (the Jacobi sweep)."""
import numpy as np
import pytest

import paper_1901_03771_b200 as gp
from paper_1901_03771_b200 import workloads as wl

pytestmark = pytest.mark.gpu


def test_scan_kats(sess):
    """SPEC.md:388-390."""
    assert np.asarray(gp.asarray(np.array([1, 2, 3])).cumsum()).tolist() == [1, 3, 6]
    assert np.asarray(gp.asarray(np.zeros(4)).cumsum()).tolist() == [0, 0, 0, 0]
    assert np.asarray(np.maximum.accumulate(gp.asarray(np.array([3, 1, 4, 1, 5])))).tolist() == [3, 3, 4, 4, 5]


@pytest.mark.parametrize("shape,axis", [((300, 50), 0), ((30, 500), 1), ((7, 9, 11), 1), ((3, 4, 5), None)])
def test_scan_lines_exact(sess, shape, axis):
    rng = np.random.default_rng(5)
    x = rng.standard_normal(shape)
    g = (gp.asarray(x) * 2 + 1).cumsum(axis=axis)
    assert np.array_equal(np.asarray(g), (x * 2 + 1).cumsum(axis=axis))   # sequential fold = NumPy


@pytest.mark.parametrize("shape", [(1000, 300), (33, 65), (4096, 64), (5, 40, 129), (64, 2), (2048, 1000)])
@pytest.mark.parametrize("kind", ["f32", "f64", "i64", "i32", "prod", "max", "rowvec", "colvec"])
def test_scan_rows_contiguous_axis(sess, shape, kind):
    """Scans along the last axis (codegen_scan._gen_rows_t: a warp per 32
    lines, coalesced through a shared tile) keep NumPy's sequential fold per
    line: bit-identical to np.cumsum / cumprod / maximum.accumulate, including
    NaN propagation, broadcast operands along either axis, and line counts and
    lengths that are not multiples of 32 or of the 64-column chunk."""
    from paper_1901_03771_b200 import codegen
    rng = np.random.default_rng([len(shape), shape[-1], len(kind)])
    if kind in ("i64", "i32"):
        x = rng.integers(-50, 50, shape).astype(np.int64 if kind == "i64" else np.int32)
    elif kind == "f64":
        x = rng.standard_normal(shape)
    else:
        x = rng.standard_normal(shape).astype(np.float32)
    g = gp.asarray(x)
    if kind == "prod":
        xs = (x * np.float32(0.01) + np.float32(1.0))
        got, ref = gp.cumprod(g * 0.01 + 1.0, axis=-1), np.cumprod(xs, axis=-1)
    elif kind == "max":
        x[..., shape[-1] // 2] = np.nan
        got, ref = np.maximum.accumulate(gp.asarray(x), axis=-1), np.maximum.accumulate(x, axis=-1)
    elif kind == "rowvec":
        c = rng.standard_normal(shape[-1]).astype(np.float32)
        got, ref = gp.cumsum(g * 2.0 + gp.asarray(c), axis=-1), np.cumsum(x * np.float32(2.0) + c, axis=-1)
    elif kind == "colvec":
        c = rng.standard_normal(shape[:-1] + (1,)).astype(np.float32)
        got, ref = gp.cumsum(g - gp.asarray(c), axis=-1), np.cumsum(x - c, axis=-1)
    else:
        got, ref = gp.cumsum(g * 3 + 1, axis=-1), np.cumsum(x * 3 + 1, axis=-1)
    out = np.asarray(got)
    assert sess.executor.last_steps[-1].cache["ks"].meta.get("label") == "scan-rows"
    assert out.dtype == ref.dtype and out.shape == ref.shape
    assert np.array_equal(out, ref, equal_nan=kind not in ("i64", "i32"))


@pytest.mark.parametrize("case", ["f32", "f64-3d", "i64", "tail", "rowvec", "transposed"])
def test_scan_flat_nd(sess, case):
    """cumsum of an n-D operand without an axis scans its flat row-major
    order: identity-mapped contiguous leaves are staged by TMA like a 1-D
    scan (tail past the last 128-byte line included); broadcast or
    transposed leaves fall back to the register-staged kernel.  Integers
    exact, floats within the 1-D scan's bound."""
    rng = np.random.default_rng(len(case))
    shape = {"f64-3d": (4, 512, 1001), "tail": (1025, 1031)}.get(case, (1024, 1500))
    if case == "i64":
        a, b = rng.integers(-50, 50, shape), rng.integers(-3, 3, shape)
    else:
        dt = np.float64 if case == "f64-3d" else np.float32
        a, b = rng.standard_normal(shape).astype(dt), rng.standard_normal(shape).astype(dt)
    ga, gb = gp.asarray(a), gp.asarray(b)
    if case == "rowvec":
        c = rng.standard_normal(shape[-1]).astype(np.float32)
        got, t = gp.cumsum(ga + gp.asarray(c)), a + c
    elif case == "transposed":
        bt = np.ascontiguousarray(b.T)
        got, t = gp.cumsum(ga * gp.asarray(bt).T), a * bt.T
    else:
        got, t = gp.cumsum(ga * gb + 1), a * b + 1
    out = np.asarray(got)
    label = sess.executor.last_steps[-1].cache["ks"].meta.get("label")
    assert label == ("scan-lookback" if case in ("rowvec", "transposed") else "scan-tma")
    if case == "i64":
        assert np.array_equal(out, np.cumsum(t))
        return
    ref = np.cumsum(t.astype(np.float64))
    bound = np.cumsum(np.abs(t.astype(np.float64)))
    tiles = -(-t.size // (8192 if t.dtype == np.float32 else 4096))
    assert np.all(np.abs(out - ref) <= (tiles + 32) * np.finfo(t.dtype).eps * bound)


@pytest.mark.parametrize("view", ["T", "step", "cols", "big-T"])
def test_scan_last_axis_of_views(sess, view):
    """Scans along the last axis of transposed / strided / column-sliced views
    (the leaves are read through their index maps, not staged): NumPy's
    sequential fold per line, bit-exact, whichever kernel takes them."""
    rng = np.random.default_rng(len(view))
    x = rng.standard_normal((2048, 3000) if view == "big-T" else (600, 700)).astype(np.float32)
    g = gp.asarray(x)
    if view in ("T", "big-T"):
        got, ref = gp.cumsum(g.T * 2.0, axis=-1), np.cumsum(x.T * np.float32(2.0), axis=-1)
    elif view == "step":
        got, ref = gp.cumsum(g[:, ::2] + 1.0, axis=1), np.cumsum(x[:, ::2] + np.float32(1.0), axis=1)
    else:
        got, ref = gp.cumsum(g[100:, 5:605] - 0.5, axis=1), np.cumsum(x[100:, 5:605] - np.float32(0.5), axis=1)
    assert np.array_equal(np.asarray(got), ref)


@pytest.mark.parametrize("shape", [(64, 65536), (4, 8, 1 << 16), (1024, 16384), (3, 1 << 20),
                                   (64, 100003), (16, 70001), (300, 16388), (7, 3, 50021)])
@pytest.mark.parametrize("kind", ["f32", "f64", "i64", "max", "colvec"])
def test_scan_rows_segmented_lookback(sess, shape, kind):
    """Few long lines scanned along the last axis run as one look-back scan per
    line (segments: a tile's fold never reaches below its line's first tile) —
    the TMA kernel when every line is whole tiles, else the register-staged
    kernel with a partial last tile per line.  Integers and max exact; float
    sums within the reassociation bound of the 1-D scan, per line."""
    rng = np.random.default_rng([shape[-1], len(kind)])
    if kind == "i64":
        x = rng.integers(-50, 50, shape)
    elif kind == "f64":
        x = rng.standard_normal(shape)
    else:
        x = rng.standard_normal(shape).astype(np.float32)
    g = gp.asarray(x)
    if kind == "max":
        x.reshape(-1)[x.size // 3] = np.nan
        out = np.asarray(np.maximum.accumulate(gp.asarray(x), axis=-1))
        assert sess.executor.last_steps[-1].cache["ks"].meta.get("label") in ("scan-tma", "scan-lookback")
        assert np.array_equal(out, np.maximum.accumulate(x, axis=-1), equal_nan=True)
        return
    if kind == "colvec":
        c = rng.standard_normal(shape[:-1] + (1,)).astype(np.float32)
        out, t = np.asarray(gp.cumsum(g * 0.5 - gp.asarray(c), axis=-1)), x * np.float32(0.5) - c
    else:
        out, t = np.asarray(gp.cumsum(g * 3 + 1, axis=-1)), x * 3 + 1
    whole = shape[-1] % (8192 if x.dtype.itemsize == 4 else 4096) == 0
    assert sess.executor.last_steps[-1].cache["ks"].meta.get("label") == ("scan-tma" if whole else "scan-lookback")
    if kind == "i64":
        assert np.array_equal(out, np.cumsum(t, axis=-1))
        return
    ref = np.cumsum(t.astype(np.float64), axis=-1)
    bound = np.cumsum(np.abs(t.astype(np.float64)), axis=-1)
    eps = np.finfo(t.dtype).eps
    tiles = -(-shape[-1] // (8192 if t.dtype == np.float32 else 4096))
    assert np.all(np.abs(out - ref) <= (tiles + 32) * eps * bound)


@pytest.mark.parametrize("n", [8193, 100000, 1 << 22])
def test_scan_lookback(sess, n):
    rng = np.random.default_rng(6)
    xi = rng.integers(-100, 100, n)
    assert np.array_equal(np.asarray(gp.asarray(xi).cumsum()), xi.cumsum())          # integers exact
    xf = rng.standard_normal(n)
    got = np.asarray(gp.exp(gp.asarray(xf) * 0.1).cumsum())
    ref = np.exp(xf * 0.1).cumsum()
    # reassociated fp64 prefix sums: measured against an extended-precision
    # prefix, the look-back scan must be no less accurate than NumPy's own
    # sequential fold (within 2x, plus one ulp of the running total)
    exact = np.cumsum(np.exp(xf * 0.1).astype(np.longdouble))
    err_ref = float(np.max(np.abs(ref - exact)))
    err_got = float(np.max(np.abs(got - exact)))
    assert err_got <= 2 * err_ref + 2.2e-16 * float(exact[-1])
    m = np.asarray(np.maximum.accumulate(gp.asarray(xf)))
    assert np.array_equal(m, np.maximum.accumulate(xf))


def test_jacobi_sweep_one_kernel(sess):
    """one slice-assign sweep is exactly one fused map kernel."""
    rng = np.random.default_rng(7)
    a = rng.standard_normal((66, 66))
    b = rng.standard_normal((66, 66))
    ga, gb = gp.asarray(a), gp.asarray(b)
    gb[1:-1, 1:-1] = 0.2 * (ga[1:-1, 1:-1] + ga[1:-1, :-2] + ga[1:-1, 2:] + ga[:-2, 1:-1] + ga[2:, 1:-1])
    k0 = sess.stats.kernels_executed
    got = np.asarray(gb)
    assert sess.stats.kernels_executed - k0 == 1
    b[1:-1, 1:-1] = 0.2 * (a[1:-1, 1:-1] + a[1:-1, :-2] + a[1:-1, 2:] + a[:-2, 1:-1] + a[2:, 1:-1])
    assert np.array_equal(got, b)


def test_views_strided(sess):
    rng = np.random.default_rng(8)
    t = rng.standard_normal((8, 6, 4)).astype(np.float32)
    g = gp.asarray(t).transpose(2, 0, 1).reshape(4, 48)[:, ::3] * 2 + gp.asarray(t)[::-1, 0, :].T.sum(1)[:, None]
    e = t.transpose(2, 0, 1).reshape(4, 48)[:, ::3] * 2 + t[::-1, 0, :].T.sum(1)[:, None]
    # the strided views themselves are exact (gathers); the f32 sum over a
    # reversed, non-contiguous axis is summed by NumPy's iterator in MEMORY
    # order (it flips negative strides), which a logical-order fold does not
    # reproduce bit-for-bit: f32 tolerance (rel 1e-5)
    assert np.array_equal(np.asarray(gp.asarray(t).transpose(2, 0, 1).reshape(4, 48)[:, ::3]),
                          t.transpose(2, 0, 1).reshape(4, 48)[:, ::3])
    assert np.array_equal(np.asarray(gp.asarray(t)[::-1, 0, :].T), t[::-1, 0, :].T)
    np.testing.assert_allclose(np.asarray(g), e, rtol=1e-5, atol=1e-6)


@pytest.mark.parametrize("shape,dt", [((256, 256), np.float32), ((258, 300), np.float32), ((6, 10), np.float32),
                                      ((130, 64), np.float64), ((3, 8), np.float64), ((1024, 12), np.int32)])
def test_jacobi_fast_interior_groups(sess, shape, dt):
    """Interior lane groups take the unclamped, vectorised form (shifted-vector
    neighbours); boundary groups the clamped select form: bit-identical."""
    from paper_1901_03771_b200 import codegen
    rng = np.random.default_rng(17)
    a = (rng.standard_normal(shape) * 8).astype(dt)
    b = wl.jacobi(gp, gp.asarray(a))
    got = np.asarray(b)
    assert np.array_equal(got, wl.jacobi(np, a))
    ks = sess.executor.last_steps[-1].cache["ks"]
    assert ks.family == "map" and (ks.meta.get("fast_group") or ks.vec == 1)


def test_shifted_vector_slices(sess):
    """Neighbour differences at constant misalignments read two aligned
    vectors (gr::pick) instead of per-lane gathers: exact for every shift."""
    rng = np.random.default_rng(18)
    x = rng.standard_normal(4096 + 8).astype(np.float32)
    g = gp.asarray(x)
    for lo, hi in ((1, 0), (0, 1), (3, 1), (2, 6), (5, 3)):
        n = 4096
        got = np.asarray(g[lo:lo + n] - g[hi:hi + n] * 0.5)
        assert np.array_equal(got, x[lo:lo + n] - x[hi:hi + n] * np.float32(0.5)), (lo, hi)
    m = rng.standard_normal((64, 72)).astype(np.float64)
    gm = gp.asarray(m)
    assert np.array_equal(np.asarray(gm[:, 1:] + gm[:, :-1]), m[:, 1:] + m[:, :-1])


def test_scan_lookback_deterministic(sess):
    """The tile-tree prefix folds a fixed association of tile aggregates:
    repeated runs are bit-identical (timing cannot change the result)."""
    rng = np.random.default_rng(9)
    x = rng.standard_normal((1 << 22) + 1234).astype(np.float32)
    g = gp.asarray(x)
    runs = [np.asarray(gp.cumsum(g * 0.5 + 1.0)) for _ in range(3)]
    assert all(np.array_equal(runs[0], r) for r in runs[1:])
    ref = np.cumsum((x * np.float32(0.5) + np.float32(1.0)).astype(np.float64))
    assert np.max(np.abs(runs[0] - ref)) <= 1e-6 * np.max(np.abs(ref)) + 1.0


@pytest.mark.parametrize("n", [1 << 20, (1 << 22) + 32, 3 << 20, (1 << 21) + 7, (1 << 24) + 96, (1 << 20) + 8191, 5 * 8192 * 148 + 33])
@pytest.mark.parametrize("kind", ["f32", "f64", "i64", "f32x2", "max"])
@pytest.mark.parametrize("tree", [True, False])
def test_scan_tma_matches_register_staged(sess, monkeypatch, n, kind, tree):
    """The TMA-fed look-back scan (codegen_scan._gen_lookback_tma) against the
    register-staged kernel, for one- and two-leaf map prologues, 4- and 8-byte
    types, sums and max; lengths that are not a multiple of the tile
    (zero-filled last box) or of the 128-byte line (the tail elements loaded
    and stored by their threads).  With the left fold of a round's aggregates
    (tree=False) the association is that of the register-staged kernel's
    nearest-prefix walk: bits identical.  With the warp tree (the default) integers and max are still
    identical and float sums stay within the 1-D scan's reassociation bound,
    the same bits on every run."""
    from paper_1901_03771_b200 import codegen, codegen_scan
    monkeypatch.setattr(codegen_scan, "SCAN_TMA_TREE", tree)
    monkeypatch.setattr(codegen_scan, "SCAN_REG_ROUNDS", tree)     # left fold: the nearest-prefix walk
    rng = np.random.default_rng([n, len(kind)])
    if kind == "i64":
        xs = [rng.integers(-1000, 1000, n)]
    elif kind == "f64":
        xs = [rng.standard_normal(n)]
    else:
        xs = [rng.standard_normal(n).astype(np.float32) for _ in range(2 if kind == "f32x2" else 1)]

    def prog():
        g = [gp.asarray(v) for v in xs]
        if kind == "max":
            return np.maximum.accumulate(g[0] * 2.0)
        if kind == "f32x2":
            return gp.cumsum(g[0] * g[1] + 1.0)
        return gp.cumsum(g[0] * 3 + 1)

    outs, labels = [], []
    for tma in (True, True, False):
        monkeypatch.setattr(codegen_scan, "SCAN_TMA", tma)
        codegen._GEN_CACHE.clear()
        sess._plan_cache.clear()
        r = prog()
        outs.append(np.asarray(r))
        labels.append(sess.executor.last_steps[-1].cache["ks"].meta.get("label"))
    codegen._GEN_CACHE.clear()
    sess._plan_cache.clear()
    assert labels == ["scan-tma", "scan-tma", "scan-lookback"]
    assert np.array_equal(outs[0], outs[1])                      # deterministic
    if kind in ("i64", "max") or not tree:
        assert np.array_equal(outs[0], outs[2])
    else:
        t = (xs[0] * xs[1] + np.float32(1.0)) if kind == "f32x2" else xs[0] * 3 + 1
        ref = np.cumsum(t.astype(np.float64))
        bound = np.cumsum(np.abs(t.astype(np.float64)))
        tiles = -(-n // (8192 if t.dtype == np.float32 else 4096))
        eps = np.finfo(t.dtype).eps
        for o in (outs[0], outs[2]):
            assert np.all(np.abs(o - ref) <= (tiles + 32) * eps * bound)
    if kind in ("i64",):
        assert np.array_equal(outs[0], np.cumsum(xs[0] * 3 + 1))
    if kind == "max":
        assert np.array_equal(outs[0], np.maximum.accumulate(xs[0] * np.float32(2.0)))


@pytest.mark.parametrize("case", ["long-f32", "long-i64", "long-tma", "long-tma-tail", "lines-axis0", "short"])
def test_seeded_scan(sess, monkeypatch, case):
    """A scan seeded with a value (the streamed chunks' carry, streaming.py)
    folds from the seed: out[k] = seed (+) x[0] (+) ... (+) x[k]; integers
    exact, floats within the scan's association bound; the eager oracle
    agrees."""
    from paper_1901_03771_b200 import codegen, codegen_scan
    from paper_1901_03771_b200.dag import Op, OpKind
    from oracle import eager
    monkeypatch.setattr(codegen_scan, "SCAN_TMA", case.startswith("long-tma"))
    codegen._GEN_CACHE.clear()
    rng = np.random.default_rng(len(case))
    g = sess.graph
    if case == "lines-axis0":
        xh = rng.standard_normal((1 << 12, 24))
        prevh = rng.standard_normal((5, 24))
        x, prev = gp.asarray(xh), gp.asarray(prevh)
        c = gp.cumsum(x * 2.0, axis=0)
        carry = g.add_op(Op(OpKind.SLICE, None, (((4, 1, 1), (0, 1, 24)),)), [prev.node])
        carry = g.add_op(Op(OpKind.RESHAPE, None, ((24,),)), [carry])
        ref = np.cumsum(np.concatenate([prevh[4:5], xh * 2.0]), axis=0)[1:]
    else:
        n = {"short": 5000, "long-tma": (1 << 21) + 32}.get(case, (1 << 21) + 7)      # long-tma-tail: + 7
        if case == "long-i64":
            xh, prevh = rng.integers(-50, 50, n), rng.integers(-9, 9, 7)
        else:
            xh, prevh = rng.standard_normal(n).astype(np.float32), rng.standard_normal(7).astype(np.float32)
        x, prev = gp.asarray(xh), gp.asarray(prevh)
        c = gp.cumsum(x * 3 if case == "long-i64" else x * np.float32(0.5))
        carry = g.add_op(Op(OpKind.SLICE, None, (((6, 1, 1),),)), [prev.node])
        t = xh * 3 if case == "long-i64" else xh * np.float32(0.5)
        ref = np.cumsum(np.concatenate([prevh[6:7], t]).astype(np.float64 if case != "long-i64" else np.int64))[1:]
    sc = g.add_op(c.node.op, [c.node.preds[0], carry])
    got = np.asarray(gp.session._wrap(sc, sess))
    codegen._GEN_CACHE.clear()
    exp = eager.evaluate(sc)
    if case == "long-i64":
        assert np.array_equal(got, ref) and np.array_equal(exp, ref)
    else:
        scale = np.cumsum(np.abs(np.concatenate([prevh[-1:] if case != "lines-axis0" else prevh[4:5], xh])), axis=0)[1:]
        assert np.all(np.abs(got - ref) <= 1e-5 * (scale + 1))
        assert np.all(np.abs(exp - ref) <= 1e-5 * (scale + 1))
    label = sess.executor.last_steps[-1].cache["ks"].meta.get("label")
    assert label == {"long-tma": "scan-tma", "long-tma-tail": "scan-tma", "long-f32": "scan-lookback",
                     "long-i64": "scan-lookback"}.get(case, label)


def _scan_case(rng, i):
    """A random scan program: shape, axis, op and dtype chosen to reach every
    scan kernel (lines, warp-per-lines, segmented TMA / register-staged,
    flat TMA with and without a tail, 1-D register-staged)."""
    kind = i % 8
    if kind == 0:
        shape, axis = (int(rng.integers(2, 40)), int(rng.integers(2, 300))), 0
    elif kind == 1:
        shape, axis = (int(rng.integers(32, 3000)), int(rng.integers(2, 700))), 1
    elif kind == 2:
        shape, axis = (int(rng.integers(1, 40)), 8192 * int(rng.integers(4, 40))), -1
    elif kind == 3:
        shape, axis = (int(rng.integers(1, 40)), int(rng.integers(20000, 200000))), -1
    elif kind == 4:
        shape, axis = (int(rng.integers(300, 1500)), int(rng.integers(700, 3000))), None
    elif kind == 5:
        shape, axis = (int(rng.integers(1 << 20, 3 << 20)),), None
    elif kind == 6:
        shape, axis = (int(rng.integers(9000, 1 << 20)),), None
    else:
        shape, axis = (int(rng.integers(2, 6)), int(rng.integers(2, 9)), int(rng.integers(20000, 90000))), -1
    dt = [np.float32, np.float64, np.int64, np.int32][int(rng.integers(0, 4))]
    op = ["sum", "max", "prod"][int(rng.integers(0, 3))] if dt != np.float64 else "sum"
    return shape, axis, dt, op


@pytest.mark.parametrize("i", range(40))
def test_scan_random_shapes(sess, i):
    """Randomized scans against NumPy: integers and max exact, sums and
    products of floats within the look-back's reassociation bound (exact
    where the kernel keeps NumPy's sequential order)."""
    rng = np.random.default_rng([7, i])
    shape, axis, dt, op = _scan_case(rng, i)
    if np.issubdtype(dt, np.integer):
        x = rng.integers(-3, 4, shape).astype(dt) if op == "prod" else rng.integers(-100, 100, shape).astype(dt)
    else:
        x = (rng.standard_normal(shape) * (0.01 if op == "prod" else 1) + (1 if op == "prod" else 0)).astype(dt)
    g = gp.asarray(x)
    if op == "sum":
        got, ref = gp.cumsum(g, axis=axis), np.cumsum(x, axis=axis)
    elif op == "prod":
        got, ref = gp.cumprod(g, axis=axis), np.cumprod(x, axis=axis)
    else:
        flat = x.reshape(-1) if axis is None else x
        got = np.maximum.accumulate(gp.asarray(flat), axis=0 if axis is None else axis)
        ref = np.maximum.accumulate(flat, axis=0 if axis is None else axis)
    out = np.asarray(got)
    assert out.shape == ref.shape and out.dtype == ref.dtype, (out.shape, ref.shape, out.dtype, ref.dtype)
    label = sess.executor.last_steps[-1].cache["ks"].meta.get("label")
    if np.issubdtype(dt, np.integer) or op == "max" or label in (None, "scan-rows"):
        assert np.array_equal(out, ref), (shape, axis, dt, op, label)
        return
    w = np.float64 if dt == np.float32 else np.longdouble
    if op == "sum":
        wide = np.cumsum(x.astype(w), axis=axis)
        mag = np.cumsum(np.abs(x).astype(w), axis=axis)
    else:
        wide = np.cumprod(x.astype(w), axis=axis)
        mag = np.abs(wide)
    n = x.size if axis is None else x.shape[axis]
    tiles = -(-n // (8192 if dt == np.float32 else 4096))
    eps = np.finfo(dt).eps
    # long products reach the subnormal range, where the storage type (as
    # NumPy's own) keeps only an absolute precision of ~tiny
    atol = 4 * np.finfo(dt).tiny if op == "prod" else 0.0
    assert np.all(np.abs(out.astype(w) - wide) <= (tiles + 32) * eps * mag * (4 if op == "prod" else 1) + atol), \
        (shape, axis, dt, op, label)
