"""One small region of every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck): map (K1, slices, slice-assign), rows
(K2-K5, keyed sums, skinny product with TMA + mbarriers), cooperative rows
(named barriers), map-scan (decoupled look-back), streamed chunks.  Each
result is checked against NumPy so a sanitizer run is also a parity run.

  compute-sanitizer --tool memcheck python tools/sanitize_check.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1901_03771_b200 as gp  # noqa: E402
from paper_1901_03771_b200 import workloads as wl  # noqa: E402

only = sys.argv[1:] or None


def case(name):
    def deco(f):
        if only is None or name in only:
            f()
            print(f"{name}: ok", flush=True)
        return f
    return deco


@case("map")
def _():
    W, a, b = wl.listing1_inputs(n=(1 << 14) + 3)
    assert np.array_equal(np.asarray(wl.listing1(gp, gp.asarray(W), gp.asarray(a), gp.asarray(b))), wl.listing1(np, W, a, b))
    S, X, T = wl.blackscholes_inputs(n=(1 << 13) + 5)
    c, p = wl.blackscholes(gp, gp.asarray(S), gp.asarray(X), gp.asarray(T))
    gp.force(c, p)
    rc, rp = wl.blackscholes(np, S, X, T)
    assert np.all(np.abs(np.asarray(c) - rc) <= 1e-5 * np.maximum(S, X))
    x = np.random.default_rng(1).standard_normal((67, 45)).astype(np.float32)
    assert np.array_equal(np.asarray(gp.asarray(x).T * 2 + 1), x.T * 2 + 1)


@case("slices")
def _():
    (a,) = wl.jacobi_inputs(n=130)
    assert np.array_equal(np.asarray(wl.jacobi(gp, gp.asarray(a))), wl.jacobi(np, a))


@case("rows")
def _():
    P, C = wl.kmeans_inputs(n=8192 + 17, k=64, d=4)
    lab, sums, counts = wl.kmeans_partials(gp, gp.asarray(P), gp.asarray(C))
    gp.force(lab, *sums, counts)
    el, es, ec = wl.kmeans_partials(np, P, C)
    assert np.array_equal(np.asarray(lab), el) and np.array_equal(np.asarray(counts), ec)
    z = np.random.default_rng(2).standard_normal((1000, 10)).astype(np.float32)
    gz = gp.asarray(z)
    pz = gp.exp(gz - gz.max(1)[:, None])
    pz = pz / pz.sum(1)[:, None]
    assert np.array_equal(np.asarray(pz.argmax(1)), (np.exp(z - z.max(1)[:, None])).argmax(1))
    t = np.random.default_rng(3).standard_normal(100003)
    assert np.asarray(gp.asarray(t).sum()) == t.sum()


@case("skinny")
def _():
    X, W1, b1, W2, b2 = wl.mlp_inputs(batch=4096 + 96, hidden=256)
    p, lab = wl.mlp(gp, *[gp.asarray(v) for v in (X, W1, b1, W2, b2)])
    gp.force(p, lab)
    ep, elab = wl.mlp(np, X, W1, b1, W2, b2)
    assert np.max(np.abs(np.asarray(p) - ep)) <= 1e-5 and np.mean(np.asarray(lab) == elab) > 0.999


@case("coop")
def _():
    (x,) = wl.rownorm_inputs(rows=256, cols=4096)
    y, t = wl.rownorm(gp, gp.asarray(x))
    gp.force(y, t)
    ey, et = wl.rownorm(np, x)
    assert np.array_equal(np.asarray(y), ey) and np.asarray(t) == et


@case("scan")
def _():
    xi = np.random.default_rng(4).integers(-100, 100, (1 << 20) + 7)
    assert np.array_equal(np.asarray(gp.asarray(xi).cumsum()), xi.cumsum())
    xf = np.random.default_rng(5).standard_normal((33, 70))
    assert np.array_equal(np.asarray(gp.cumsum(gp.asarray(xf) * 2, axis=1)), np.cumsum(xf * 2, axis=1))
    # TMA ring + round-tree look-back: 1-D with a tail, segmented lines,
    # flat n-D; register-staged with segments and with a broadcast operand
    rng = np.random.default_rng(6)
    for shape, axis in [((1 << 20) + 7, None), ((16, 65536), 1), ((1024, 1024), None), ((16, 70001), 1)]:
        v = rng.integers(-50, 50, shape)
        assert np.array_equal(np.asarray(gp.cumsum(gp.asarray(v) * 3, axis=axis)), np.cumsum(v * 3, axis=axis))
    m = rng.integers(-50, 50, (1024, 1024))
    r = rng.integers(-5, 5, 1024)
    assert np.array_equal(np.asarray(gp.cumsum(gp.asarray(m) + gp.asarray(r))), np.cumsum(m + r))


@case("stream")
def _():
    from paper_1901_03771_b200 import streaming
    streaming.MIN_BYTES = 1
    streaming.CHUNK_BYTES = 1 << 18
    S, X, T = wl.blackscholes_inputs(n=1 << 15)
    c, p = wl.blackscholes(gp, gp.asarray(S), gp.asarray(X), gp.asarray(T))
    gc, gpt = gp.materialize(c, p)
    rc, rp = wl.blackscholes(np, S, X, T)
    assert np.all(np.abs(gc - rc) <= 1e-5 * np.maximum(S, X))

print("sanitize_check done", flush=True)
