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

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
NPROG = int(os.environ.get("GRUMPY_RANDOM_PROGRAMS", "120"))


def _rand_shape(rng, rank):
    return tuple(int(rng.integers(1, 17)) for _ in range(rank))


def make_program(seed):
    rng = np.random.default_rng(seed)
    rank = int(rng.integers(1, 4))
    shape = _rand_shape(rng, rank)
    dt = rng.choice([np.float32, np.float64, np.int32, np.int64])
    pool = []
    for _ in range(int(rng.integers(1, 4))):
        s = list(shape)
        if rng.random() < 0.3:          # broadcastable operand
            s[int(rng.integers(0, rank))] = 1
        a = rng.standard_normal(s) * 4 if np.dtype(dt).kind == "f" else rng.integers(-20, 20, s)
        pool.append(gp.asarray(np.asarray(a, dtype=dt)))
    depth = int(rng.integers(1, 13))
    cur = pool[0]
    transcendental = False   # exp is ulp-accurate, not bit-exact: no branching on it afterwards
    viewed = False
    for _ in range(depth):
        k = rng.integers(0, 14)
        other = pool[int(rng.integers(0, len(pool)))]
        try:
            if k == 0:
                cur = cur + other
            elif k == 1:
                cur = cur * other - 1
            elif k == 2:
                cur = gp.maximum(cur, other)
            elif k == 3 and cur.dtype.kind == "f":
                cur = gp.exp(cur * 0.1) + gp.sqrt(gp.abs(cur))
                transcendental = True
            elif k == 4 and not transcendental:
                cur = gp.where(cur > other, cur, other * 2)
            elif k == 5 and cur.ndim >= 2:
                cur = cur.transpose()
                viewed = True
            elif k == 6 and cur.ndim >= 1 and cur.shape[-1] > 2:
                cur = cur[..., 1:] if rng.random() < 0.5 else cur[..., ::2]
                viewed = True
            elif k == 7 and cur.ndim >= 2:
                cur = cur.reshape(-1, cur.shape[-1])
            elif k == 8 and cur.ndim >= 2:
                ax = int(rng.integers(0, cur.ndim))
                cur = cur.sum(axis=ax, keepdims=bool(rng.random() < 0.5))
                # NumPy reduces a strided view in memory order, the kernel in C
                # order: same value up to reassociation, so not bit-exact
                transcendental = transcendental or (viewed and cur.dtype.kind == "f")
            elif k == 9 and cur.ndim >= 1:
                ax = int(rng.integers(0, cur.ndim))
                cur = cur.max(axis=ax) if rng.random() < 0.5 else cur.min(axis=ax)
            elif k == 10 and cur.ndim >= 1:
                cur = cur.astype(np.float64) / 3
            elif k == 11 and cur.ndim == 2 and cur.dtype.kind == "f":
                # np.dot boundary: GEMM, optionally + bias row and ReLU (the
                # cuBLASLt epilogue pattern); reassociated, so inexact after
                W = gp.asarray(rng.standard_normal((cur.shape[1], int(rng.integers(1, 17)))).astype(cur.dtype))
                cur = cur @ W
                if rng.random() < 0.6:
                    cur = cur + gp.asarray(rng.standard_normal(cur.shape[1]).astype(cur.dtype))
                    if rng.random() < 0.5:
                        cur = gp.maximum(cur, 0)
                transcendental = True
            elif k == 12 and cur.ndim >= 1:
                ax = int(rng.integers(0, cur.ndim))
                cur = gp.cumsum(cur, axis=ax)
                transcendental = transcendental or cur.dtype.kind == "f"
            elif k == 13 and cur.ndim >= 1 and cur.shape[-1] >= 2:
                nxt = cur.copy()
                nxt[..., ::2] = cur[..., ::2] * 2 + 1
                cur = nxt
        except gp.LazyFuseError:
            continue
    finals = [cur]
    if cur.ndim >= 1 and rng.random() < 0.5 and not transcendental:
        finals.append(cur.argmax(axis=int(rng.integers(0, cur.ndim))))
    if rng.random() < 0.5:
        finals.append(cur.sum())
    return finals, transcendental


def _close(got, exp, dtype, transcendental=False):
    if dtype.kind in "biu":
        return np.array_equal(got, exp)
    # f32 transcendental ancestry carries f32 ulp error into f64 results
    rtol = 1e-5 if (dtype == np.float32 or transcendental) else 1e-12
    fin = np.isfinite(exp)
    if not np.array_equal(np.isfinite(got), fin) or not np.array_equal(got[~fin], exp[~fin]) and \
            not np.array_equal(np.isnan(got[~fin]), np.isnan(exp[~fin])):
        return False
    scale = np.max(np.abs(exp[fin])) if fin.any() else 0.0
    return np.allclose(got[fin], exp[fin], rtol=rtol, atol=rtol * max(1.0, scale) * 64)


@pytest.mark.parametrize("seed", range(NPROG))
def test_random_program(sess, seed):
    outs, transcendental = make_program(seed)
    expect = [eager.evaluate(o.node) for o in outs]
    gp.force(*outs)
    for o, e in zip(outs, expect):
        got = np.asarray(o)
        assert got.shape == e.shape and got.dtype == e.dtype
        assert _close(got, e, e.dtype, transcendental), (seed, o.node, got, e)
        if not transcendental and e.dtype.kind == "f" and o.node.kind.value == "MapElementwise":
            # +,-,*,/,sqrt,max and casts are IEEE-exact: bit-identical to NumPy
            assert np.array_equal(got, e, equal_nan=True), (seed, "not bit-exact", o.node)


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
