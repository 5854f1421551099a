"""The certified nearest-centre search (gr_nearest.cuh) emulated in NumPy on
CPU: whenever the device certificate accepts a row, its label must equal
np.argmin over NumPy's own float32 distances.  Adversarial inputs: exact and
near ties (points on bisectors), duplicated centres, large offsets, tiny
magnitudes, random scales."""
import numpy as np
import pytest

from paper_1901_03771_b200 import codegen_rows, workloads as wl

F = np.float32


def _fma32(a, b, c):
    # float32 fma via float64: a*b is exact in f64; the f64 add can round once
    # before the f32 rounding (double rounding) — a test-only approximation
    return (a.astype(np.float64) * b.astype(np.float64) + c.astype(np.float64)).astype(F)


def _pack(C):
    K, D = C.shape
    o = (C.astype(np.float64).sum(0) / K).astype(F)
    cp = (C - o).astype(F)
    cc64 = (cp.astype(np.float64) ** 2).sum(1)
    bad = not np.all(np.isfinite(C))
    CC = np.nan if bad else np.nextafter(F(cc64.max() * (1 + 1e-6)), F(np.inf))
    return o, cp, cc64.astype(F), F(CC)


def emulate(P, C):
    """(labels, certified) exactly as gr::nearest_centre computes them."""
    K, D = C.shape
    bits = max(1, int(np.ceil(np.log2(K))))
    mask = np.uint32((1 << bits) - 1)
    o, cp, cc, CC = _pack(C)
    with np.errstate(all="ignore"):
        pk = (P - o).astype(F)
        q = (F(-2) * pk).astype(F)
        pp = np.zeros(len(P), F)
        for k in range(D):
            pp = _fma32(pk[:, k], pk[:, k], pp)
        acc = (np.broadcast_to(cc, (len(P), K)).astype(F) + pp[:, None]).astype(F)
        for k in range(D):
            acc = _fma32(q[:, k:k + 1], cp[None, :, k], acc)
        keys = ((acc.view(np.uint32) & ~mask) | np.arange(K, dtype=np.uint32)).view(F)
        srt = np.sort(keys, axis=1)     # finite keys only matter when certified
        m1, m2 = srt[:, 0], srt[:, 1]
        lab = (m1.view(np.uint32) & mask).astype(np.int64)
        E = F(1.01 * 2.0 ** (bits - 23))
        R = (pp + F(2) * CC).astype(F)
        dc = (F(24 * 2.0 ** -24) * R).astype(F)
        a1, a2 = np.abs(m1), np.abs(m2)
        NP = F(2.1 * (D + 2) * 2.0 ** -24)
        thr = (F(2.1) * dc + E * (a1 + a2) + NP * np.maximum((m1 + E * a1 + dc).astype(F), F(0))
               + F(1e-35)).astype(F)
        ok = (R < F(1e37)) & ((m2 - m1).astype(F) > thr)
    return lab, ok


def _check(P, C, min_cert=0.0):
    lab, ok = emulate(P, C)
    ref = wl.kmeans_assign(np, P, C)
    bad = np.nonzero(ok & (lab != ref))[0]
    assert bad.size == 0, (bad[:10], lab[bad[:10]], ref[bad[:10]])
    assert ok.mean() >= min_cert, ok.mean()
    return ok.mean()


def test_pattern_matched():
    import paper_1901_03771_b200 as gp
    P, C = wl.kmeans_inputs(n=4096)
    d = ((gp.asarray(P)[:, None, :] - gp.asarray(C)[None]) ** 2).sum(-1)
    assert codegen_rows.match_nearest(d.node, (1,)) is not None
    d2 = ((gp.asarray(P)[:, None, :] - gp.asarray(C)[None]) * 2).sum(-1)
    assert codegen_rows.match_nearest(d2.node, (1,)) is None


def test_certified_labels_named_data():
    P, C = wl.kmeans_inputs(n=1 << 16, k=64, d=4)
    # nearly every row certifies on the C5 data
    assert _check(P, C, min_cert=0.999) > 0.999


@pytest.mark.parametrize("seed", range(8))
@pytest.mark.parametrize("K,D", [(2, 1), (8, 3), (64, 4), (256, 8), (16, 2)])
def test_certified_labels_adversarial(seed, K, D):
    rng = np.random.default_rng([seed, K, D])
    scale = [1e-20, 1e-3, 1.0, 50.0, 1e4][seed % 5]
    C = (rng.standard_normal((K, D)) * scale).astype(F)
    if K >= 4:
        C[K // 2] = C[1]                                  # duplicated centre
    n = 20000
    P = (C[rng.integers(0, K, n)] + rng.standard_normal((n, D)).astype(F) * F(scale * 0.5)).astype(F)
    # points on bisectors of random centre pairs (exact ties in the reals)
    i, j = rng.integers(0, K, 2000), rng.integers(0, K, 2000)
    P[:2000] = ((C[i].astype(np.float64) + C[j]) / 2).astype(F)
    # and within a few ulps of them
    P[2000:4000] = (P[:2000] * (1 + rng.integers(-4, 5, (2000, 1)) * F(2 ** -23))).astype(F)
    P[4000:4100] = C[rng.integers(0, K, 100)]             # zero distance
    P[4100] += F(scale) * F(1e3)                          # far away
    _check(P, C)


def test_nonfinite_never_certified():
    P, C = wl.kmeans_inputs(n=4096, k=64, d=4)
    P[0, 1] = np.nan
    P[1] = np.inf
    P[2, 0] = 3e19                                        # products near overflow
    lab, ok = emulate(P, C)
    assert not ok[:3].any()
    C2 = C.copy()
    C2[5, 2] = np.nan
    _lab, ok2 = emulate(P, C2)
    assert not ok2.any()
