"""The BASELINE.json configs written as NumPy programs over a module ``xp``.

Each function is the user program: run it with ``xp=numpy`` (+ scipy erf) and
it is the reference's eager NumPy baseline; run it with
``xp=grumpy`` and every region materializes as one fused B200 kernel.  Input
generators use ``numpy.random.default_rng(seed)`` (SURVEY.md
§8(d)).

C1 Listing 1 chain     (reconstructed)
C2 Black-Scholes       (erf normal CDF)
C3 row-normalise + sum (BASELINE.json configs[2])
C4 MNIST-style MLP     (np.dot -> library)
C5 k-means assignment
Jacobi sweep           (SPEC.md:248 — §8(f) rank 2)
"""

from __future__ import annotations

import numpy as np


def _erf(xp):
    if xp is np:
        from scipy.special import erf
        return erf
    return xp.erf


# ---- C1 -----------------------------------------------------------------------
def listing1_inputs(n=1 << 24, seed=42, dtype=np.float64):
    rng = np.random.default_rng(seed)
    W = rng.random(n, dtype=np.float64).astype(dtype)
    a = rng.random(n, dtype=np.float64).astype(dtype)
    b = rng.random(n, dtype=np.float64).astype(dtype)
    return W, a, b


def listing1(xp, W, a, b):
    """4 multiplies + 2 adds (SURVEY.md §8(d) C1 reconstruction)."""
    x = a * W
    y = b * W
    z = x * y
    return z * W + a + b


# ---- C2 -----------------------------------------------------------------------
BS_R = 0.02
BS_V = 0.30


def blackscholes_inputs(n=1 << 28, seed=42, dtype=np.float32):
    rng = np.random.default_rng(seed)
    S = rng.uniform(5.0, 30.0, n).astype(dtype)
    X = rng.uniform(1.0, 100.0, n).astype(dtype)
    T = rng.uniform(0.25, 10.0, n).astype(dtype)
    return S, X, T


def blackscholes(xp, S, X, T, r=BS_R, v=BS_V):
    """European call/put with the erf-based CND."""
    erf = _erf(xp)
    sqT = xp.sqrt(T)
    d1 = (xp.log(S / X) + (r + 0.5 * v * v) * T) / (v * sqT)
    d2 = d1 - v * sqT
    cnd1 = 0.5 * (1.0 + erf(d1 * 0.7071067811865476))
    cnd2 = 0.5 * (1.0 + erf(d2 * 0.7071067811865476))
    e = xp.exp(-r * T)
    call = S * cnd1 - X * e * cnd2
    put = X * e * (1.0 - cnd2) - S * (1.0 - cnd1)
    return call, put


# ---- C3 -----------------------------------------------------------------------
def rownorm_inputs(rows=65536, cols=4096, seed=42, dtype=np.float32):
    rng = np.random.default_rng(seed)
    x = (rng.standard_normal((rows, cols), dtype=np.float32) * 2 + 5).astype(dtype)
    return (x,)


def rownorm(xp, x):
    y = (x - x.mean(1)[:, None]) / x.std(1)[:, None]
    return y, y.sum()


# ---- C4 -----------------------------------------------------------------------
def mlp_inputs(batch=65536, hidden=1024, seed=42):
    rng = np.random.default_rng(seed)
    X = rng.random((batch, 784), dtype=np.float32)
    W1 = (rng.standard_normal((784, hidden), dtype=np.float32) / np.float32(np.sqrt(784))).astype(np.float32)
    b1 = rng.uniform(-0.1, 0.1, hidden).astype(np.float32)
    W2 = (rng.standard_normal((hidden, 10), dtype=np.float32) / np.float32(np.sqrt(hidden))).astype(np.float32)
    b2 = rng.uniform(-0.1, 0.1, 10).astype(np.float32)
    return X, W1, b1, W2, b2


def mlp(xp, X, W1, b1, W2, b2):
    h = xp.maximum(X @ W1 + b1, 0)
    z = h @ W2 + b2
    p = xp.exp(z - z.max(1)[:, None])
    p = p / p.sum(1)[:, None]
    return p, p.argmax(1)


# ---- C5 -----------------------------------------------------------------------
def kmeans_inputs(n=1 << 26, k=64, d=4, seed=42):
    rng = np.random.default_rng(seed)
    centres = rng.uniform(-10, 10, (k, d)).astype(np.float32)
    lab = rng.integers(0, k, n)
    P = (centres[lab] + rng.standard_normal((n, d), dtype=np.float32)).astype(np.float32)
    C0 = P[rng.choice(n, k, replace=False)].copy()
    return P, C0


def kmeans_assign(xp, P, C):
    d = ((P[:, None, :] - C[None]) ** 2).sum(-1)
    return d.argmin(1)


def kmeans_partials(xp, P, C):
    """Assignment + per-cluster partial sums (fp64) and counts: the quantities
    each shard allreduces before the centroid update."""
    k, D = C.shape
    lab = kmeans_assign(xp, P, C)
    sums = [xp.bincount(lab, weights=P[:, d], minlength=k) for d in range(D)]
    counts = xp.bincount(lab, minlength=k)
    return lab, sums, counts


def kmeans_centroids(sums, counts, C_old):
    """Host-side centroid update from (allreduced) partials; empty clusters keep
    their previous centre."""
    S = np.stack([np.asarray(s) for s in sums], axis=1)
    n = np.asarray(counts)
    out = np.array(C_old, dtype=np.float64, copy=True)
    nz = n > 0
    out[nz] = S[nz] / n[nz, None]
    return out.astype(np.float32)


# ---- Jacobi -------------------------------------------
def jacobi_inputs(n=16384, seed=42, dtype=np.float32):
    rng = np.random.default_rng(seed)
    return (rng.random((n, n), dtype=np.float32).astype(dtype),)


def jacobi(xp, a):
    """One 5-point Jacobi sweep with fixed boundary: in
    grumpy the slice-assign lowers to a select over the grid (SPEC.md:304,
    336), one fused kernel per sweep."""
    b = a.copy()
    b[1:-1, 1:-1] = 0.2 * (a[1:-1, 1:-1] + a[1:-1, :-2] + a[1:-1, 2:] + a[:-2, 1:-1] + a[2:, 1:-1])
    return b


# ---- transposed operand (north_star: shared-memory staging of strided operands)
def transpose_add(xp, x, y):
    """x.T + y: the transposed leaf is staged through shared memory tiles
    (codegen_tile.py), the output and y move row-wise."""
    return x.T + y


# ---- map-scan ------------------------------------------
def scan_inputs(n=1 << 28, seed=42, dtype=np.float32):
    rng = np.random.default_rng(seed)
    return (rng.standard_normal(n, dtype=np.float32).astype(dtype),)


def scan(xp, x):
    """Map-scan: a fused map prologue feeding one inclusive scan."""
    return xp.cumsum(x * 0.5 + 1.0)


def scan_rows(xp, x):
    """Map-scan along the contiguous axis of a matrix (one scan
    axis of the operand): every row its own sequential fold."""
    return xp.cumsum(x * 0.5 + 1.0, axis=1)


# ---- named-shape inputs generated in fixed row blocks ---------------------------
# The bench shards the named shape along its leading axis.
# Generating the global array from fixed row blocks, block b from
# default_rng([seed, b]), makes rank r's shard identical to rows [lo, hi) of the
# single-GPU input for any GPU count, and lets the blocks be generated on
# several host threads.  Replicated operands (weights, centroids) come from
# default_rng(seed).

def _bs_rows(dtype):
    def gen(rng, rows):
        S = rng.uniform(5.0, 30.0, rows).astype(dtype)
        X = rng.uniform(1.0, 100.0, rows).astype(dtype)
        T = rng.uniform(0.25, 10.0, rows).astype(dtype)
        return [S, X, T]
    return gen


def _km_centres(seed, k=64, d=4):
    rng = np.random.default_rng(seed)
    centres = rng.uniform(-10, 10, (k, d)).astype(np.float32)
    C0 = (centres + rng.standard_normal((k, d), dtype=np.float32)).astype(np.float32)
    return centres, C0


def _km_rows(seed):
    centres, _ = _km_centres(seed)

    def gen(rng, rows):
        lab = rng.integers(0, centres.shape[0], rows)
        return [(centres[lab] + rng.standard_normal((rows, centres.shape[1]), dtype=np.float32)).astype(np.float32)]
    return gen


def _mlp_weights(seed, hidden=1024):
    rng = np.random.default_rng(seed)
    W1 = (rng.standard_normal((784, hidden), dtype=np.float32) / np.float32(np.sqrt(784))).astype(np.float32)
    b1 = rng.uniform(-0.1, 0.1, hidden).astype(np.float32)
    W2 = (rng.standard_normal((hidden, 10), dtype=np.float32) / np.float32(np.sqrt(hidden))).astype(np.float32)
    b2 = rng.uniform(-0.1, 0.1, 10).astype(np.float32)
    return [W1, b1, W2, b2]


# name -> (global leading extent, rows per block, row generator factory,
#          replicated-operand factory, input order: "S" sharded / "R" replicated)
NAMED = {
    "listing1": (1 << 24, 1 << 20, lambda s: (lambda rng, r: [rng.random(r), rng.random(r), rng.random(r)]),
                 lambda s: [], "SSS"),
    "blackscholes-f32": (1 << 28, 1 << 22, lambda s: _bs_rows(np.float32), lambda s: [], "SSS"),
    "blackscholes-f64": (1 << 28, 1 << 22, lambda s: _bs_rows(np.float64), lambda s: [], "SSS"),
    "rownorm": (65536, 1024,
                lambda s: (lambda rng, r: [(rng.standard_normal((r, 4096), dtype=np.float32) * 2 + 5).astype(np.float32)]),
                lambda s: [], "S"),
    "mlp": (65536, 1024, lambda s: (lambda rng, r: [rng.random((r, 784), dtype=np.float32)]),
            lambda s: _mlp_weights(s), "SRRRR"),
    "kmeans": (1 << 26, 1 << 20, lambda s: _km_rows(s), lambda s: [_km_centres(s)[1]], "SR"),
    "cumsum": (1 << 28, 1 << 22, lambda s: (lambda rng, r: [rng.standard_normal(r, dtype=np.float32)]),
               lambda s: [], "S"),
    "cumsum-rows": (65536, 1024,
                    lambda s: (lambda rng, r: [rng.standard_normal((r, 4096), dtype=np.float32)]),
                    lambda s: [], "S"),
    "jacobi": (16384, 256, lambda s: (lambda rng, r: [rng.random((r, 16384), dtype=np.float32)]),
               lambda s: [], "S"),
}
NAMED["rownorm-y"] = NAMED["rownorm"]
NAMED["transpose"] = (16384, 256, lambda s: (lambda rng, r: [rng.random((r, 16384), dtype=np.float32),
                                                             rng.random((r, 16384), dtype=np.float32)]),
                      lambda s: [], "SS")


def named_inputs(name, lo=0, hi=None, seed=42, threads=None):
    """Rows [lo, hi) of the named-shape input of workload ``name`` (block
    generated, see above), plus its replicated operands, in program order."""
    from concurrent.futures import ThreadPoolExecutor
    import os as _os

    n, blk, rows_f, rep_f, order = NAMED[name]
    hi = n if hi is None else hi
    gen = rows_f(seed)
    b0, b1 = lo // blk, (hi + blk - 1) // blk
    threads = threads or max(1, min(len(_os.sched_getaffinity(0)), 32))

    def block(b):
        parts = gen(np.random.default_rng([seed, b]), blk)
        s, e = max(lo, b * blk) - b * blk, min(hi, (b + 1) * blk) - b * blk
        return [p[s:e] for p in parts]

    with ThreadPoolExecutor(max_workers=threads) as ex:
        blocks = list(ex.map(block, range(b0, b1)))
    sharded = [np.concatenate([bl[i] for bl in blocks]) if len(blocks) > 1 else np.ascontiguousarray(blocks[0][i])
               for i in range(len(blocks[0]))]
    rep = rep_f(seed)
    out, si, ri = [], 0, 0
    for c in order:
        if c == "S":
            out.append(sharded[si])
            si += 1
        else:
            out.append(rep[ri])
            ri += 1
    return out
