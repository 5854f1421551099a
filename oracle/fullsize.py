"""ORACLE — test infrastructure.  Parity of a whole named-shape run.

Checks the outputs of one bench step (or one full-size GPU test) against the
NumPy program of the same config evaluated on the same inputs — the reference's
eager baseline (the bench's VerificationFailed rule SPEC.md:497-502).
At 2^28 elements the eager program is evaluated on row blocks over host
threads (SURVEY.md §7 hard part 8: chunked oracle, exact for row-local results,
bounded for reductions).  Tolerances:

  listing1, jacobi,     bit-exact (only + and * in NumPy order, no contraction)
  transpose
  blackscholes f32/f64  |Δ| <= 1e-5 / 1e-12 · max(S, X)   (prices cancel)
  rownorm y             |Δ| <= 1e-5 · (1 + |y|); bit-exact mismatches reported
  rownorm total         |Δ| <= 4·log2(n)·eps32·Σ|y|; single shard of a power-
                        of-two row count: NumPy's own pairwise total, which the
                        kernel reproduces bit-exactly (reported as total_bitexact)
  mlp probs / labels    |Δp| <= 1e-5; a label may differ only where NumPy's
                        top-2 probability gap is <= 1e-5 (counted near-ties)
  kmeans                labels and counts exact; fp64 sums |Δ| <= 1e-12·Σ|p|
  cumsum f32            |Δ_i| <= (tiles + 32)·eps32·Σ_{j<=i}|t_j| against the
                        float64 prefix of the same f32 terms (the kernel's
                        association: a sequential chain over 8192-element tiles)
  cumsum-rows           bit-exact (a sequential fold per row, NumPy's order)

``comm_sum`` sums a float64 vector over ranks (gloo) for results that were
allreduced on the device (totals, k-means partials); identity on one rank.
"""

from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import programs

EPS32 = float(np.finfo(np.float32).eps)


def _threads(threads):
    return threads or max(1, min(len(os.sched_getaffinity(0)), 32))


def _blocks(n, nblocks):
    nblocks = max(1, min(nblocks, n))
    e = np.linspace(0, n, nblocks + 1).astype(np.int64)
    return [(int(e[i]), int(e[i + 1])) for i in range(nblocks)]


def _pow2_blocks(n, target):
    """Equal power-of-two row blocks (for NumPy's pairwise tree) when n is a
    power of two; else None."""
    if n <= 0 or n & (n - 1):
        return None
    b = 1
    while b * 2 <= max(1, n // target):
        b *= 2
    return [(i, i + b) for i in range(0, n, b)]


def _tree(parts):
    parts = list(parts)
    while len(parts) > 1:
        parts = [parts[i] + parts[i + 1] for i in range(0, len(parts), 2)]
    return parts[0]


def _result(ok, checked, mismatches, max_err, tol, **kw):
    d = {"ok": bool(ok), "checked": int(checked), "mismatches": int(mismatches),
         "max_err": float(max_err), "tol": tol}
    d.update(kw)
    return d


def check(name, inputs, outputs, threads=None, comm_sum=None, world=1, **kw):
    wl = programs.load()
    threads = _threads(threads)
    comm_sum = comm_sum or (lambda v: np.asarray(v, dtype=np.float64))
    fn = globals()["_check_" + name.replace("-", "_").replace("_y", "")]
    return fn(wl, name, [np.asarray(x) for x in inputs], [np.asarray(o) for o in outputs], threads, comm_sum, world, **kw)


def _map_blocks(threads, n, f):
    with ThreadPoolExecutor(max_workers=threads) as ex:
        return list(ex.map(f, _blocks(n, threads * 4)))


def _check_listing1(wl, name, inp, out, threads, comm_sum, world):
    W, a, b = inp
    got = out[0]

    def f(blk):
        lo, hi = blk
        e = wl.listing1(np, W[lo:hi], a[lo:hi], b[lo:hi])
        g = got[lo:hi]
        return int(np.count_nonzero(e.view(np.uint64) != g.view(np.uint64))), float(np.max(np.abs(e - g), initial=0))

    r = _map_blocks(threads, len(W), f)
    mm = sum(x[0] for x in r)
    return _result(mm == 0, len(W), mm, max(x[1] for x in r), "bit-exact")


def _check_blackscholes_f32(wl, name, inp, out, threads, comm_sum, world):
    S, X, T = inp
    call, put = out
    tol = 1e-5 if S.dtype == np.float32 else 1e-12

    def f(blk):
        lo, hi = blk
        c, p = wl.blackscholes(np, S[lo:hi], X[lo:hi], T[lo:hi])
        sc = np.maximum(S[lo:hi], X[lo:hi]).astype(np.float64)
        ec = np.abs(call[lo:hi].astype(np.float64) - c) / sc
        ep = np.abs(put[lo:hi].astype(np.float64) - p) / sc
        bad = np.count_nonzero(~(ec <= tol)) + np.count_nonzero(~(ep <= tol))
        return bad, float(max(ec.max(initial=0), ep.max(initial=0)))

    r = _map_blocks(threads, len(S), f)
    mm = sum(x[0] for x in r)
    return _result(mm == 0, 2 * len(S), mm, max(x[1] for x in r), f"|d| <= {tol:g}*max(S,X)",
                   err_unit="|d|/max(S,X)")


_check_blackscholes_f64 = _check_blackscholes_f32


def _check_rownorm(wl, name, inp, out, threads, comm_sum, world):
    (x,) = inp
    if len(out) == 2:
        y_got, total = out
    else:
        y_got, total = None, out[0]
    rows = x.shape[0]
    blocks = _pow2_blocks(rows, threads * 4) or _blocks(rows, threads * 4)

    def f(blk):
        lo, hi = blk
        y, _t = wl.rownorm(np, x[lo:hi])
        part = np.add.reduce(y.reshape(-1))
        y64 = y.astype(np.float64)
        res = [part, float(np.sum(y64)), float(np.sum(np.abs(y64))), 0, 0, 0.0]
        if y_got is not None:
            g = y_got[lo:hi]
            d = np.abs(g.astype(np.float64) - y64)
            res[3] = int(np.count_nonzero(~(d <= 1e-5 * (1 + np.abs(y64)))))
            res[4] = int(np.count_nonzero(g.view(np.uint32) != y.view(np.uint32)))
            res[5] = float(d.max(initial=0))
        return res

    with ThreadPoolExecutor(max_workers=threads) as ex:
        r = list(ex.map(f, blocks))
    s64, a64 = comm_sum(np.array([sum(v[1] for v in r), sum(v[2] for v in r)]))
    n_global = int(comm_sum(np.array([x.size], dtype=np.float64))[0])
    tol_t = 4 * math.log2(max(n_global, 2)) * EPS32 * a64
    total = float(np.asarray(total).reshape(-1)[0])
    err_t = abs(total - s64)
    extra = {"total": total, "total_ref_f64": s64, "total_tol": tol_t, "total_err": err_t}
    if world == 1 and _pow2_blocks(rows, 1) is not None:
        extra["total_bitexact"] = bool(np.float32(total) == _tree([v[0] for v in r]))
    bad = sum(v[3] for v in r)
    ok = err_t <= tol_t and bad == 0
    if y_got is not None:
        extra["y_bitexact_mismatches"] = sum(v[4] for v in r)
        extra["y_max_abs_err"] = max(v[5] for v in r)
    return _result(ok, x.size + 1, bad + (0 if err_t <= tol_t else 1), err_t / max(a64, 1e-300),
                   "y: |d| <= 1e-5*(1+|y|); total: |d| <= 4*log2(n)*eps32*sum|y|", err_unit="|d total|/sum|y|", **extra)


def _check_mlp(wl, name, inp, out, threads, comm_sum, world):
    X, W1, b1, W2, b2 = inp
    p_got, lab_got = out
    # one call: OpenBLAS threads the GEMMs itself
    p, lab = wl.mlp(np, X, W1, b1, W2, b2)
    d = np.abs(p_got.astype(np.float64) - p)
    bad_p = int(np.count_nonzero(~(d <= 1e-5)))
    diff = np.nonzero(lab_got != lab)[0]
    top2 = np.sort(p[diff], axis=1)[:, -2:] if len(diff) else np.zeros((0, 2))
    near = int(np.count_nonzero(top2[:, 1] - top2[:, 0] <= 1e-5)) if len(diff) else 0
    unexplained = len(diff) - near
    return _result(bad_p == 0 and unexplained == 0, p.size + lab.size, bad_p + unexplained, float(d.max(initial=0)),
                   "probs |d| <= 1e-5; labels exact except NumPy top-2 gap <= 1e-5",
                   label_mismatches=int(len(diff)), near_tie_flips=near)


def _check_kmeans(wl, name, inp, out, threads, comm_sum, world):
    P, C = inp
    lab_got, sums_got, counts_got = out[0], out[1:-1], out[-1]
    k, D = C.shape

    def f(blk):
        lo, hi = blk
        lab = wl.kmeans_assign(np, P[lo:hi], C)
        mm = int(np.count_nonzero(lab != lab_got[lo:hi]))
        cnt = np.bincount(lab, minlength=k)
        s = np.stack([np.bincount(lab, weights=P[lo:hi, d], minlength=k) for d in range(D)])
        a = np.stack([np.bincount(lab, weights=np.abs(P[lo:hi, d]).astype(np.float64), minlength=k) for d in range(D)])
        return mm, cnt, s, a

    r = _map_blocks(threads, len(P), f)
    mm = sum(v[0] for v in r)
    cnt = comm_sum(_tree([v[1].astype(np.float64) for v in r]))
    s = comm_sum(_tree([v[2] for v in r]).reshape(-1)).reshape(D, k)
    a = comm_sum(_tree([v[3] for v in r]).reshape(-1)).reshape(D, k)
    cnt_bad = int(np.count_nonzero(np.asarray(counts_got, dtype=np.float64) != cnt))
    sg = np.stack([np.asarray(x, dtype=np.float64) for x in sums_got])
    ds = np.abs(sg - s)
    sum_bad = int(np.count_nonzero(~(ds <= 1e-12 * a)))
    err = float(np.max(ds / np.maximum(a, 1e-300)))
    return _result(mm == 0 and cnt_bad == 0 and sum_bad == 0, len(P) + k * (D + 1), mm + cnt_bad + sum_bad, err,
                   "labels, counts exact; sums |d| <= 1e-12*sum|p|", label_mismatches=mm, count_mismatches=cnt_bad,
                   sum_err_rel=err)


def _check_cumsum(wl, name, inp, out, threads, comm_sum, world, tile=8192):
    (x,) = inp
    got = out[0]
    n = len(x)
    blocks = _blocks(n, threads * 4)

    def f(blk):
        lo, hi = blk
        t = (x[lo:hi] * np.float32(0.5) + np.float32(1.0)).astype(np.float64)
        return np.cumsum(t), np.cumsum(np.abs(t))

    with ThreadPoolExecutor(max_workers=threads) as ex:
        r = list(ex.map(f, blocks))
    gamma = (n / tile + 32) * EPS32
    off, aoff, worst, bad = 0.0, 0.0, 0.0, 0
    for (lo, hi), (c, a) in zip(blocks, r):
        ref = c + off
        ab = a + aoff
        d = np.abs(got[lo:hi].astype(np.float64) - ref)
        q = d / np.maximum(ab, 1e-300)
        worst = max(worst, float(q.max(initial=0)))
        bad += int(np.count_nonzero(~(d <= gamma * ab)))
        off, aoff = ref[-1], ab[-1]
    return _result(bad == 0, n, bad, worst, f"|d_i| <= {gamma:.3g}*prefix sum|t|", err_unit="|d_i|/prefix sum|t|")


def _check_cumsum_rows(wl, name, inp, out, threads, comm_sum, world):
    """Per-row sequential fold: NumPy's own association, bit-exact."""
    (x,) = inp
    got = out[0]

    def f(blk):
        lo, hi = blk
        e = wl.scan_rows(np, x[lo:hi])
        g = got[lo:hi]
        return int(np.count_nonzero(e.view(np.uint32) != g.view(np.uint32))), float(np.max(np.abs(e - g), initial=0))

    r = _map_blocks(threads, len(x), f)
    mm = sum(v[0] for v in r)
    return _result(mm == 0, x.size, mm, max(v[1] for v in r), "bit-exact")


def _check_jacobi(wl, name, inp, out, threads, comm_sum, world):
    (a,) = inp
    got = out[0]
    e = wl.jacobi(np, a)
    mm = int(np.count_nonzero(e.view(np.uint32) != got.view(np.uint32)))
    return _result(mm == 0, e.size, mm, float(np.max(np.abs(e - got))), "bit-exact")


def _check_transpose(wl, name, inp, out, threads, comm_sum, world):
    x, y = inp
    got = out[0]

    def f(blk):
        lo, hi = blk
        e = wl.transpose_add(np, x[:, lo:hi], y[lo:hi])
        return int(np.count_nonzero(e.view(np.uint32) != got[lo:hi].view(np.uint32)))

    mm = sum(_map_blocks(threads, y.shape[0], f))
    return _result(mm == 0, got.size, mm, 0.0 if mm == 0 else float("nan"), "bit-exact")
