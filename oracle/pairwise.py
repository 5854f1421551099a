"""ORACLE — test infrastructure only.  Reduction/scan/library restatements.

The reference's executor oracles are sequential
folds, a three-phase blocked scan and naive triple-loop gemm/gemv.  Its
arithmetic dependency NumPy (pkg/pyproject.toml:11, numpy 2.3.5 here) reduces
floats *pairwise* along the contiguous axis; the B200 kernels reproduce that
order, so the oracle restates it here and tests/test_oracle_pins.py pins the
restatement against numpy.add.reduce for many lengths and layouts:

  pairwise_sum(a)   numpy/_core/src/umath/loops_utils.h.src (pairwise_sum):
                    n < 8: sequential fold starting at -0.0;
                    8 <= n <= 128: eight strided accumulators r[j] = a[j],
                    r[j] += a[i+j] per block of 8, combined
                    ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then a sequential tail;
                    n > 128: split at n2 = n/2 - (n/2) % 8, recurse, add.
  add.reduce result = identity 0.0 + pairwise_sum (contiguous inner axis) or
                    a sequential fold over outer axes.
"""

from __future__ import annotations

import numpy as np


def pairwise_sum(a: np.ndarray):
    """NumPy's pairwise summation of a 1-D float array, in its dtype."""
    t = a.dtype.type
    n = len(a)
    if n < 8:
        res = t(-0.0)
        for i in range(n):
            res = t(res + a[i])
        return res
    if n <= 128:
        r = [t(a[j]) for j in range(8)]
        i = 8
        while i < n - (n % 8):
            for j in range(8):
                r[j] = t(r[j] + a[i + j])
            i += 8
        res = t(t(t(r[0] + r[1]) + t(r[2] + r[3])) + t(t(r[4] + r[5]) + t(r[6] + r[7])))
        while i < n:
            res = t(res + a[i])
            i += 1
        return res
    n2 = n // 2
    n2 -= n2 % 8
    return t(pairwise_sum(a[:n2]) + pairwise_sum(a[n2:]))


def add_reduce_1d(a: np.ndarray):
    """np.add.reduce of a contiguous 1-D float array: 0.0 + pairwise_sum."""
    t = a.dtype.type
    return t(t(0.0) + pairwise_sum(a))


def sequential_fold(a, op, ident):
    """SPEC.md:376 per-thread fold from the identity (T = 1 oracle)."""
    acc = ident
    for v in np.asarray(a).ravel():
        acc = op(acc, v)
    return acc


def blocked_fold(a, op, ident, threads: int):
    """per-thread folds over a blocked partition, partials
    folded in thread-index order."""
    a = np.asarray(a).ravel()
    n = len(a)
    edges = [n * t // threads for t in range(threads + 1)]
    parts = [sequential_fold(a[edges[t]:edges[t + 1]], op, ident) for t in range(threads)]
    return sequential_fold(np.asarray(parts), op, ident)


def scan_three_phase(a, op, block: int):
    """SPEC.md:385 three-phase blocked inclusive scan: per-block sequential
    scan, exclusive scan of block totals, per-block offset add."""
    a = np.asarray(a)
    out = np.empty_like(a)
    n = len(a)
    totals = []
    for s in range(0, n, block):
        acc = None
        for i in range(s, min(n, s + block)):
            acc = a[i] if acc is None else op(acc, a[i])
            out[i] = acc
        totals.append(acc)
    carry = None
    for bi, s in enumerate(range(0, n, block)):
        if carry is not None:
            for i in range(s, min(n, s + block)):
                out[i] = op(carry, out[i])
        carry = totals[bi] if carry is None else op(carry, totals[bi])
    return out


def naive_gemm(A, B, trans_a=False, trans_b=False):
    """naive triple loop (float64 accumulation)."""
    A = np.asarray(A).T if trans_a else np.asarray(A)
    B = np.asarray(B).T if trans_b else np.asarray(B)
    m, k = A.shape
    k2, n = B.shape
    assert k == k2
    C = np.zeros((m, n), dtype=np.result_type(A, B))
    for i in range(m):
        for j in range(n):
            s = 0.0
            for p in range(k):
                s += float(A[i, p]) * float(B[p, j])
            C[i, j] = s
    return C


def naive_gemv(A, x, trans_a=False):
    return naive_gemm(A, np.asarray(x).reshape(-1, 1), trans_a=trans_a).reshape(-1)
