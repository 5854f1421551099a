"""Randomised lazy programs (ranks <= 3, extents <= 16,
depth <= 12, every op kind) written once over an array namespace, so the same
seed records a grumpy DAG (``GP``), runs eagerly in NumPy (``Numpy``), in
extended precision (``Numpy(wide=True)``: float64 for f32 programs, x87 long
double for f64 ones) and as a magnitude run (``Numpy(absolute=True)``: inputs
|x|, every subtraction an addition — per element an upper bound of the
sum of |terms| the rounding errors scale with, SURVEY.md §7 hard part 2).

Test infrastructure only.
"""

from __future__ import annotations

import numpy as np


class GP:
    """grumpy (the product) as the array namespace."""

    def __init__(self):
        import paper_1901_03771_b200 as gp
        self.gp = gp
        self.errors = (gp.LazyFuseError,)

    def asarray(self, a):
        return self.gp.asarray(a)

    def sub(self, a, b):
        return a - b

    def maximum(self, a, b):
        return self.gp.maximum(a, b)

    def exp(self, a):
        return self.gp.exp(a)

    def sqrt_abs(self, a):
        return self.gp.sqrt(self.gp.abs(a))

    def where_gt(self, a, b, c):
        return self.gp.where(a > b, a, c)

    def cumsum(self, a, axis):
        return self.gp.cumsum(a, axis=axis)

    def relu(self, a):
        return self.gp.maximum(a, 0)

    def copy(self, a):
        return a.copy()

    def minmax(self, a, axis, use_max):
        return a.max(axis=axis) if use_max else a.min(axis=axis)


class Numpy(GP):
    """NumPy eager evaluation of the same program; ``wide`` evaluates floats
    one precision up, ``absolute`` gives the magnitude run."""

    def __init__(self, wide=False, absolute=False):
        self.errors = (ValueError, TypeError)
        self.wide = wide
        self.absolute = absolute

    def asarray(self, a):
        a = np.asarray(a)
        if self.absolute:
            a = np.abs(a)
        if (self.wide or self.absolute) and a.dtype.kind == "f":
            a = a.astype(np.float64 if a.dtype == np.float32 else np.longdouble)
        return a

    def sub(self, a, b):
        return a + b if self.absolute else a - b

    def maximum(self, a, b):
        return np.maximum(a, b)

    def exp(self, a):
        return np.exp(np.abs(a) if self.absolute else a)

    def sqrt_abs(self, a):
        return np.sqrt(np.abs(a))

    def where_gt(self, a, b, c):
        if self.absolute:
            return np.maximum(np.maximum(a, c), np.zeros_like(a))
        return np.where(a > b, a, c)

    def cumsum(self, a, axis):
        return np.cumsum(a, axis=axis)

    def relu(self, a):
        return np.maximum(a, 0)

    def minmax(self, a, axis, use_max):
        if self.absolute:
            return a.max(axis=axis)
        return a.max(axis=axis) if use_max else a.min(axis=axis)


def _rand_shape(rng, rank):
    return tuple(int(rng.integers(1, 17)) for _ in range(rank))


def _header(rng):
    rank = int(rng.integers(1, 4))
    shape = _rand_shape(rng, rank)
    dt = rng.choice([np.float32, np.float64, np.int32, np.int64])
    return rank, shape, dt


def input_dtype(seed):
    return np.dtype(_header(np.random.default_rng(seed))[2])


def within(got, wide, native, mag, eps, depth):
    """Per element: the device's error against an extended-precision run of
    the same program is at most 4x NumPy's own error plus
    64*(depth+2)*eps times the element's magnitude run (sum of |terms|);
    non-finite values must match NumPy's exactly (NaN positions, inf signs)."""
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


def check_outputs(seed, got, eager_expect=None):
    """Check a run's outputs (host arrays, program order) for ``seed``:
    integers/bools exact against NumPy (and the eager oracle), floats within
    the per-element bound.  Returns a list of failures."""
    native, transcendental, depth = make_program(seed, Numpy())
    wide, _t, _d = make_program(seed, Numpy(wide=True))
    mag, _t, _d = make_program(seed, Numpy(absolute=True))
    f32 = input_dtype(seed) == np.float32
    bad = []
    for k, (g, nv, wv, mv) in enumerate(zip(got, native, wide, mag)):
        g, nv = np.asarray(g), np.asarray(nv)
        if g.shape != nv.shape or g.dtype != nv.dtype:
            bad.append((k, "shape/dtype", g.shape, nv.shape, g.dtype, nv.dtype))
            continue
        if eager_expect is not None:
            e = eager_expect[k]
            if e.shape != g.shape or e.dtype != g.dtype:
                bad.append((k, "eager shape/dtype"))
                continue
        if g.dtype.kind in "biu":
            if not np.array_equal(g, nv) or (eager_expect is not None and not np.array_equal(g, eager_expect[k])):
                bad.append((k, "integer mismatch"))
            continue
        eps = 2.0 ** -24 if (g.dtype == np.float32 or f32) else 2.0 ** -53
        ok, why = within(g, np.asarray(wv), nv, np.asarray(mv), eps, depth)
        if not ok:
            bad.append((k, why))
    return bad


def make_program(seed, xp=None):
    """(outputs, transcendental, depth): ``transcendental`` marks programs whose
    float results carry libm (ulp-accurate, not correctly rounded) error."""
    xp = xp or GP()
    rng = np.random.default_rng(seed)
    rank, shape, dt = _header(rng)
    fdt = np.dtype(dt).kind == "f"
    pool = []
    for _ in range(int(rng.integers(1, 4))):
        s = list(shape)
        if rng.random() < 0.3:          # broadcastable operand
            s[int(rng.integers(0, rank))] = 1
        a = rng.standard_normal(s) * 4 if fdt else rng.integers(-20, 20, s)
        pool.append(xp.asarray(np.asarray(a, dtype=dt)))
    depth = int(rng.integers(1, 13))
    cur = pool[0]
    transcendental = False   # exp is ulp-accurate, not bit-exact: no branching on it afterwards
    viewed = False
    for _ in range(depth):
        k = rng.integers(0, 14)
        other = pool[int(rng.integers(0, len(pool)))]
        # every random draw happens before the op, so a namespace whose op
        # fails (and is skipped) stays in step with the others
        r1, r2, r3 = rng.random(), rng.random(), rng.random()
        ax_i = int(rng.integers(0, 3))
        n_out = int(rng.integers(1, 17))
        w_seed = int(rng.integers(0, 2 ** 31))
        try:
            kind = getattr(cur, "dtype").kind
            ndim = cur.ndim
            if k == 0:
                cur = cur + other
            elif k == 1:
                cur = xp.sub(cur * other, 1)
            elif k == 2:
                cur = xp.maximum(cur, other)
            elif k == 3 and kind == "f":
                cur = xp.exp(cur * 0.1) + xp.sqrt_abs(cur)
                transcendental = True
            elif k == 4 and not transcendental:
                cur = xp.where_gt(cur, other, other * 2)
            elif k == 5 and ndim >= 2:
                cur = cur.transpose()
                viewed = True
            elif k == 6 and ndim >= 1 and cur.shape[-1] > 2:
                cur = cur[..., 1:] if r1 < 0.5 else cur[..., ::2]
                viewed = True
            elif k == 7 and ndim >= 2:
                cur = cur.reshape(-1, cur.shape[-1])
            elif k == 8 and ndim >= 2:
                ax = ax_i % ndim
                cur = cur.sum(axis=ax, keepdims=bool(r1 < 0.5))
                # NumPy reduces a strided view in memory order, the kernel in C
                # order: same value up to reassociation, so not bit-exact
                transcendental = transcendental or (viewed and cur.dtype.kind == "f")
            elif k == 9 and ndim >= 1:
                cur = xp.minmax(cur, ax_i % ndim, r1 < 0.5)
            elif k == 10 and ndim >= 1:
                cur = cur.astype(np.float64) / 3 if not isinstance(xp, Numpy) or not (xp.wide or xp.absolute) \
                    or cur.dtype.kind != "f" else cur / 3
            elif k == 11 and ndim == 2 and kind == "f":
                # np.dot boundary: GEMM, optionally + bias row and ReLU (the
                # cuBLASLt epilogue pattern); reassociated, so inexact after
                wr = np.random.default_rng(w_seed)
                W = xp.asarray(wr.standard_normal((cur.shape[1], n_out)).astype(dt))
                cur = cur @ W
                if r1 < 0.6:
                    cur = cur + xp.asarray(wr.standard_normal(n_out).astype(dt))
                    if r2 < 0.5:
                        cur = xp.relu(cur)
                transcendental = True
            elif k == 12 and ndim >= 1:
                cur = xp.cumsum(cur, ax_i % ndim)
                transcendental = transcendental or cur.dtype.kind == "f"
            elif k == 13 and ndim >= 1 and cur.shape[-1] >= 2:
                nxt = cur.copy()
                nxt[..., ::2] = cur[..., ::2] * 2 + 1
                cur = nxt
        except xp.errors:
            continue
    finals = [cur]
    r_arg, r_ax, r_sum = rng.random(), int(rng.integers(0, 3)), rng.random()
    if cur.ndim >= 1 and r_arg < 0.5 and not transcendental:
        finals.append(cur.argmax(axis=r_ax % cur.ndim))
    if r_sum < 0.5:
        finals.append(cur.sum())
    return finals, transcendental, depth
