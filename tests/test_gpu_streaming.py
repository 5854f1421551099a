"""Streamed materialisation (streaming.py) on the GPU: results bit-identical
to a plain force, one fused kernel per region per chunk, inputs and roots
left device-resident."""
import numpy as np
import pytest

import paper_1901_03771_b200 as gp
from paper_1901_03771_b200 import runtime, streaming, workloads as wl

pytestmark = pytest.mark.gpu


@pytest.fixture
def small_chunks(monkeypatch):
    monkeypatch.setattr(streaming, "MIN_BYTES", 1)
    monkeypatch.setattr(streaming, "CHUNK_BYTES", 1 << 20)


def _plain(fn, host):
    s = gp.Session()
    outs = fn(*[gp.asarray(h, session=s) for h in host])
    gp.force(*outs)
    return [np.asarray(o) for o in outs]


@pytest.mark.parametrize("pinned", [True, False])
def test_blackscholes_streamed_matches_plain(sess, small_chunks, pinned):
    host = wl.blackscholes_inputs(n=(1 << 18) + 1000)
    fn = lambda S, X, T: wl.blackscholes(gp, S, X, T)
    expect = _plain(fn, host)
    rt = runtime.get()
    if pinned:
        ins = [rt.pinned_empty(h.shape, h.dtype) for h in host]
        for a, h in zip(ins, host):
            a[...] = h
        outs = [rt.pinned_empty(e.shape, e.dtype) for e in expect]
    else:
        ins, outs = list(host), None
    arrs = [gp.asarray(h) for h in ins]
    call, put = fn(*arrs)
    k0 = sess.stats.kernels_executed
    got = gp.materialize(call, put, out=outs)
    nchunks = sess.stats.kernels_executed - k0
    assert nchunks > 4
    for g, e in zip(got, expect):
        assert np.array_equal(g, e)
    assert call.is_materialized and arrs[0].node.data.device is not None
    assert np.array_equal(np.asarray(call + 0.0), expect[0])      # device copy of the root is intact


def test_listing1_and_rowlocal_streamed(sess, small_chunks):
    W, a, b = wl.listing1_inputs(n=1 << 18)
    out = wl.listing1(gp, gp.asarray(W), gp.asarray(a), gp.asarray(b))
    (g,) = gp.materialize(out)
    assert np.array_equal(g, wl.listing1(np, W, a, b))
    (x,) = wl.rownorm_inputs(rows=4096, cols=256)
    y, _tot = wl.rownorm(gp, gp.asarray(x))
    (gy,) = gp.materialize(y)
    ey = _plain(lambda xx: (wl.rownorm(gp, xx)[0],), (x,))[0]
    assert np.array_equal(gy, ey)


def test_mlp_streamed_with_library_steps(sess, small_chunks):
    host = wl.mlp_inputs(batch=8192, hidden=64)
    fn = lambda *a: wl.mlp(gp, *a)
    ep, elab = _plain(fn, host)
    p, lab = fn(*[gp.asarray(h) for h in host])
    gp_, glab = gp.materialize(p, lab)
    # row blocks of a GEMM are computed by the same cuBLAS algorithm family;
    # probabilities within fp32 tolerance, labels exact
    np.testing.assert_allclose(gp_, ep, rtol=1e-5, atol=1e-7)
    assert np.array_equal(glab, elab)


def test_partials_streamed(sess, small_chunks):
    """Partial roots (a total, bincounts) are combined across chunks; row-local
    roots stay bit-identical."""
    (x,) = wl.rownorm_inputs(rows=4096, cols=256)
    y, tot = wl.rownorm(gp, gp.asarray(x))
    c0 = sess.stats.streamed_chunks
    gy, gt = gp.materialize(y, tot)
    assert sess.stats.streamed_chunks - c0 > 4
    ey, et = wl.rownorm(np, x)
    assert np.array_equal(gy, np.asarray(_plain(lambda xx: (wl.rownorm(gp, xx)[0],), (x,))[0]))
    # |total| is rounding noise around 0: bound by eps * sum|y|
    assert abs(float(gt) - float(et)) <= 4 * np.finfo(np.float32).eps * float(np.abs(ey).sum())
    assert np.asarray(tot).shape == () and tot.is_materialized

    P, C = wl.kmeans_inputs(n=1 << 16, k=64, d=4)
    lab, sums, counts = wl.kmeans_partials(gp, gp.asarray(P), gp.asarray(C))
    got = gp.materialize(lab, *sums, counts)
    elab, esums, ecounts = wl.kmeans_partials(np, P, C)
    assert np.array_equal(got[0], elab)
    assert np.array_equal(got[-1], ecounts)
    for g, e in zip(got[1:-1], esums):
        np.testing.assert_allclose(g, e, rtol=1e-12, atol=1e-9)
    m = gp.asarray(np.arange(1 << 18, dtype=np.float64))
    (s,) = gp.materialize((m * 0.5).max(0) + 0 * (m * 0.5).sum())
    assert float(s) == 0.5 * ((1 << 18) - 1)


@pytest.mark.parametrize("seed", range(60))
def test_streamed_random_program(sess, monkeypatch, seed):
    """The randomised programs of test_gpu_programs.py through materialize()
    with tiny chunks: streamed whenever eligible, same answers as the oracle
    (row-local results bit-identical to the plain force)."""
    from oracle import eager
    from random_programs import check_outputs, make_program
    monkeypatch.setattr(streaming, "MIN_BYTES", 1)
    monkeypatch.setattr(streaming, "ROW_ALIGN", 1)
    monkeypatch.setattr(streaming, "CHUNK_BYTES", 96)
    outs, transcendental, _depth = make_program(seed)
    expect = [eager.evaluate(o.node) for o in outs]
    got = gp.materialize(*outs)
    bad = check_outputs(seed, got, expect)
    assert not bad, (seed, bad)



def test_scans_streamed_with_carry(sess, small_chunks):
    """Scans along the streamed axis ("C" roots): each chunk scans its rows
    and continues from the previous chunk's last value.  Integers exact;
    floats no less accurate than NumPy's own sequential fold."""
    rng = np.random.default_rng(12)
    xi = rng.integers(-50, 50, 1 << 18)
    c0 = sess.stats.streamed_chunks
    (gi,) = gp.materialize(gp.cumsum(gp.asarray(xi) * 3 + 1))
    assert sess.stats.streamed_chunks - c0 >= 4
    assert np.array_equal(gi, np.cumsum(xi * 3 + 1))
    xm = rng.standard_normal((1 << 16, 8))
    (gm,) = gp.materialize(np.maximum.accumulate(gp.asarray(xm), axis=0))
    assert np.array_equal(gm, np.maximum.accumulate(xm, axis=0))
    (g2,) = gp.materialize(gp.cumsum(gp.asarray(xm) * 2, axis=0))
    assert np.array_equal(np.asarray(g2)[:1], xm[:1] * 2)
    xf = rng.standard_normal(1 << 18)
    (gf,) = gp.materialize(gp.cumsum(gp.exp(gp.asarray(xf) * 0.1)))
    ref = np.cumsum(np.exp(xf * 0.1))
    exact = np.cumsum(np.exp(xf * 0.1).astype(np.longdouble))
    assert np.max(np.abs(gf - exact)) <= 2 * np.max(np.abs(ref - exact)) + 2.2e-16 * float(exact[-1])
    e2 = np.cumsum((xm * 2).astype(np.longdouble), axis=0)
    r2 = np.cumsum(xm * 2, axis=0)
    assert np.max(np.abs(g2 - e2)) <= 2 * np.max(np.abs(r2 - e2)) + 2.2e-16 * float(np.abs(e2).max())


def test_streamed_with_device_operand(sess, small_chunks):
    """x_host + y_device of the same extent: y is chunked as row views of its
    device buffer; results equal NumPy's."""
    rng = np.random.default_rng(31)
    xh = rng.standard_normal((1 << 16, 4))
    yh = rng.standard_normal((1 << 16, 4))
    y = gp.asarray(yh)
    gp.force(y * 1.0)
    y.node.data.device = runtime.get().upload(yh)
    k0 = sess.stats.streamed_chunks
    (got,) = gp.materialize(gp.asarray(xh) * 2 + y)
    assert sess.stats.streamed_chunks > k0
    assert np.array_equal(got, xh * 2 + yh)


def test_partial_and_carried_roots_read_by_other_roots(sess, small_chunks):
    """materialize(t, x - t) with t = x.sum(0) and (s, s + a) with s a scan:
    not streamed (the consumer needs the combined value) and exact."""
    rng = np.random.default_rng(32)
    xh = rng.standard_normal((1 << 16, 3))
    x = gp.asarray(xh)
    t = x.sum(0)
    got_t, got_d = gp.materialize(t, x - t)
    assert np.array_equal(got_t, xh.sum(0)) and np.array_equal(got_d, xh - xh.sum(0))
    ah = rng.integers(-5, 5, 1 << 16)
    a = gp.asarray(ah)
    s = gp.cumsum(a * 2)
    got_s, got_u = gp.materialize(s, s + a)
    assert np.array_equal(got_s, np.cumsum(ah * 2)) and np.array_equal(got_u, np.cumsum(ah * 2) + ah)
