"""Eligibility of streamed materialisation (streaming.py) — DAG analysis only."""
import numpy as np
import pytest

import paper_1901_03771_b200 as gp
from paper_1901_03771_b200 import streaming, workloads as wl


@pytest.fixture(autouse=True)
def small_chunks(monkeypatch):
    monkeypatch.setattr(streaming, "MIN_BYTES", 1)
    monkeypatch.setattr(streaming, "CHUNK_BYTES", 64 << 10)


def test_blackscholes_streams():
    S, X, T = wl.blackscholes_inputs(n=1 << 16)
    call, put = wl.blackscholes(gp, gp.asarray(S), gp.asarray(X), gp.asarray(T))
    p = streaming.plan([call.node, put.node])
    assert p is not None and p.N == 1 << 16 and p.rows % streaming.ROW_ALIGN == 0 and p.rows < p.N
    assert len(p.leaves) == 3


def test_row_local_and_library_stream():
    (x,) = wl.rownorm_inputs(rows=4096, cols=64)
    y, tot = wl.rownorm(gp, gp.asarray(x))
    assert streaming.plan([y.node]) is not None            # row statistics are row-local
    p2 = streaming.plan([y.node, tot.node])                # the total: a partial combined over chunks
    assert p2 is not None and p2.dist[tot.node.id] == "P:sum"
    X, W1, b1, W2, b2 = wl.mlp_inputs(batch=4096, hidden=32)
    p, lab = wl.mlp(gp, *[gp.asarray(a) for a in (X, W1, b1, W2, b2)])
    assert streaming.plan([p.node, lab.node]) is not None  # X@W1 with W1 replicated


def test_partials_and_ineligible():
    P, C = wl.kmeans_inputs(n=4096, k=8, d=4)
    lab, sums, counts = wl.kmeans_partials(gp, gp.asarray(P), gp.asarray(C))
    p = streaming.plan([lab.node] + [s.node for s in sums] + [counts.node])   # bincount partials
    assert p is not None and p.dist[counts.node.id] == "P:sum"
    a = gp.asarray(np.arange(65536.0))
    assert streaming.plan([(a * 2).sum().node]) is not None             # a total alone
    assert streaming.plan([(a * 2).argmax().node]) is None              # arg-reduction over the streamed axis
    x = gp.asarray(np.ones((4096, 3)))
    assert streaming.plan([(x - x.mean(0)).node]) is None               # a partial consumed inside
    ps = streaming.plan([gp.cumsum(a * 2).node])                         # scan along the streamed axis: carried
    assert ps is not None and list(ps.dist.values()).count("C:sum") == 1
    assert streaming.plan([(gp.cumsum(a * 2) + 1).node]) is None         # a carried scan consumed inside
    small = gp.asarray(np.ones(100))
    assert streaming.plan([(small + 1).node]) is None                   # too few rows


def test_streamed_random_programs_do_stream(monkeypatch):
    """Enough of the random programs are streaming-eligible for the test above
    to exercise the chunked path (not just the fallback)."""
    from random_programs import make_program
    monkeypatch.setattr(streaming, "MIN_BYTES", 1)
    monkeypatch.setattr(streaming, "ROW_ALIGN", 1)
    monkeypatch.setattr(streaming, "CHUNK_BYTES", 96)
    streamed = 0
    for seed in range(200):
        s = gp.Session()
        old = gp.set_default_session(s)
        try:
            outs, _t, _d = make_program(seed)
            if streaming.plan([o.node for o in outs]) is not None:
                streamed += 1
        finally:
            gp.set_default_session(old)
    assert streamed >= 8, streamed


def test_partial_or_carried_root_read_by_another_root_is_ineligible():
    """A partial (total) or carried scan that is itself a root but also read by
    another root would feed each chunk its chunk-local value."""
    x = gp.asarray(np.ones((4096, 3)))
    t = x.sum(0)
    assert streaming.plan([t.node, (x - t).node]) is None
    a = gp.asarray(np.arange(65536.0))
    s = gp.cumsum(a * 2)
    assert streaming.plan([s.node, (s + a).node]) is None
    assert streaming.plan([s.node, (a + 1).node]) is not None        # independent roots still stream


class _FakeDev:
    """Stands in for a device allocation (plan() only reads ptr/nbytes)."""

    def __init__(self, nbytes):
        self.ptr = 1 << 20
        self.nbytes = nbytes


def test_device_operand_with_streamed_extent_is_chunked():
    """A device-resident operand of the streamed extent is a chunked leaf (a
    row view of its buffer), not a full-size operand inside every chunk."""
    xh = np.ones((65536, 4))
    y = gp.asarray(np.ones((65536, 4)))
    y.node.data.device = _FakeDev(y.node.data.nbytes)
    y.node.data.host = None
    p = streaming.plan([(gp.asarray(xh) + y).node])
    assert p is not None and [l.id for l in p.dev_leaves] == [y.node.id] and p.dist[y.node.id] == "S"
