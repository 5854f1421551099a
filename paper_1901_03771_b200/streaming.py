"""Streamed materialisation: host inputs -> fused kernels -> host outputs with
the PCIe copies overlapping the kernels.

The reference moves every kernel's inputs to the device and its results back
around each launch ("automatic H2D/D2H"), serially.  When a
forced region reads host-resident arrays and its result is wanted on the host
(``to_external``), the device sits idle during the copies.
Here such a force is cut along the leading axis into chunks that run through
three streams:

    copy-in stream   H2D of chunk c's inputs            (waits: nothing new)
    runtime stream   chunk c's plan steps (one fused kernel per region)
                                                         (waits: chunk c in)
    copy-out stream  D2H of chunk c's results            (waits: chunk c done)

so H2D(c+1), kernels(c) and D2H(c-1) overlap.  Eligibility is the sharding
analysis of distributed.py with the host inputs as the sharded set: every
forced root is *sharded* (row-local along the leading axis) or a partial over
it (a total, a reduction over axis 0, a bincount): partials are combined
across chunks in a binary tree over chunk order once the last chunk ran.  Each chunk re-
records the DAG on row slices (same ops, leading extent rewritten), so each
chunk's region is the same fused kernel as the whole force, and results are
bit-identical to the unchunked force (rows are independent).  Inputs and
results land in full-size device buffers (chunks are views), so after the
call the forced roots and the inputs are device-resident exactly as after a
plain force.
"""

from __future__ import annotations

import os
from typing import Dict, List, Optional, Sequence

import numpy as np

from .dag import ElemCode, Node, Op, OpKind
from .errors import LazyFuseError
from .tensor import TensorBuffer, element_count

CHUNK_BYTES = int(os.environ.get("GRUMPY_STREAM_CHUNK_MB", "128")) << 20   # host bytes (in + out) per chunk
MIN_BYTES = 48 << 20        # smaller forces gain nothing from overlap
ROW_ALIGN = 256             # chunk row counts: 16-byte aligned views, full vectors

_ALLOWED = {OpKind.MAP, OpKind.CAST, OpKind.BROADCAST, OpKind.TRANSPOSE, OpKind.RESHAPE,
            OpKind.SLICE, OpKind.REDUCE, OpKind.ARGREDUCE, OpKind.MATMUL, OpKind.MATVEC, OpKind.KEYED_SUM,
            OpKind.SCAN}


class DeviceView:
    """A byte range of a pool allocation (keeps the allocation alive)."""

    __slots__ = ("ptr", "nbytes", "base")

    def __init__(self, base, offset: int, nbytes: int):
        self.base = base
        self.ptr = base.ptr + offset
        self.nbytes = nbytes


class StreamPlan:
    __slots__ = ("roots", "nodes", "leaves", "dev_leaves", "dist", "N", "rows")


def _walk(roots: Sequence[Node]):
    """Unmaterialized nodes reachable from roots (pred-first) and the frontier."""
    order, frontier, seen = [], {}, set()
    stack = [(r, False) for r in roots]
    while stack:
        n, done = stack.pop()
        if done:
            order.append(n)
            continue
        if n.id in seen:
            continue
        seen.add(n.id)
        if n.is_materialized:
            frontier[n.id] = n
            continue
        stack.append((n, True))
        stack.extend((p, False) for p in n.preds)
    return order, list(frontier.values())


_COMBINE = {"sum": ElemCode.add, "prod": ElemCode.mul, "max": ElemCode.maximum, "min": ElemCode.minimum}


def plan(roots: Sequence[Node], chunk_bytes: Optional[int] = None) -> Optional[StreamPlan]:
    """A chunked plan for forcing ``roots`` to host, or None if ineligible.

    Roots are row-local along the streamed axis ("S": their leading extent is
    the host inputs') or partials over it ("P:<op>": full/leading-axis
    reductions and bincounts, combined across chunks after the last chunk)."""
    from . import distributed as D
    chunk_bytes = chunk_bytes or CHUNK_BYTES
    roots = list(dict((r.id, r) for r in roots).values())
    if not roots or any(r.is_materialized for r in roots):
        return None
    nodes, frontier = _walk(roots)
    if any(n.kind not in _ALLOWED for n in nodes if n.preds):
        return None
    host = [f for f in frontier if f.data.device is None and f.data.host is not None and f.shape]
    if not host:
        return None
    N = max(host, key=lambda f: f.data.nbytes).shape[0]
    leaves = [f for f in host if f.shape[0] == N]
    if any(not l.data.host.flags.c_contiguous for l in leaves):
        return None
    # device-resident operands with the streamed extent are chunked too (row
    # views of their buffer, no copy); used at full size inside a chunk they
    # would not match the chunk's rows
    dev_leaves = [f for f in frontier if f.data.device is not None and f.shape and f.shape[0] == N]
    if N < 2 * ROW_ALIGN:
        return None
    try:
        dist = D.classify(roots, sharded={l.id for l in leaves + dev_leaves}, scans=True)
    except LazyFuseError:
        return None
    root_ids = {r.id for r in roots}
    for r in roots:
        d = dist.get(r.id, "R")
        if d == "S" or d.startswith("C:"):
            if not r.shape or r.shape[0] != N or (d.startswith("C:") and d[2:] not in _COMBINE):
                return None
        elif not (d.startswith("P:") and d[2:] in _COMBINE):
            return None
    for n in nodes:
        if n.id in dist and dist[n.id][0] in "PAC" and n.id not in root_ids:
            return None                      # a partial or carried scan inside the region
        for q in n.preds:
            if dist.get(q.id, "R")[0] in "PAC":
                # a partial / carried scan (root or not) consumed inside the
                # region: each chunk would read its chunk-local value, before
                # the cross-chunk combine or carry
                return None
    srows = [r for r in roots if dist[r.id] == "S" or dist[r.id].startswith("C:")]
    total = sum(l.data.nbytes for l in leaves) + sum(element_count(r.shape) * r.dtype.itemsize for r in srows)
    if total < MIN_BYTES:
        return None
    per_row = total / N
    rows = max(ROW_ALIGN, int(chunk_bytes / per_row) // ROW_ALIGN * ROW_ALIGN)
    if rows >= N:
        return None
    p = StreamPlan()
    p.roots, p.nodes, p.leaves, p.dist, p.N, p.rows = roots, nodes, leaves, dist, N, rows
    p.dev_leaves = dev_leaves
    return p


def _rewrite(op: Op, c: int) -> Op:
    """``op`` with the sharded leading extent replaced by the chunk's ``c``."""
    k = op.kind
    if k in (OpKind.RESHAPE, OpKind.BROADCAST):
        shape = tuple(op.attrs[0])
        return Op(k, op.code, ((c,) + shape[1:],) + tuple(op.attrs[1:]))
    if k is OpKind.SLICE:
        sl = tuple(op.attrs[0])
        return Op(k, op.code, (((0, 1, c),) + sl[1:],) + tuple(op.attrs[1:]))
    return op


def _row_bytes(n: Node) -> int:
    return element_count(n.shape[1:]) * n.dtype.itemsize


class _Streams:
    """Per-runtime copy streams and a reusable event pool."""

    def __init__(self, rt):
        self.rt = rt
        self.h2d = rt.stream_create()
        self.d2h = rt.stream_create()
        self.events: List[int] = []

    def event(self, i: int) -> int:
        while len(self.events) <= i:
            self.events.append(self.rt.event())
        return self.events[i]


def _streams(rt) -> _Streams:
    s = getattr(rt, "_gr_streams", None)
    if s is None:
        s = _Streams(rt)
        rt._gr_streams = s
    return s


def run(sess, p: StreamPlan, outs: Sequence[np.ndarray]) -> List[np.ndarray]:
    """Execute plan ``p``: results land in ``outs`` (host, C-contiguous, ideally
    page-locked) and in device buffers attached to the forced roots."""
    ex = sess.executor
    rt = ex.rt
    st = _streams(rt)
    g = sess.graph
    N, rows = p.N, p.rows
    srows = [r for r in p.roots if p.dist[r.id] == "S" or p.dist[r.id].startswith("C:")]
    carried = {r.id for r in p.roots if p.dist[r.id].startswith("C:")}   # scans along the streamed axis
    parts = {r.id: [] for r in p.roots if r not in srows}   # per-chunk partial nodes
    prev_final: Dict[int, Node] = {}
    # full-size device buffers: inputs and row-local results (chunks are views)
    dev_in = {l.id: rt.alloc(l.data.nbytes) for l in p.leaves}
    dev_out = {r.id: rt.alloc(element_count(r.shape) * r.dtype.itemsize) for r in srows}
    chunks = [(lo, min(rows, N - lo)) for lo in range(0, N, rows)]
    sess.stats.streamed_chunks += len(chunks)
    ev = 0
    keep = []
    try:
        # copies into freshly handed-out pool blocks start only after the
        # work already queued on the runtime stream (which may still be
        # reading those blocks' previous contents)
        e_start = st.event(ev)
        ev += 1
        rt.record(e_start)
        rt.set_stream(st.h2d)
        rt.wait_event(e_start)
        rt.set_stream(st.d2h)
        rt.wait_event(e_start)
        rt.set_stream(0)

        def stage_in(ci):
            nonlocal ev
            lo, c = chunks[ci]
            rt.set_stream(st.h2d)
            for l in p.leaves:
                rb = _row_bytes(l)
                rt.h2d_async(dev_in[l.id].ptr + lo * rb, l.data.host[lo:lo + c])
                sess.stats.h2d_bytes += c * rb
            e = st.event(ev)
            ev += 1
            rt.record(e)
            rt.set_stream(0)
            return e

        def compute(ci, e_in):
            nonlocal ev
            lo, c = chunks[ci]
            rt.wait_event(e_in)
            memo: Dict[int, Node] = {}
            for l in p.leaves:
                rb = _row_bytes(l)
                buf = TensorBuffer(l.dtype, (c,) + tuple(l.shape[1:]), device=DeviceView(dev_in[l.id], lo * rb, c * rb))
                memo[l.id] = g.add_input(buf)
            for l in p.dev_leaves:
                rb = _row_bytes(l)
                buf = TensorBuffer(l.dtype, (c,) + tuple(l.shape[1:]),
                                   device=DeviceView(l.data.device, lo * rb, c * rb))
                memo[l.id] = g.add_input(buf)
            for n in p.nodes:
                if p.dist.get(n.id, "R") == "S" or n.id in parts or n.id in carried:
                    memo[n.id] = g.add_op(_rewrite(n.op, c), [memo.get(q.id, q) for q in n.preds])
            for r in p.roots:
                if r.id in carried and ci > 0:
                    # continue from the previous chunk's last row (its scan
                    # result is already on the device, stream-ordered): the
                    # chunk's scan is SEEDED with it — one kernel writes the
                    # chunk once (a second map pass re-read and
                    # re-wrote every chunk)
                    pf = prev_final[r.id]
                    sl = ((pf.shape[0] - 1, 1, 1),) + tuple((0, 1, e) for e in pf.shape[1:])
                    carry = g.add_op(Op(OpKind.SLICE, None, (sl,)), [pf])
                    sc = memo[r.id]
                    axis = sc.op.attrs[1]
                    xs = sc.preds[0].shape
                    kept = (1,) if axis is None or len(xs) == 1 else tuple(d for i, d in enumerate(xs) if i != axis)
                    if tuple(carry.shape) != kept:
                        carry = g.add_op(Op(OpKind.RESHAPE, None, (kept,)), [carry])
                    memo[r.id] = g.add_op(sc.op, [sc.preds[0], carry])
            croots = [memo[r.id] for r in p.roots]
            views = {}
            for r, cr in zip(p.roots, croots):
                if r.id in dev_out:
                    rb = _row_bytes(r)
                    views[cr.id] = TensorBuffer(cr.dtype, cr.shape, device=DeviceView(dev_out[r.id], lo * rb, c * rb))
            ex.out_bind = dict(views)
            try:
                sess.force_nodes(croots)
            finally:
                ex.out_bind = {}
            for r, cr in zip(p.roots, croots):
                if r.id in parts:
                    parts[r.id].append(cr)
                elif cr.data is not views[cr.id]:
                    # produced by a library call (cuBLAS output): move it in
                    rb = _row_bytes(r)
                    rt.d2d_raw(dev_out[r.id].ptr + lo * rb, cr.data.device.ptr, c * rb)
            for r, cr in zip(p.roots, croots):
                if r.id in carried:
                    prev_final[r.id] = cr
            keep.append(croots)
            e = st.event(ev)
            ev += 1
            rt.record(e)
            return e

        def stage_out(ci, e_k):
            lo, c = chunks[ci]
            rt.set_stream(st.d2h)
            rt.wait_event(e_k)
            for r, o in zip(p.roots, outs):
                if r.id not in dev_out:
                    continue
                rb = _row_bytes(r)
                rt.d2h_async(o[lo:lo + c], dev_out[r.id].ptr + lo * rb)
                sess.stats.d2h_bytes += c * rb
            rt.set_stream(0)

        # software pipeline in enqueue order too (pageable copies block the
        # host): in(c+1) is queued before out(c)
        e_in = [stage_in(0)]
        for ci in range(len(chunks)):
            e_k = compute(ci, e_in[ci])
            if ci + 1 < len(chunks):
                e_in.append(stage_in(ci + 1))
            stage_out(ci, e_k)
        # partials: combine the chunks' values in a binary tree over chunk
        # order (one small fused map kernel, on the runtime stream after the
        # chunk kernels)
        finals = {}
        for r in p.roots:
            if r.id in parts:
                code = _COMBINE[p.dist[r.id][2:]]
                level = list(parts[r.id])
                while len(level) > 1:
                    nxt = [g.add_op(Op(OpKind.MAP, code), [level[i], level[i + 1]]) for i in range(0, len(level) - 1, 2)]
                    if len(level) % 2:
                        nxt.append(level[-1])
                    level = nxt
                finals[r.id] = level[0]
        if finals:
            sess.force_nodes(list(finals.values()))
        rt.sync()
    finally:
        rt.set_stream(0)
    del keep
    for l in p.leaves:
        if l.data.device is None:
            l.data.device = dev_in[l.id]
    for r, o in zip(p.roots, outs):
        if r.is_materialized:
            continue
        if r.id in dev_out:
            g.mark_materialized(r, TensorBuffer(r.dtype, r.shape, device=dev_out[r.id]))
        else:
            f = finals[r.id]
            if f.dtype is not r.dtype or tuple(f.shape) != tuple(r.shape):
                raise LazyFuseError(f"streamed partial of node {r.id} combined to {f.dtype.value}{f.shape}")
            g.mark_materialized(r, TensorBuffer(r.dtype, r.shape, device=f.data.device))
            f.data.device.copy_to_host(o)
            sess.stats.d2h_bytes += o.nbytes
    return list(outs)
