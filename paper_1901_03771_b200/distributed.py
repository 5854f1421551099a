"""Leading-axis sharding of fused regions across GPUs (one process per GPU).

north_star: "Fused regions shard along the leading axis across 1, 2, 4 and 8
GPUs of one 8×B200 box, and reduction partials are combined with NCCL
allreduce over NVLink".  The reference has no distributed
layer (single process, worker pool — SPEC.md:412-413), so this module is new:

* ``init()`` — one process per GPU (torchrun env); the NCCL communicator is
  created by the C-ABI shim (ncclCommInitRank) from a unique id broadcast over
  torch.distributed's gloo group (plumbing only); collectives then run on the
  runtime's single stream, ordered after the kernels that produce the partials;
* ``shard_rows(arr)`` — this rank's contiguous slice of a host array's leading
  axis as a grumpy input marked *sharded*;
* ``classify`` — distribution of every DAG node: ``S`` sharded, ``R``
  replicated, ``P:<op>`` partial (a reduction over the sharded axis, a bincount
  of sharded keys, a matmul contracting a sharded axis) or ``A:<max|min>``
  (first-index arg-reduction over the sharded axis).  Partial nodes are forced
  to be step roots; after their kernel the executor allreduces them in place
  (sum/prod/max/min → ncclAllReduce).  Arg partials are combined on the
  device: ncclAllGather of every rank's (best value, global index), then an
  arg-reduction over the rank axis (lower ranks hold lower global indices, so
  NumPy's first-index and NaN rules carry over) selects the index.

Elementwise regions need no communication at all (weak or strong scaling is
the caller's choice of shard size).
"""

from __future__ import annotations

import os
from typing import Dict, Optional

import numpy as np

from .dag import Node, OpKind, ReduceOp
from .errors import ShapeMismatch

_SHARDED: "Dict[int, tuple]" = {}   # input node id -> (global extent, offset)

GR_OP = {ReduceOp.sum: 0, ReduceOp.prod: 1, ReduceOp.max: 2, ReduceOp.min: 3}


class Comm:
    """Partial-combination interface; ``rank``/``world`` of the process group."""

    rank = 0
    world = 1

    def allreduce_host(self, arr: np.ndarray, op: ReduceOp) -> np.ndarray:
        raise NotImplementedError

    def allgather_host(self, arr: np.ndarray) -> np.ndarray:
        raise NotImplementedError

    def allreduce_device(self, buf, count: int, dtype, op: ReduceOp):
        raise NotImplementedError

    def allgather_device(self, rt, buf, count: int, dtype):
        """Rank-ordered concatenation of every rank's ``count`` elements of
        ``buf`` into a new device buffer of world * count elements."""
        raise NotImplementedError

    def group(self):
        """Context manager batching the collectives issued inside it."""
        import contextlib
        return contextlib.nullcontext()


class TorchHostComm(Comm):
    """torch.distributed (gloo) on host arrays: CPU tests and host-side combines."""

    def __init__(self):
        import torch.distributed as td
        self.td = td
        self.rank = td.get_rank()
        self.world = td.get_world_size()

    def allreduce_host(self, arr, op):
        import torch
        arr = np.asarray(arr)
        t = torch.from_numpy(np.array(arr, copy=True).reshape(-1))
        top = {ReduceOp.sum: self.td.ReduceOp.SUM, ReduceOp.prod: self.td.ReduceOp.PRODUCT,
               ReduceOp.max: self.td.ReduceOp.MAX, ReduceOp.min: self.td.ReduceOp.MIN}[op]
        self.td.all_reduce(t, op=top)
        return t.numpy().reshape(arr.shape)

    def allgather_host(self, arr):
        import torch
        arr = np.asarray(arr)
        t = torch.from_numpy(np.array(arr, copy=True).reshape(-1))
        out = [torch.empty_like(t) for _ in range(self.world)]
        self.td.all_gather(out, t)
        return np.stack([o.numpy().reshape(arr.shape) for o in out])


class NcclComm(TorchHostComm):
    """NCCL over NVLink for device partials (the shim's communicator), gloo for
    the unique-id bootstrap and small host-side exchanges."""

    def __init__(self, rt):
        super().__init__()
        self.rt = rt
        rt.nccl_load()
        uid = [rt.nccl_unique_id() if self.rank == 0 else None]
        self.td.broadcast_object_list(uid, src=0)
        rt.nccl_init(self.rank, self.world, uid[0])

    def allreduce_device(self, buf, count, dtype, op):
        self.rt.nccl_allreduce(buf.ptr, buf.ptr, count, dtype, GR_OP[op])

    def allgather_device(self, rt, buf, count, dtype):
        out = rt.alloc(max(1, self.world * count * dtype.itemsize))
        self.rt.nccl_allgather(buf.ptr, out.ptr, count, dtype)
        return out

    def group(self):
        """ncclGroupStart/End: the step's allreduces go out as one launch."""
        import contextlib

        @contextlib.contextmanager
        def cm():
            self.rt.nccl_group_start()
            try:
                yield
            finally:
                self.rt.nccl_group_end()
        return cm()


class HostStagedComm(TorchHostComm):
    """Device partials combined through host memory over gloo — used when two
    ranks of the group share one GPU, where NCCL refuses to build a
    communicator (a single-GPU box running a multi-rank job)."""

    def __init__(self, rt):
        super().__init__()
        self.rt = rt

    def allreduce_device(self, buf, count, dtype, op):
        host = buf.to_numpy(dtype, (count,))
        buf.copy_from_host(np.ascontiguousarray(self.allreduce_host(host, op).astype(host.dtype)))

    def allgather_device(self, rt, buf, count, dtype):
        host = buf.to_numpy(dtype, (count,))
        return rt.upload(np.ascontiguousarray(self.allgather_host(host).reshape(-1).astype(host.dtype)))


def _ranks_share_a_device(rt) -> bool:
    import socket
    import torch.distributed as td
    me = (socket.gethostname(), int(getattr(rt, "device", 0)))
    allv = [None] * td.get_world_size()
    td.all_gather_object(allv, me)
    return len(set(allv)) < len(allv)


def init(backend: Optional[str] = None, session=None) -> Comm:
    """Join the process group launched by torchrun (RANK/WORLD_SIZE/MASTER_*)."""
    import torch.distributed as td
    from . import session as _s
    sess = session or _s.default_session()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world <= 1 and backend is None:
        sess.comm = None
        return None
    if not td.is_initialized():
        td.init_process_group("gloo")
    if backend == "gloo":
        comm = TorchHostComm()
    else:
        from . import runtime
        rt = runtime.get()
        comm = HostStagedComm(rt) if _ranks_share_a_device(rt) else NcclComm(rt)
    sess.comm = comm
    return comm


def split(n: int, world: int, rank: int):
    """Balanced contiguous split of n rows: (offset, length) of ``rank``."""
    base, rem = divmod(n, world)
    off = rank * base + min(rank, rem)
    return off, base + (1 if rank < rem else 0)


def shard_rows(arr, comm: Optional[Comm] = None, session=None):
    """This rank's slice of ``arr`` along axis 0, as a sharded grumpy input."""
    from . import session as _s
    sess = session or _s.default_session()
    comm = comm or sess.comm
    arr = np.asarray(arr)
    rank, world = (comm.rank, comm.world) if comm is not None else (0, 1)
    off, ln = split(arr.shape[0], world, rank)
    a = _s.asarray(np.ascontiguousarray(arr[off:off + ln]), session=sess)
    _SHARDED[a.node.id] = (arr.shape[0], off)
    return a


def local_input(arr, global_rows: int, offset: int, session=None):
    """Register an already-local shard (e.g. generated per rank)."""
    from . import session as _s
    a = _s.asarray(arr, session=session)
    _SHARDED[a.node.id] = (global_rows, offset)
    return a


def shard_info(node: Node):
    return _SHARDED.get(node.id)


def leaf_dist(node: Node) -> str:
    """Distribution tag of a materialized leaf (a plan-cache key part)."""
    if node.id in _SHARDED:
        return "S"
    return getattr(node, "dist", None) or "R"


def shard_of(node: Node):
    """(global leading extent, this rank's offset) of the sharded input that
    ``node``'s leading axis comes from, or None."""
    stack = [node]
    seen = set()
    while stack:
        n = stack.pop()
        if n.id in seen:
            continue
        seen.add(n.id)
        info = _SHARDED.get(n.id)
        if info is not None:
            return info
        stack.extend(n.preds)
    return None


def classify(roots, memo: Optional[dict] = None, sharded=None, scans: bool = False) -> Dict[int, str]:
    """Distribution of every unmaterialized node reachable from roots (plus the
    materialized frontier): "S", "R", "P:<op>", "A:<max|min>".  ``sharded``
    (node ids) replaces the registered shard inputs, e.g. the host inputs of a
    streamed force (streaming.py)."""
    memo = {} if memo is None else memo
    shards = _SHARDED if sharded is None else sharded

    def dist(n: Node) -> str:
        d = memo.get(n.id)
        if d is not None:
            return d
        d = _dist(n)
        memo[n.id] = d
        return d

    def _dist(n: Node) -> str:
        if n.id in shards:
            return "S"
        if n.is_materialized:
            return getattr(n, "dist", None) or "R"
        k = n.kind
        ps = [dist(p) for p in n.preds]
        if any(p.startswith(("P", "A", "C")) for p in ps):
            # a partial consumed before its allreduce: planner makes it a root
            ps = ["R" if p.startswith(("P", "A", "C")) else p for p in ps]
        if not any(p == "S" for p in ps):
            return "R"
        if k in (OpKind.MAP, OpKind.CAST, OpKind.BROADCAST, OpKind.SLICE_ASSIGN):
            for p, dp in zip(n.preds, ps):
                if dp == "S" and (len(p.shape) != len(n.shape) or p.shape[0] != n.shape[0]):
                    raise ShapeMismatch("a sharded operand must keep its leading axis in an elementwise op")
            return "S"
        if k is OpKind.TRANSPOSE:
            if n.op.attrs[0][0] != 0:
                raise ShapeMismatch("transposing the sharded leading axis is not supported")
            return "S"
        if k is OpKind.RESHAPE:
            if not n.shape or n.shape[0] != n.preds[0].shape[0]:
                raise ShapeMismatch("reshaping across the sharded leading axis is not supported")
            return "S"
        if k is OpKind.SLICE:
            st, step, ln = n.op.attrs[0][0]
            if not (st == 0 and step == 1 and ln == n.preds[0].shape[0]):
                raise ShapeMismatch("slicing the sharded leading axis is not supported")
            return "S"
        if k is OpKind.REDUCE:
            rop, axes = n.op.attrs[0], n.op.attrs[1]
            return f"P:{rop.value}" if 0 in axes else "S"
        if k is OpKind.ARGREDUCE:
            which, axis = n.op.attrs[0], n.op.attrs[1]
            return f"A:{which}" if axis in (None, 0) else "S"
        if k is OpKind.KEYED_SUM:
            return "P:sum"
        if k is OpKind.MATMUL:
            a, b = ps
            if a == "S" and b == "R":
                return "S"
            if a == "R" and b == "S":
                return "P:sum"
            raise ShapeMismatch("matmul of two sharded operands is not supported")
        if k is OpKind.MATVEC:
            trans = n.op.attrs[0]
            m, x = ps
            if not trans and m == "S" and x == "R":
                return "S"
            if (not trans and m == "R" and x == "S") or (trans and m == "S" and x == "S"):
                return "P:sum"
            if trans and m == "S" and x == "R":
                raise ShapeMismatch("x @ M with M sharded on its rows needs x sharded too")
            raise ShapeMismatch("unsupported sharding of a matrix-vector product")
        if k is OpKind.SCAN:
            axis = n.op.attrs[1]
            if axis not in (None, 0):
                return "S"                       # along a row-local axis
            if scans and (axis == 0 or len(n.preds[0].shape) == 1):
                # along the sharded axis: "C:<op>" = carried — each part scans
                # its rows and continues from the previous part's last value
                # (streamed to_external, streaming.py)
                return f"C:{n.op.attrs[0].value}"
            raise ShapeMismatch("cumulative ops along a sharded axis are not supported yet")
        raise ShapeMismatch(f"{n.op!r} on a sharded operand")

    for r in roots:
        dist(r)
    return memo


def combine_arg(which: str, local_idx: np.ndarray, local_val: np.ndarray, offset: int, comm: Comm) -> np.ndarray:
    """Global first-index arg-reduction from per-rank (value, local index).

    ranks hold consecutive row ranges, so lower ranks have lower global
    indices; NaN beats numbers, ties go to the lower index (np.argmax)."""
    gidx = comm.allgather_host(np.asarray(local_idx, dtype=np.int64) + offset)
    gval = comm.allgather_host(np.asarray(local_val))
    best_v = gval[0].copy()
    best_i = gidx[0].copy()
    for r in range(1, gval.shape[0]):
        v, i = gval[r], gidx[r]
        bn = np.isnan(best_v) if best_v.dtype.kind == "f" else np.zeros(best_v.shape, bool)
        vn = np.isnan(v) if v.dtype.kind == "f" else np.zeros(v.shape, bool)
        better = (v > best_v) if which == "max" else (v < best_v)
        take = (~bn) & (vn | better)
        best_v = np.where(take, v, best_v)
        best_i = np.where(take, i, best_i)
    return best_i
