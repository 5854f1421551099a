"""Multi-process (gloo, world_size 2) tests of the leading-axis sharding logic.

The GPU executor cannot run here, so each rank evaluates its shard with the
eager oracle and combines partials with the same rules the executor applies
after its kernels (distributed.classify / combine_arg, allreduce of partials).
The result must equal NumPy on the unsharded arrays.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as td
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_sharded(outs, comm, offset_rows):
    """Evaluate roots on this rank like the sharded executor would."""
    import paper_1901_03771_b200.distributed as D
    from oracle import eager
    from paper_1901_03771_b200.dag import OpKind, ReduceOp

    nodes = [o.node for o in outs]
    dist = D.classify(nodes)
    cache = {}
    # partial nodes are materialised (evaluated + combined) before consumers
    order = sorted(dist, key=lambda i: i)
    by_id = {}
    stack = list(nodes)
    while stack:
        n = stack.pop()
        if n.id in by_id:
            continue
        by_id[n.id] = n
        stack.extend(n.preds)
    for nid in order:
        d = dist[nid]
        n = by_id[nid]
        if d.startswith("P:"):
            local = eager.evaluate(n, cache)
            cache[nid] = comm.allreduce_host(local, ReduceOp(d[2:])).astype(n.dtype.np)
        elif d.startswith("A:"):
            x = eager.evaluate(n.preds[0], cache)
            which, axis, _ = n.op.attrs
            li = eager.evaluate(n, cache)
            f = np.max if which == "max" else np.min
            lv = f(x, axis=axis)
            off = offset_rows * (int(np.prod(x.shape[1:])) if axis is None else 1)
            cache[nid] = D.combine_arg(which, li, lv, off, comm).astype(np.int64)
    return [eager.evaluate(n, cache) for n in nodes]


def _worker(rank, world, port, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    td.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1901_03771_b200 as gp
        import paper_1901_03771_b200.distributed as D
        from paper_1901_03771_b200 import workloads as wl

        sess = gp.Session()
        gp.set_default_session(sess)
        comm = D.init(backend="gloo", session=sess)
        assert comm.world == world and comm.rank == rank
        rng = np.random.default_rng(0)
        x = rng.standard_normal((37, 16))
        P, C = wl.kmeans_inputs(n=1000, k=8, d=4)
        off, ln = D.split(37, world, rank)
        gx = D.shard_rows(x)
        gP = D.shard_rows(P)
        gC = gp.asarray(C)
        checks = {}
        outs = [gx.sum(), gx.sum(0), gx.sum(1), gx.max(), gx.argmax(), gx.argmin(axis=0), gx.mean(),
                gx.std(axis=0)]
        got = _oracle_sharded(outs, comm, off)
        checks["sum"] = np.allclose(got[0], x.sum())
        checks["sum0"] = np.allclose(got[1], x.sum(0))
        checks["sum1_local"] = np.allclose(got[2], x.sum(1)[off:off + ln])
        checks["max"] = got[3] == x.max()
        checks["argmax"] = got[4] == x.argmax()
        checks["argmin0"] = np.array_equal(got[5], x.argmin(axis=0))
        checks["mean"] = np.allclose(got[6], x.mean())
        checks["std0"] = np.allclose(got[7], x.std(axis=0))
        poff, _ = D.split(P.shape[0], world, rank)
        lab, sums, counts = wl.kmeans_partials(gp, gP, gC)
        g2 = _oracle_sharded([counts] + sums, comm, poff)
        elab, esums, ecounts = wl.kmeans_partials(np, P, C)
        checks["kmeans_counts"] = np.array_equal(g2[0], ecounts)
        checks["kmeans_sums"] = all(np.allclose(a, b, rtol=1e-12) for a, b in zip(g2[1:], esums))
        results[rank] = checks
    finally:
        td.destroy_process_group()


def test_sharded_partials_two_ranks():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, port, results), nprocs=world, join=True)
    for r in range(world):
        assert all(results[r].values()), results[r]


def test_split_covers_rows():
    from paper_1901_03771_b200.distributed import split
    for n in (0, 1, 7, 37, 1 << 20):
        for w in (1, 2, 3, 8):
            parts = [split(n, w, r) for r in range(w)]
            assert sum(l for _, l in parts) == n
            assert all(parts[i][0] + parts[i][1] == parts[i + 1][0] for i in range(w - 1))


def test_classify_rules():
    import paper_1901_03771_b200 as gp
    import paper_1901_03771_b200.distributed as D
    from paper_1901_03771_b200.errors import ShapeMismatch

    sess = gp.Session()
    x = D.local_input(np.ones((8, 4)), 16, 0, session=sess)
    w = gp.asarray(np.ones((4, 3)), session=sess)
    cases = {
        "map": ((x * 2 + 1), "S"), "rowsum": (x.sum(1), "S"), "total": (x.sum(), "P:sum"),
        "colmax": (x.max(0), "P:max"), "matmul": (x @ w, "S"), "argmax": (x.argmax(), "A:max"),
        "gram": (x.T @ x, None),
    }
    for name, (arr, want) in cases.items():
        if want is None:
            with pytest.raises(ShapeMismatch):
                D.classify([arr.node])
        else:
            assert D.classify([arr.node])[arr.node.id] == want, name
