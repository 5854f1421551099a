"""bench.py's multi-rank logic on CPU: shard arithmetic of the named shapes,
the shared `config` dict of both arms, and the full-size parity check of
allreduced results over a real gloo process group (world_size 2)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import bench  # noqa: E402


@pytest.mark.parametrize("name", sorted(bench.WORKLOADS))
@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_strong_shards_partition_the_named_shape(name, world):
    spans = [bench.rows_of(name, "strong", world, r) for r in range(world)]
    n = bench.global_rows(name)
    if bench.WORKLOADS[name].get("shardable", True):
        assert spans[0][1] == 0 and spans[-1][2] == n
        for (g0, lo0, hi0), (g1, lo1, hi1) in zip(spans, spans[1:]):
            assert g0 == g1 == n and hi0 == lo1
    else:
        assert all(s == (n, 0, n) for s in spans)     # replicas


def test_weak_shards_grow_the_shape():
    spans = [bench.rows_of("blackscholes-f32", "weak", 4, r) for r in range(4)]
    n = bench.global_rows("blackscholes-f32")
    assert spans == [(4 * n, r * n, (r + 1) * n) for r in range(4)]


def test_config_is_arm_independent():
    c1 = bench.config_of("blackscholes-f32", "strong", 8)
    assert c1 == bench.config_of("blackscholes-f32", "strong", 8)
    assert c1["elements"] == 1 << 28 and c1["parallelism"].startswith("shard8")
    assert bench.config_of("jacobi", "strong", 4)["parallelism"] == "replicas4"


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, q):
    import torch
    import torch.distributed as td
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    td.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import fullsize, programs
        wl = programs.load()

        def comm_sum(v):
            t = torch.from_numpy(np.array(v, dtype=np.float64, copy=True).reshape(-1))
            td.all_reduce(t)
            return t.numpy().reshape(np.shape(v))

        res = {}
        # row-normalise: each rank checks its rows; the total was allreduced
        rows = 256
        lo, hi = rank * rows // world, (rank + 1) * rows // world
        x_all = wl.named_inputs("rownorm", 0, rows)[0]
        y_all, t_all = wl.rownorm(np, x_all)
        total64 = float(np.sum(y_all.astype(np.float64)))
        r = fullsize.check("rownorm-y", [x_all[lo:hi]], [y_all[lo:hi], np.float32(total64)],
                           threads=2, comm_sum=comm_sum, world=world)
        res["rownorm"] = r["ok"]
        bad = fullsize.check("rownorm", [x_all[lo:hi]], [np.float32(total64 + 100.0)],
                             threads=2, comm_sum=comm_sum, world=world)
        res["rownorm_bad"] = bad["ok"]
        # k-means: labels per rank, sums/counts allreduced
        n = 1 << 14
        P, C = wl.named_inputs("kmeans", 0, n)
        lab, sums, counts = wl.kmeans_partials(np, P, C)
        lo, hi = rank * n // world, (rank + 1) * n // world
        r = fullsize.check("kmeans", [P[lo:hi], C], [lab[lo:hi], *sums, counts], threads=2,
                           comm_sum=comm_sum, world=world)
        res["kmeans"] = r["ok"]
        q.put((rank, res))
    finally:
        td.destroy_process_group()


def test_fullsize_parity_over_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in range(2):
        assert out[r]["rownorm"] and out[r]["kmeans"], out
        assert not out[r]["rownorm_bad"], out
