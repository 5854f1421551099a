"""Sharded execution through the real executor + NCCL communicator.

Only one GPU is available to the test harness, so the process group has one
rank; the code path (NCCL init from a gloo-broadcast unique id, partial roots,
in-stream ncclAllReduce, arg combine) is the one every rank runs at N > 1.
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def dsess():
    import torch.distributed as td
    import paper_1901_03771_b200 as gp
    import paper_1901_03771_b200.distributed as D
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_port()), RANK="0", WORLD_SIZE="1")
    sess = gp.Session()
    old = gp.set_default_session(sess)
    comm = D.init(backend="nccl", session=sess)
    assert comm is not None
    yield sess
    gp.set_default_session(old)
    td.destroy_process_group()


def test_sharded_reductions(dsess):
    import paper_1901_03771_b200.distributed as D
    rng = np.random.default_rng(11)
    x = rng.standard_normal((300, 64)).astype(np.float32)
    gx = D.shard_rows(x, session=dsess)
    c0 = dsess.stats.collectives
    assert np.asarray(gx.sum()) == x.sum()
    assert np.asarray(gx.argmax()) == x.argmax()
    assert np.array_equal(np.asarray(gx.argmin(axis=0)), x.argmin(axis=0))
    np.testing.assert_allclose(np.asarray(gx.mean(0)), x.mean(0), rtol=1e-6)
    np.testing.assert_allclose(np.asarray((gx * 2).sum(1)), (x * 2).sum(1), rtol=1e-6)
    assert dsess.stats.collectives > c0


def test_sharded_kmeans_partials(dsess):
    import paper_1901_03771_b200 as gp
    import paper_1901_03771_b200.distributed as D
    from paper_1901_03771_b200 import workloads as wl
    P, C = wl.kmeans_inputs(n=1 << 14, k=64, d=4)
    gP = D.shard_rows(P, session=dsess)
    lab, sums, counts = wl.kmeans_partials(gp, gP, gp.asarray(C, session=dsess))
    gp.force(*sums, counts)
    elab, esums, ecounts = wl.kmeans_partials(np, P, C)
    assert np.array_equal(np.asarray(counts), ecounts)
    for s, e in zip(sums, esums):
        np.testing.assert_allclose(np.asarray(s), e, rtol=1e-12, atol=1e-9)
    newC = wl.kmeans_centroids(sums, counts, C)
    np.testing.assert_allclose(newC, wl.kmeans_centroids(esums, ecounts, C), rtol=1e-6)


def test_two_ranks_one_gpu_partials():
    """Two torchrun ranks on the one GPU: shards of k-means and row-normalise
    inputs, partials combined through host memory (NCCL cannot pair two
    ranks on one device); every rank checks its results against NumPy."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, GRUMPY_DEVICE="0", PYTHONPATH=root)
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    p = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(_port()),
                        os.path.join(root, "tools", "two_rank_check.py")],
                       env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    assert p.stdout.count(" ok (HostStagedComm)") == 2, p.stdout


def test_sharded_plan_cache(dsess):
    """Repeated sharded forces of one structure reuse the cached plan (one
    classification + region pass) and stay exact on fresh data."""
    import paper_1901_03771_b200 as gp
    import paper_1901_03771_b200.distributed as D
    rng = np.random.default_rng(12)
    n0 = len(dsess._shard_cache)
    for it in range(3):
        x = rng.standard_normal((256, 64)).astype(np.float32)
        gx = D.shard_rows(x, session=dsess)
        y = (gx - gx.mean(1)[:, None])
        tot, am = y.sum(), gx.argmax()
        gp.force(tot, am)
        ey = x - x.mean(1)[:, None]
        assert np.asarray(tot) == ey.sum()
        assert np.asarray(am) == x.argmax()
    assert len(dsess._shard_cache) == n0 + 1


def test_two_ranks_two_gpus_nccl():
    """Two ranks on two distinct GPUs build a real NCCL communicator (never the
    host-staged fallback); skipped on a one-GPU box."""
    import subprocess
    import sys
    from paper_1901_03771_b200 import runtime
    if runtime.device_count() < 2:
        pytest.skip("needs two GPUs")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PYTHONPATH=root)
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT", "GRUMPY_DEVICE"):
        env.pop(k, None)
    p = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(_port()),
                        os.path.join(root, "tools", "two_rank_check.py")],
                       env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    assert p.stdout.count(" ok (NcclComm)") == 2, p.stdout
