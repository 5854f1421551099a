"""Multi-rank correctness on one box: run under torchrun (any N); each rank
shards the same global k-means / row-normalise inputs along the leading axis
and the allreduced partials must equal NumPy's on the full arrays.
    GRUMPY_DEVICE=0 python -m torch.distributed.run --nproc-per-node 2 \
        --master-addr 127.0.0.1 --master-port 29555 tools/two_rank_check.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1901_03771_b200 as gp  # noqa: E402
import paper_1901_03771_b200.distributed as D  # noqa: E402
from paper_1901_03771_b200 import workloads as wl  # noqa: E402

comm = D.init(backend="nccl")
rank, world = comm.rank, comm.world
P, C = wl.kmeans_inputs(n=1 << 16, seed=3)
off, ln = D.split(P.shape[0], world, rank)
gP = D.local_input(P[off:off + ln], P.shape[0], off)
lab, sums, counts = wl.kmeans_partials(gp, gP, gp.asarray(C))
gp.force(lab, *sums, counts)
elab, esums, ecounts = wl.kmeans_partials(np, P, C)
assert np.array_equal(np.asarray(lab), elab[off:off + ln])
assert np.array_equal(np.asarray(counts), ecounts), (np.asarray(counts)[:5], ecounts[:5])
for s, e in zip(sums, esums):
    np.testing.assert_allclose(np.asarray(s), e, rtol=1e-12, atol=1e-9)
(x,) = wl.rownorm_inputs(rows=512, cols=256, seed=4)
off, ln = D.split(x.shape[0], world, rank)
y, tot = wl.rownorm(gp, D.local_input(x[off:off + ln], x.shape[0], off))
gp.force(y, tot)
ey, etot = wl.rownorm(np, x)
np.testing.assert_allclose(np.asarray(y), ey[off:off + ln], rtol=1e-5, atol=1e-5)
assert abs(float(np.asarray(tot)) - float(etot)) < 1e-2
# full-array and axis-0 arg-reductions over the sharded axis: device combine
# (allgather of (value, global index), arg-reduction over the rank axis)
z = np.random.default_rng(5).standard_normal((1000, 37))
z[700, 3] = z.max() + 1.0               # global max on the last rank
off, ln = D.split(z.shape[0], world, rank)
gz = D.local_input(z[off:off + ln], z.shape[0], off)
am, amin0 = gz.argmax(), gz.argmin(axis=0)
gp.force(am, amin0)
assert int(np.asarray(am)) == z.argmax(), (int(np.asarray(am)), z.argmax())
assert np.array_equal(np.asarray(amin0), z.argmin(axis=0))
zt = z.copy()
zt[10, :] = zt.max()                      # ties: the first (lowest-rank) index wins
zt[990, :] = zt.max()
gt = D.local_input(zt[off:off + ln], zt.shape[0], off)
assert np.array_equal(np.asarray(gt.argmax(axis=0)), zt.argmax(axis=0))
zn = z.copy()
zn[600, 5] = np.nan                       # NaN is the extreme value (np.argmax)
gn = D.local_input(zn[off:off + ln], zn.shape[0], off)
assert int(np.asarray(gn.argmax())) == zn.argmax()
print(f"rank {rank}/{world} ok ({type(comm).__name__})", flush=True)
