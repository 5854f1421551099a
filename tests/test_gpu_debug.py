"""Debug-run switches on the GPU, each in its own process (they are read at
import): GRUMPY_DEBUG_BOUNDS=1 bounds-checks every leaf read of the generated
kernels and GRUMPY_NVTX=1 wraps every plan step in an NVTX
range.  The config programs run under them with NumPy's results."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

PROGRAM = r'''
import numpy as np
import paper_1901_03771_b200 as gp
from paper_1901_03771_b200 import workloads as wl
S, X, T = wl.blackscholes_inputs(n=(1 << 16) + 3)
c, p = wl.blackscholes(gp, *map(gp.asarray, (S, X, T)))
ce, pe = wl.blackscholes(np, S, X, T)
assert np.allclose(np.asarray(c), ce, atol=1e-3) and np.allclose(np.asarray(p), pe, atol=1e-3)
(x,) = wl.rownorm_inputs(rows=256, cols=4096)
y, t = wl.rownorm(gp, gp.asarray(x))
ye, te = wl.rownorm(np, x)
assert np.array_equal(np.asarray(y), ye) and float(np.asarray(t)) == float(te)
P, C = wl.kmeans_inputs(n=1 << 14)
lab = np.asarray(((gp.asarray(P)[:, None, :] - gp.asarray(C)[None]) ** 2).sum(-1).argmin(1))
assert np.array_equal(lab, ((P[:, None, :] - C[None]) ** 2).sum(-1).argmin(1))
a = np.random.default_rng(1).random((300, 257), dtype=np.float32)
g = gp.asarray(a)
assert np.array_equal(np.asarray(g.T + g.T * 2), a.T + a.T * np.float32(2))
assert np.array_equal(np.asarray(g[1:, :] - g[:-1, :]), a[1:] - a[:-1])
assert np.array_equal(np.asarray(gp.cumsum(g * 2, axis=1)), np.cumsum(a * np.float32(2), axis=1))
v = np.random.default_rng(2).standard_normal((1 << 20) + 7).astype(np.float32)
got = np.asarray(gp.cumsum(gp.asarray(v) * 0.5))
assert np.allclose(got, np.cumsum((v * np.float32(0.5)).astype(np.float64)), atol=1e-2, rtol=1e-4)
print("debug ok")
'''


@pytest.mark.parametrize("flag", ["GRUMPY_DEBUG_BOUNDS", "GRUMPY_NVTX"])
def test_debug_switch_runs_config_programs(flag):
    env = dict(os.environ, **{flag: "1"})
    r = subprocess.run([sys.executable, "-c", PROGRAM], cwd=REPO, env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "debug ok" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]
