"""Debug aid: a long 1-D cumsum at size n, repeated r times (timeouts expose hangs)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1901_03771_b200 as gp  # noqa: E402

n = int(sys.argv[1])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
x = np.random.default_rng(1).standard_normal(n).astype(np.float32)
g = gp.asarray(x)
for i in range(reps):
    t0 = time.time()
    r = np.asarray(gp.cumsum(g * 0.5 + 1.0))
    print(n, i, "ok", round(time.time() - t0, 3), float(r[-1]), flush=True)
