import sys, time; sys.path.insert(0,'/root/repo')
import numpy as np, paper_1901_03771_b200 as gp
from paper_1901_03771_b200 import runtime
rt=runtime.get()
for dt, n in ((np.float32, 1<<28), (np.int32, 1<<28), (np.float64, 1<<27), (np.int64, 1<<27)):
    x = (np.random.default_rng(0).integers(-3, 4, n)).astype(dt)
    g = gp.asarray(x); g.node.data.device = rt.upload(x)
    s = gp.Session(); gp.set_default_session(s)
    g = gp.asarray(x); g.node.data.device = rt.upload(x)
    y = gp.cumsum(g); gp.force(y)
    ts=[]
    for i in range(5):
        e0,e1=rt.event(),rt.event(); rt.record(e0)
        y = gp.cumsum(g); gp.force(y)
        rt.record(e1); rt.sync(); ts.append(rt.elapsed_ms(e0,e1))
    out_it = np.dtype(np.asarray(y[:1]).dtype).itemsize
    ms=min(ts); gb=(n*x.itemsize + n*out_it)/ms/1e6
    print(dt.__name__, n, "->", np.asarray(y[:1]).dtype, f"{ms:.3f} ms {gb:.0f} GB/s", flush=True)
