import sys, time; sys.path.insert(0, '/root/repo')
import numpy as np
t0=time.perf_counter()
import paper_1901_03771_b200 as gp
from paper_1901_03771_b200 import workloads as wl, runtime
rt = runtime.get(); print("runtime init", round(time.perf_counter()-t0,3), rt.gemm_math, flush=True)
X,W1,b1,W2,b2 = wl.mlp_inputs()
args=[gp.asarray(a) for a in (X,W1,b1,W2,b2)]
t=time.perf_counter(); p, lab = wl.mlp(gp, *args); gp.force(p, lab); rt.sync()
s=gp.default_session().stats
print("first step", round(time.perf_counter()-t,3), "plan", round(s.plan_time,3), "exec", round(s.exec_time,3), "compile_ms", round(s.compile_ms,1), flush=True)
t=time.perf_counter(); p, lab = wl.mlp(gp, *args); gp.force(p, lab); rt.sync(); print("second", round(time.perf_counter()-t,4))
