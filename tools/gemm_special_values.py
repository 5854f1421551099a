import sys; sys.path.insert(0,'/root/repo')
import numpy as np, paper_1901_03771_b200 as gp
from paper_1901_03771_b200 import runtime
rng=np.random.default_rng(0)
X=rng.random((64,32)).astype(np.float32); W=rng.random((32,16)).astype(np.float32)
X[3,5]=np.inf; X[7,1]=-np.inf; X[9,2]=3e38; X[10,:]=1e-40; X[11,0]=np.nan
for mode in ("bf16x9","fp32"):
    runtime.get().set_gemm_math(mode)
    s=gp.Session(); gp.set_default_session(s)
    got=np.asarray(gp.asarray(X)@gp.asarray(W))
    with np.errstate(all='ignore'): exp=X@W
    print(mode, "inf rows", got[3,:3], got[7,:3], "big", got[9,:2], exp[9,:2], "denorm", got[10,:2], exp[10,:2], "nan", got[11,:2])
    print("  mismatched nonfinite:", int(np.sum(np.isfinite(got)!=np.isfinite(exp))), "max rel finite", float(np.nanmax(np.abs(got-exp)[np.isfinite(exp)]/ (np.abs(exp)[np.isfinite(exp)]+1e-30))))
