"""Debug: streamed vs plain Black-Scholes (ptxas-contracted map bodies) —
first mismatching index, and whether the two runs used the same kernel
source / register build."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1901_03771_b200 as gp  # noqa: E402
from paper_1901_03771_b200 import runtime, streaming, workloads as wl  # noqa: E402

streaming.MIN_BYTES = 1
streaming.CHUNK_BYTES = 1 << 20
host = wl.blackscholes_inputs(n=(1 << 18) + 1000)
s = gp.Session()
outs = wl.blackscholes(gp, *[gp.asarray(h, session=s) for h in host])
gp.force(*outs)
plain = [np.asarray(o) for o in outs]
ks_plain = s.executor.last_steps[0].cache["ks"]
k_plain = s.executor.last_steps[0].cache["kernel"]
s2 = gp.Session()
gp.set_default_session(s2)
arrs = [gp.asarray(h) for h in host]
call, put = wl.blackscholes(gp, *arrs)
got = gp.materialize(call, put)
ks_str = s2.executor.last_steps[0].cache["ks"]
k_str = s2.executor.last_steps[0].cache["kernel"]
print("same source modulo NGROUPS:", ks_plain.source.split("NGROUPS")[1][30:] == ks_str.source.split("NGROUPS")[1][30:])
print("regs plain/stream:", k_plain.num_regs, k_str.num_regs, "occ:", k_plain.blocks_per_sm, k_str.blocks_per_sm)
for g, e in zip(got, plain):
    bad = np.nonzero(g != e)[0]
    print("mismatches:", bad.size, bad[:10], g[bad[:3]], e[bad[:3]])
    print("chunk rows:", [st for st in []])
print("launch log:", list(s2.executor.launch_log)[-3:])
os.makedirs("gpurun_out/r2x", exist_ok=True)
open("gpurun_out/r2x/plain.cu", "w").write(ks_plain.source)
open("gpurun_out/r2x/stream.cu", "w").write(ks_str.source)
