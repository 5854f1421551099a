"""Experiment: time the long-scan kernel of bench.py's cumsum workload with
source prefixes (e.g. GR_SCAN_NOLB = no look-back, the streaming floor;
GR_SCAN_STATS = mean look-back distance).  usage: scan_probe.py [NAME:PREFIX]..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1901_03771_b200 as gp  # noqa: E402
from paper_1901_03771_b200 import codegen, runtime  # noqa: E402

n = int(os.environ.get("N", 1 << 28))
rt = runtime.get()
x = np.random.default_rng(1).standard_normal(n).astype(np.float32)
g = gp.asarray(x)
c = gp.cumsum(g * 0.5 + 1.0)
st = gp.default_session().plan([c.node])[0]
ks = codegen.generate(codegen.canonicalize(codegen.Region(st.roots, st.leaves, st.nodes)))
dx = rt.upload(x)
out = rt.alloc(n * 4)
scratch = rt.alloc(ks.scratch_bytes)
for spec in ["base:"] + sys.argv[1:]:
    name, _, pre = spec.partition(":")
    src = "".join(f"#define {d.replace('=', ' ', 1)}\n" for d in pre.split(",") if d) + ks.source
    if "REPL=" in pre:
        src = ks.source
        for pair in pre.split("REPL=", 1)[1].split("@@"):
            a, b = pair.split("=>")
            assert a in src, a
            src = src.replace(a, b)
    k = rt.kernel(src, ks.name, ks.block, ks.meta.get("smem", 0))
    grid = codegen.grid_for(ks, rt.sm_count, k.blocks_per_sm)
    ms = []
    for i in range(12):
        rt.memset(scratch, 0)
        e0, e1 = rt.event(), rt.event()
        rt.record(e0)
        rt.launch(k, grid, ks.block, runtime.pack_params([dx.ptr, out.ptr, scratch.ptr]), smem=ks.meta.get("smem", 0))
        rt.record(e1)
        rt.sync()
        if i >= 2:
            ms.append(rt.elapsed_ms(e0, e1))
    extra = ""
    if "GR_SCAN_STATS" in pre:
        addr, _ = rt.module_global(k, "_ZN2gr13gr_scan_statsE")
        buf = rt.alloc(64)
        rt.d2d_raw(buf.ptr, addr, 64)
        st_ = buf.to_numpy(gp.DType.i64, (8,))
        extra = (f" mean_distance={st_[0] / max(st_[1], 1):.1f} tiles (over {st_[1]} look-backs)"
                 f" lookback_cycles={st_[2] / max(st_[1], 1):.0f} lookback_idle_cycles={st_[3] / max(st_[1], 1):.0f}")
    r = out.to_numpy(gp.DType.f32, (n,))
    print(f"{name:10s} regs={k.num_regs} occ={k.blocks_per_sm} grid={grid} mean={np.mean(ms):.4f} ms min={np.min(ms):.4f}"
          f" last={float(r[-1]):.6g}{extra}", flush=True)
