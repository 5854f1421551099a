"""Time source-level variants of one workload's dominant fused kernel.

usage: python tools/variant_bench.py WORKLOAD VARIANT... ; VARIANT is
"name:prefix" where prefix (e.g. "#define GR_PAIR_MUL 1") is prepended to the
generated source, or "name:U=2" to change the map unroll.  Prints mean kernel
ms over 20 launches (CUDA events) per variant.  Experiments only.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_1901_03771_b200 as gp  # noqa: E402
from paper_1901_03771_b200 import codegen, runtime  # noqa: E402


def main():
    wname = sys.argv[1]
    rt = runtime.get()
    w = bench.WORKLOADS[wname]
    host = bench.make_inputs(wname, w["n"], 42)
    sess = gp.Session()
    gp.set_default_session(sess)
    dev = [gp.asarray(x) for x in host]
    for d in dev:
        d.node.data.device = rt.upload(d.node.data.host)
    outs = bench.make_program(wname)(gp, dev)
    gp.force(*outs)
    steps = sess.executor.last_steps
    st = max((s for s in steps if s.kind == "Fused"), key=lambda s: sum(r.size for r in s.roots))
    ks0 = st.cache["ks"]
    for spec in ["base:"] + sys.argv[2:]:
        name, _, pre = spec.partition(":")
        src = ks0.source
        block, grid_over, smem, tmap = ks0.block, None, ks0.meta.get("smem", 0), False
        if ";" in pre and not pre.startswith("REPL="):
            pre, *opts = pre.split(";")
            for o in opts:
                kk, vv = o.split("=")
                if kk == "BLOCK":
                    block = int(vv)
                elif kk == "GRID":
                    grid_over = int(vv)
                elif kk == "SMEM":
                    smem = int(vv)
                elif kk == "TMAP":
                    tmap = True
        if pre.startswith("FILE="):
            src = open(pre[5:]).read()
        elif pre.startswith("REPL="):
            # REPL=old=>new[@@old2=>new2...]: literal source substitutions
            for pair in pre[5:].split("@@"):
                a, b = pair.split("=>")
                assert a in src, a
                src = src.replace(a, b)
        elif pre.startswith("U="):
            src = src.replace("static constexpr int U = 1;", f"static constexpr int U = {pre[2:]};")
            src = src.replace("static constexpr int U = 2;", f"static constexpr int U = {pre[2:]};")
        elif pre.startswith("LB="):
            src = src.replace(f"__launch_bounds__({ks0.block})", f"__launch_bounds__({ks0.block}, {pre[3:]})")
            src = src.replace(f"__launch_bounds__({ks0.block}, 3)", f"__launch_bounds__({ks0.block}, {pre[3:]})")
        elif pre:
            src = pre.replace("\\n", "\n") + "\n" + src
        k = rt.kernel(src, ks0.name, block, smem)
        grid = grid_over or codegen.grid_for(ks0, rt.sm_count, k.blocks_per_sm) * ks0.block // block
        leaves = [st.leaves[i] for i in st.cache["perm"]]
        bufs = [sess.executor.new_buffer(r) for r in st.roots]
        ptrs = [sess.executor.device_ptr(l) for l in leaves] + [b.device.ptr for b in bufs]
        scratch = rt.alloc(max(ks0.scratch_bytes, 256))
        ptrs.append(scratch.ptr)
        if ks0.meta.get("ticket"):
            tk = rt.alloc(256)
            rt.memset(tk, 0)
            ptrs.append(tk.ptr)
        if "REDO" in spec or ks0.meta.get("redo_words"):
            if not ks0.meta.get("ticket"):
                ptrs.append(0)
            rd = rt.alloc(1 << 16)
            rt.memset(rd, 0)
            ptrs.append(rd.ptr)
        for i, sym, nb in ks0.meta.get("cbank") or ():
            rt.d2d_raw(rt.module_global(k, sym)[0], ptrs[i], nb)
        for i, psym, _b, _np, rname in ks0.meta.get("cbank_pair") or ():
            rt.launch(rt.function(k, rname), 1, 256, runtime.pack_params([ptrs[i], rt.module_global(k, psym)[0]]))
        params = runtime.pack_params(ptrs)
        if tmap:
            # leaf 0 as [n/32][32] f32 lines, box 128 lines (one 4096-float row), 128B swizzle
            l0 = leaves[0]
            nel = int(np.prod(l0.shape))
            params = params + bytes(64 - len(params) % 64) if len(params) % 64 else params
            params += rt.tensor_map_2d(ptrs[0], l0.dtype, 32, nel // 32, 128, 32, 128, 128)
        ts = []
        for i in range(25):
            e0, e1 = rt.event(), rt.event()
            rt.record(e0)
            rt.launch(k, grid, block, params, smem=smem)
            rt.record(e1)
            ts.append((e0, e1))
        ms = [rt.elapsed_ms(a, b) for a, b in ts[5:]]
        if len(bufs) == 1 and bufs[0].shape == ():
            print("   result", bufs[0].device.to_numpy(bufs[0].dtype, ()))
        print(f"{wname} {name:12s} regs={k.num_regs:3d} occ={k.blocks_per_sm} grid={grid} mean={np.mean(ms):.4f} ms min={np.min(ms):.4f}", flush=True)


if __name__ == "__main__":
    main()
