"""Experiment: row-normalise total (C3) cooperative kernel variants timed
directly (CUDA events), checked bit-for-bit against the generated kernel.

Variant "rotate": the row group's register stage S1 is carried across
groups; pass 3 refills S1[m] with the NEXT group's chunk m as soon as the
last pass has consumed it, so the next group's loads are in flight during
this group's last pass and its cross-thread reductions (no extra registers).
usage: coop_probe.py [variant ...]"""
import os
import re
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1901_03771_b200 as gp  # noqa: E402
from paper_1901_03771_b200 import codegen, runtime, workloads as wl  # noqa: E402


BARRIER = False


def rotate(src: str) -> str:
    # rows(): S1 comes from the caller on the fast pass
    src = src.replace("const long long gnext) {", "const long long gnext, float (&S1x)[16][4]) {", 1)
    m = re.search(r"    float (S\d+)\[16\]\[4\];\n    #pragma unroll\n    for \(int mm = 0; mm < 16; \+\+mm\) "
                  r"gr::ldv<float, 4>\(\1\[mm\], (p\.in\d+) \+ r \* 4096LL \+ cb \+ 8 \* mm\);\n", src)
    assert m, "stage pattern"
    S, ptr = m.group(1), m.group(2)
    src = src.replace(m.group(0), f"    float (&{S})[16][4] = S1x;\n    if constexpr (!FAST) {{\n    #pragma unroll\n"
                                  f"    for (int mm = 0; mm < 16; ++mm) gr::ldv<float, 4>({S}[mm], {ptr} + r * 4096LL + cb + 8 * mm);\n    }}\n"
                                  f"    const long long rn = gnext * 4 + ri < NROWS ? gnext * 4 + ri : NROWS - 1;\n", 1)
    # the last pass over S: refill chunk i after its last use
    loops = [mm for mm in re.finditer(r"  #pragma unroll\n    for \(long long (i\d+) = 0; \1 < 16LL; \+\+\1\) \{\n", src)]
    last = None
    for lp in loops:
        body_start = lp.end()
        if f"{S}[{lp.group(1)}]" in src[body_start:body_start + 600]:
            last = lp
    assert last is not None
    iv = last.group(1)
    # find the end of that loop: the matching closing brace at 4 spaces
    close = src.index("\n    }\n", src.index("\n      }\n", last.end()))
    fence = 'asm volatile("" ::: "memory"); ' if BARRIER else ""
    ins = f"\n      if constexpr (FAST) {{ {fence}if (gnext < NG) gr::ldv<float, 4>({S}[{iv}], {ptr} + rn * 4096LL + cb + 8 * {iv}); }}"
    src = src[:close] + ins + src[close:]
    # kernel: carry the stage, preload the first group
    src = src.replace("  for (long long g = blockIdx.x; g < K::NG; g += gridDim.x) {\n    if (K::rows<true>(p, g * 4, nullptr, nullptr, 0))",
                      "  float S1c[16][4];\n  {\n    const int tr = threadIdx.x % 64, ri = threadIdx.x / 64;\n"
                      "    const long long r0 = blockIdx.x * 4 + ri < K::NROWS ? blockIdx.x * 4 + ri : K::NROWS - 1;\n"
                      "    const long long cb = (long long)(tr / 2) * 128 + (tr % 2) * 4;\n"
                      f"    if (blockIdx.x < K::NG)\n#pragma unroll\n    for (int mm = 0; mm < 16; ++mm) gr::ldv<float, 4>(S1c[mm], p.{ptr[2:]} + r0 * 4096LL + cb + 8 * mm);\n  }}\n"
                      "  for (long long g = blockIdx.x; g < K::NG; g += gridDim.x) {\n    if (K::rows<true>(p, g * 4, nullptr, nullptr, g + gridDim.x, S1c))", 1)
    src = src.replace("K::rows<false>(p, g * 4, nullptr, nullptr, K::NG);", "K::rows<false>(p, g * 4, nullptr, nullptr, K::NG, S1c);", 1)
    return src


def rotate_fenced(src):
    global BARRIER
    BARRIER = True
    try:
        return rotate(src)
    finally:
        BARRIER = False


def no_final_fold(src):
    """timing only: the last CTA's fold of the row partials skipped"""
    import re as _re
    return _re.sub(r"gr::block_tree<[^;]*;", "0.0f;", src)


VARIANTS = {"base": lambda s: s, "rotate": rotate, "rotate_fenced": rotate_fenced, "nofold": no_final_fold,
            "rotate_fenced_mb2": lambda s: rotate_fenced(s).replace("__launch_bounds__(256, 3)", "__launch_bounds__(256, 2)"),
            "rotate_mb2": lambda s: rotate(s).replace("__launch_bounds__(256, 3)", "__launch_bounds__(256, 2)"),
            "rotate_mb4": lambda s: rotate(s).replace("__launch_bounds__(256, 3)", "__launch_bounds__(256, 4)")}


def main():
    rt = runtime.get()
    (x,) = wl.named_inputs("rownorm")
    y, t = wl.rownorm(gp, gp.asarray(x))
    st = gp.default_session().plan([t.node])[0]
    ks = codegen.generate(codegen.canonicalize(codegen.Region(st.roots, st.leaves, st.nodes)))
    dx = rt.upload(x)
    out = rt.alloc(256)
    scratch = rt.alloc(ks.scratch_bytes)
    ticket = rt.alloc(256)
    rt.memset(ticket, 0)
    redo = rt.alloc(4 * ks.meta["redo_words"])
    rt.memset(redo, 0)
    ref = None
    for name in (sys.argv[1:] or list(VARIANTS)):
        src = VARIANTS[name](ks.source)
        if name == "rotate" and os.environ.get("DUMP"):
            open("gpurun_out/coop_rotate.cu", "w").write(src)
        k = rt.kernel(src, ks.name, ks.block, 0)
        grid = codegen.grid_for(ks, rt.sm_count, k.blocks_per_sm)
        params = runtime.pack_params([dx.ptr, out.ptr, scratch.ptr, ticket.ptr, redo.ptr])
        ms = []
        for i in range(15):
            e0, e1 = rt.event(), rt.event()
            rt.record(e0)
            rt.launch(k, grid, ks.block, params)
            rt.record(e1)
            rt.sync()
            if i >= 3:
                ms.append(rt.elapsed_ms(e0, e1))
        tot = out.to_numpy(gp.DType.f32, (1,))[0]
        if ref is None:
            ref = tot
        print(f"{name:12s} regs={k.num_regs} occ={k.blocks_per_sm} grid={grid} mean={np.mean(ms):.4f} ms "
              f"min={np.min(ms):.4f} frac={1073741824 / np.mean(ms) / 1e6 / 6549.8:.3f} total={tot!r} same={tot == ref}", flush=True)





FOLD_SRC = r'''
#include "gr_ops.cuh"
#include "gr_reduce.cuh"
extern "C" __global__ void __launch_bounds__(256) fold(const float* p, float* o, long long n) {
  const float v = gr::block_tree<gr::OpSum, float>(p, n, 0.0f);
  if (threadIdx.x == 0) o[0] = v;
}
'''


def fold_time():
    """One CTA's block_tree over 65536 partials (the coop kernel's final fold)."""
    rt = runtime.get()
    n = 65536
    x = rt.upload(np.random.default_rng(0).standard_normal(n).astype(np.float32))
    o = rt.alloc(256)
    k = rt.kernel(FOLD_SRC, "fold", 256, 0)
    ms = []
    for i in range(20):
        e0, e1 = rt.event(), rt.event()
        rt.record(e0)
        rt.launch(k, 1, 256, runtime.pack_params([x.ptr, o.ptr, n]))
        rt.record(e1)
        rt.sync()
        if i >= 3:
            ms.append(rt.elapsed_ms(e0, e1))
    print(f"block_tree over {n} f32 by one CTA: {np.mean(ms) * 1e3:.1f} us (min {np.min(ms) * 1e3:.1f})", flush=True)


if __name__ == "__main__":
    if sys.argv[1:] == ["fold"]:
        fold_time()
    else:
        main()
