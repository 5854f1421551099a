import sys
import os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1901_03771_b200 as gp
from paper_1901_03771_b200 import workloads as wl, codegen
def dump(roots, which=None):
    sess = gp.session.default_session()
    steps = sess.plan([r.node for r in roots])
    for i, st in enumerate(steps):
        if st.kind != "Fused":
            print("//", st.kind, getattr(st, "call", None)); continue
        region = codegen.canonicalize(codegen.Region(st.roots, st.leaves, st.nodes))
        ks = codegen.generate(region)
        print("// step", i, ks.family, ks.name, ks.block, ks.meta.keys())
        if which is None or i == which:
            print(ks.source)
if __name__ == "__main__":
    w = sys.argv[1]
    if w == "kmeans":
        P, C = wl.kmeans_inputs(n=1<<14)
        lab, sums, counts = wl.kmeans_partials(gp, gp.asarray(P), gp.asarray(C))
        dump([lab] + sums + [counts])
    elif w == "rownorm":
        (x,) = wl.rownorm_inputs(rows=1024)
        y, t = wl.rownorm(gp, gp.asarray(x)); dump([t])
    elif w == "rownorm-y":
        (x,) = wl.rownorm_inputs(rows=1024)
        y, t = wl.rownorm(gp, gp.asarray(x)); dump([y, t])
    elif w == "bs":
        S, X, T = wl.blackscholes_inputs(n=1<<20)
        c, p = wl.blackscholes(gp, *map(gp.asarray, (S, X, T))); dump([c, p])
    elif w == "bs64":
        S, X, T = wl.blackscholes_inputs(n=1<<20, dtype=np.float64)
        c, p = wl.blackscholes(gp, *map(gp.asarray, (S, X, T))); dump([c, p])
    elif w == "cumsum":
        (x,) = wl.scan_inputs(n=1<<24)
        dump([wl.scan(gp, gp.asarray(x))])


def sass_mix(source, name="gr_region"):
    """Compile one generated source with NVRTC (sm_100a) and return the SASS
    opcode histogram of ``name`` (cuobjdump)."""
    import collections, subprocess, tempfile
    from paper_1901_03771_b200 import runtime
    cub = runtime.compile_cubin(source)
    with tempfile.NamedTemporaryFile(suffix=".cubin") as f:
        f.write(cub)
        f.flush()
        out = subprocess.run(["cuobjdump", "-sass", "-fun", name, f.name], capture_output=True, text=True).stdout
    ops = collections.Counter()
    for line in out.splitlines():
        line = line.strip()
        if line.startswith("/*") and "*/" in line:
            ins = line.split("*/", 1)[1].strip().split()
            if ins and not ins[0].startswith("/*"):
                op = ins[0] if not ins[0].startswith("@") else ins[1]
                ops[op.split(".")[0]] += 1
    return ops
