"""Cold-start cost of a multi-step plan with and without JIT/execute
pipelining (GRUMPY_PRECOMPILE), each in a fresh process with an empty cubin
cache.  usage: python tools/jit_pipeline_probe.py"""
import json
import os
import subprocess
import sys
import tempfile

PROG = r'''
import json, time, numpy as np, sys
sys.path.insert(0, %r)
import paper_1901_03771_b200 as gp
import paper_1901_03771_b200.runtime
rng = np.random.default_rng(0)
x = rng.standard_normal((4096, 512)).astype(np.float32)
gp.runtime.get()                        # CUDA context + NVRTC loaded outside the timed region
gp.asarray(np.ones(4, np.float32)).sum().item()
t0 = time.perf_counter()
g = gp.asarray(x)
c = g.sum(axis=0)                       # column sums: a step of its own
m = (g - c / 4096.0)                    # broadcast of a reduction over the reduced axis: cut
s = gp.cumsum(m.ravel() * 0.5)          # long scan
r = (m * m).sum(axis=1)                 # row reduction
a = m.argmax(axis=1)
gp.force(s, r, a)
cold = time.perf_counter() - t0
st = gp.default_session().stats   # (includes the warm-up kernel)
print(json.dumps({"cold_s": cold, "kernels": st.kernels_executed, "compile_ms": st.compile_ms,
                  "ok": bool(np.allclose(np.asarray(r), ((x - x.sum(0) / 4096.0) ** 2).sum(1), rtol=1e-4))}))
'''


def main():
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for pre in ("0", "1", "0", "1"):
        with tempfile.TemporaryDirectory() as d:
            env = dict(os.environ, GRUMPY_CACHE_DIR=d, GRUMPY_PRECOMPILE=pre)
            out = subprocess.run([sys.executable, "-c", PROG % root], env=env, capture_output=True, text=True,
                                 timeout=600)
            line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-500:]
            print(f"precompile={pre}", line, flush=True)


if __name__ == "__main__":
    main()
