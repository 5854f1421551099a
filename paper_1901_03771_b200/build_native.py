"""Build the native parts in-tree (they travel to the GPU box with the repo).

* ``libgrumpy_rt.so`` — the C-ABI shim (g++, CUDA headers, NVRTC + cuBLAS
  linked, libcuda/libnccl loaded at run time);
* ``kernels/aot_check.cubin`` — nvcc compile of every hand-written skeleton
  and device-function template instantiated on representative point programs
  for sm_100a, so template errors surface at build time rather than first use.
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
KDIR = os.path.join(CSRC, "kernels")
REPO = os.path.dirname(HERE)
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
LIB = os.path.join(HERE, "libgrumpy_rt.so")


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return r


def _stale(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def build_shim(force=False) -> str:
    src = os.path.join(CSRC, "grumpy_rt.cpp")
    hdr = os.path.join(REPO, "include", "grumpy_rt.h")
    if force or _stale(LIB, [src, hdr]):
        _run([
            "g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-Wall", "-Wno-unused-function",
            f"-I{CUDA}/include", src, "-o", LIB,
            f"-L{CUDA}/lib64", "-lnvrtc", "-lcublas", "-lcublasLt", "-ldl", f"-Wl,-rpath,{CUDA}/lib64",
        ])
    return LIB


def build_aot_check(force=False) -> str:
    """nvcc -gencode arch=compute_100a,code=sm_100a over the template check TU."""
    src = os.path.join(KDIR, "aot_check.cu")
    out = os.path.join(KDIR, "aot_check.cubin")
    deps = [src] + [os.path.join(KDIR, f) for f in os.listdir(KDIR) if f.endswith(".cuh")]
    if force or _stale(out, deps):
        _run([
            os.path.join(CUDA, "bin", "nvcc"), "-gencode", "arch=compute_100a,code=sm_100a",
            "-cubin", "-lineinfo", "-O3", "--fmad=false", "-std=c++17", "-Xptxas", "-v",
            f"-I{KDIR}", src, "-o", out,
        ])
    return out


def build_all(force=False):
    build_shim(force)
    build_aot_check(force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
    print("built", LIB)
