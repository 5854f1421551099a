"""Benchmark CLI of the reference's bench module.

    python -m paper_1901_03771_b200.bench_cli run <name> --size N --iters K --seed S --json PATH
    python -m paper_1901_03771_b200.bench_cli dot --target dag|plan --out PATH [--name NAME --size N]

``run`` executes the eager NumPy program and the grumpy program on identical
inputs, verifies the outputs and writes a BenchReport:
per-engine cold and warm wall times, the speedup, ``kernels_executed``,
``library_calls`` and ``max_abs_err``; cold = first execution in the process
(plan + lower + NVRTC compile or disk-cache load + H2D + kernels + D2H), warm
= the same program re-run on fresh inputs of the same shape.
Exit code 0 on pass, 1 on verification failure (``VerificationFailed``).
``--inputs-npy DIR`` / ``--outputs-npy DIR`` write the tensors as npy v1.0
(SPEC.md:525).  ``dot`` writes the DAG or the plan of a recorded benchmark
program as DOT.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

from . import npyio
from . import workloads as wl
from .errors import VerificationFailed

SCHEMA_VERSION = 1
REPORT_KEYS = ("schema", "name", "size", "iters", "seed", "dtype", "engines", "speedup_warm", "speedup_cold",
               "kernels_executed", "library_calls", "max_abs_err", "tolerance", "status", "device")


def _bs(size, seed, dtype):
    ins = wl.blackscholes_inputs(size, seed, dtype)
    tol = (1e-12 if dtype == np.float64 else 1e-5) * max(100.0, 30.0)     # |Δ| ≤ tol·max(S,X)
    return ins, (lambda xp, *a: wl.blackscholes(xp, *a)), tol


def _jacobi(size, seed, dtype, sweeps):
    ins = wl.jacobi_inputs(size, seed, dtype)

    def prog(xp, a):
        for _ in range(sweeps):
            a = wl.jacobi(xp, a)
        return (a,)
    return ins, prog, (1e-12 if dtype == np.float64 else 1e-5)


def _inner(size, seed, dtype):
    rng = np.random.default_rng(seed)
    a = rng.random(size, dtype=np.float64).astype(dtype)
    b = rng.random(size, dtype=np.float64).astype(dtype)
    # a reassociated f32 sum of n products: |Δ| ≤ log2(n)·eps·Σ|tᵢ|
    eps = np.finfo(dtype).eps
    tol = float(np.log2(max(size, 2)) * eps * np.sum(np.abs(a.astype(np.float64) * b)))
    return (a, b), (lambda xp, a, b: ((a * b).sum(),)), tol


def _listing1(size, seed, dtype):
    return wl.listing1_inputs(size, seed, dtype), (lambda xp, *a: (wl.listing1(xp, *a),)), 0.0


def _rownorm(size, seed, dtype):
    ins = wl.rownorm_inputs(size, 4096, seed, dtype)
    n = ins[0].size
    tol = float(np.log2(n) * np.finfo(dtype).eps * n * 4)      # |y| ≲ 4 per element
    return ins, (lambda xp, x: wl.rownorm(xp, x)), tol


def _kmeans(size, seed, dtype, iters):
    P, C = wl.kmeans_inputs(size, 64, 4, seed)

    def prog(xp, P, C):
        # Lloyd iterations; labels are compared exactly, centroids by tolerance
        for _ in range(iters):
            lab, sums, counts = wl.kmeans_partials(xp, P, C)
            C = wl.kmeans_centroids(sums, counts, C)
            if xp is not np:
                C = xp.asarray(C)
        return lab, C
    return (P, C), prog, 1e-4


def _cumsum(size, seed, dtype):
    ins = wl.scan_inputs(size, seed, dtype)
    # a reassociated prefix sum, no less accurate than NumPy's own sequential
    # fold against the float64 prefix (within 2x, plus one ulp of the running
    # total): |got - numpy| <= 3 e_numpy + ulp — the tolerance is per input
    x = ins[0]
    exact = np.cumsum(x.astype(np.float64) * 0.5 + 1.0)
    ref = wl.scan(np, x)
    tol = 3 * float(np.max(np.abs(ref - exact))) + float(np.finfo(dtype).eps * abs(exact[-1]))
    return ins, (lambda xp, x: (wl.scan(xp, x),)), tol


BENCHES = {
    "blackscholes": lambda n, s, d, k: _bs(n, s, d),
    "jacobi": lambda n, s, d, k: _jacobi(n, s, d, k),
    "innerproduct": lambda n, s, d, k: _inner(n, s, d),
    "listing1": lambda n, s, d, k: _listing1(n, s, d),
    "rownorm": lambda n, s, d, k: _rownorm(n, s, d),
    "kmeans": lambda n, s, d, k: _kmeans(n, s, d, k),
    "cumsum": lambda n, s, d, k: _cumsum(n, s, d),
}
DEFAULT_DTYPE = {"blackscholes": "f64", "jacobi": "f64", "innerproduct": "f32", "listing1": "f64",
                 "rownorm": "f32", "kmeans": "f32", "cumsum": "f32"}


def _as_tuple(x):
    return tuple(x) if isinstance(x, (tuple, list)) else (x,)


def _run_grumpy(gp, prog, host):
    outs = _as_tuple(prog(gp, *[gp.asarray(h) for h in host]))
    lazy = [o for o in outs if isinstance(o, gp.ndarray)]
    if lazy:
        gp.force(*lazy)              # every root of the program in one plan
    return [np.asarray(o) for o in outs]


def run(name, size, iters=1, seed=42, dtype=None, inputs_npy=None, outputs_npy=None):
    """One BenchReport (a dict with REPORT_KEYS)."""
    import paper_1901_03771_b200 as gp
    if name not in BENCHES:
        raise ValueError(f"unknown benchmark {name!r}; choose from {sorted(BENCHES)}")
    dts = dtype or DEFAULT_DTYPE[name]
    dt = {"f32": np.float32, "f64": np.float64}[dts]
    host, prog, tol = BENCHES[name](size, seed, dt, iters)
    host2, _, _ = BENCHES[name](size, seed + 1, dt, iters)    # warm: fresh inputs, same shapes
    sess = gp.Session()
    old = gp.set_default_session(sess)
    try:
        t0 = time.perf_counter()
        got = _run_grumpy(gp, prog, host)
        cold = time.perf_counter() - t0
        before = sess.stats.snapshot()
        t0 = time.perf_counter()
        got2 = _run_grumpy(gp, prog, host2)
        warm = time.perf_counter() - t0
        kern = sess.stats.kernels_executed - before.kernels_executed
        lib = sess.stats.library_calls - before.library_calls
        compile_ms = sess.stats.compile_ms
    finally:
        gp.set_default_session(old)
    t0 = time.perf_counter()
    exp = [np.asarray(e) for e in _as_tuple(prog(np, *host))]
    np_cold = time.perf_counter() - t0
    t0 = time.perf_counter()
    exp2 = [np.asarray(e) for e in _as_tuple(prog(np, *host2))]
    np_warm = time.perf_counter() - t0
    err = 0.0
    ok = True
    for g, e in zip(got + got2, exp + exp2):
        if g.shape != e.shape:
            ok = False
            err = float("inf")
            continue
        if e.dtype.kind in "iub":
            same = bool(np.array_equal(g, e))
            ok &= same
            err = max(err, 0.0 if same else float(np.max(np.abs(g.astype(np.float64) - e.astype(np.float64)))))
        else:
            d = np.abs(g.astype(np.float64) - e.astype(np.float64))
            nan_ok = bool(np.array_equal(np.isnan(g), np.isnan(e)))
            m = float(np.nanmax(d)) if d.size and not np.all(np.isnan(d)) else 0.0
            err = max(err, m)
            ok &= nan_ok and m <= tol
    if inputs_npy:
        os.makedirs(inputs_npy, exist_ok=True)
        for i, h in enumerate(host):
            npyio.save(os.path.join(inputs_npy, f"{name}_in{i}.npy"), h)
    if outputs_npy:
        os.makedirs(outputs_npy, exist_ok=True)
        for i, g in enumerate(got):
            npyio.save(os.path.join(outputs_npy, f"{name}_out{i}.npy"), g)
    from . import runtime
    return {
        "schema": SCHEMA_VERSION, "name": name, "size": size, "iters": iters, "seed": seed, "dtype": dts,
        "engines": {"numpy_eager": {"cold_s": np_cold, "warm_s": np_warm},
                    "grumpy_b200": {"cold_s": cold, "warm_s": warm, "compile_ms": compile_ms}},
        "speedup_warm": np_warm / warm if warm > 0 else None,
        "speedup_cold": np_cold / cold if cold > 0 else None,
        "kernels_executed": kern, "library_calls": lib,
        "max_abs_err": err, "tolerance": tol, "status": "PASSED" if ok else "FAILED",
        "device": runtime.get().name,
    }


def _dot(args):
    import paper_1901_03771_b200 as gp
    sess = gp.Session()
    old = gp.set_default_session(sess)
    try:
        if args.name:
            dt = {"f32": np.float32, "f64": np.float64}[args.dtype or DEFAULT_DTYPE[args.name]]
            host, prog, _ = BENCHES[args.name](args.size, args.seed, dt, 1)
            outs = _as_tuple(prog(gp, *[gp.asarray(h) for h in host]))
            roots = [o for o in outs if isinstance(o, gp.ndarray)]
        else:
            roots = []
        npyio.dump_dot(args.target, args.out, roots=roots if args.target == "plan" else None, session=sess)
    finally:
        gp.set_default_session(old)
    return 0


def main(argv=None):
    ap = argparse.ArgumentParser(prog="bench")
    sub = ap.add_subparsers(dest="cmd", required=True)
    r = sub.add_parser("run")
    r.add_argument("name")
    r.add_argument("--size", type=int, required=True)
    r.add_argument("--iters", type=int, default=1)
    r.add_argument("--threads", type=int, default=None, help="accepted for CLI compatibility (one GPU)")
    r.add_argument("--seed", type=int, default=42)
    r.add_argument("--dtype", choices=("f32", "f64"), default=None)
    r.add_argument("--json", default=None)
    r.add_argument("--inputs-npy", default=None)
    r.add_argument("--outputs-npy", default=None)
    d = sub.add_parser("dot")
    d.add_argument("--target", choices=("dag", "plan"), required=True)
    d.add_argument("--out", required=True)
    d.add_argument("--name", default=None, choices=sorted(BENCHES))
    d.add_argument("--size", type=int, default=1024)
    d.add_argument("--seed", type=int, default=42)
    d.add_argument("--dtype", choices=("f32", "f64"), default=None)
    args = ap.parse_args(argv)
    if args.cmd == "dot":
        return _dot(args)
    rep = run(args.name, args.size, args.iters, args.seed, args.dtype, args.inputs_npy, args.outputs_npy)
    text = json.dumps(rep)
    if args.json:
        with open(args.json, "w") as f:
            f.write(text + "\n")
    print(text)
    if rep["status"] != "PASSED":
        err = VerificationFailed(f"{args.name}: max_abs_err {rep['max_abs_err']:.3g} > tolerance {rep['tolerance']:.3g}")
        print(f"bench: {err}", file=sys.stderr)
        return 1
    return 0


if __name__ == "__main__":
    sys.exit(main())
