#!/usr/bin/env python
"""Benchmark of the fused-region path (BASELINE.json metric) — one JSON line.

Default workload = BASELINE.json configs[1], Black-Scholes on 2^28 options in
fp32 (the headline config; it fits one B200).  A "step" is one pass of the hot
path over one batch: record the pricing expression on device-resident inputs
and force call+put, which runs as ONE fused kernel.

  value     elements/s of the whole job with inputs resident in HBM, CUDA-event
            timed on the runtime stream, K steps bracketed by barrier + sync,
            max over ranks
  parity    the last timed step's outputs checked against the NumPy program
            at the full size (oracle/fullsize.py); a violation prints the line
            and exits 1 (the reference bench's VerificationFailed)
  e2e       the same through the public API from pinned host buffers:
            H2D of the inputs + kernels + D2H of every output each step
            (``e2e_pageable``: the same from ordinary NumPy arrays)
  roofline  algorithmic bytes per launch / mean kernel time (CUDA events)
            against MEASURED_PEAKS.json hbm_gbs
  cpu_baseline  the eager NumPy program (the paper's baseline) on a bounded
            sample, single thread, rank 0 at N=1

Multi-GPU: one process per GPU.  ``--gpus N`` without a
torchrun environment re-launches itself under torch.distributed.run.  The
default is strong scaling of the NAMED shape: rank r owns rows
[lo_r, hi_r) of the 2^28-option / 65536-row / 2^26-point problem; regions with
reduction partials (row-normalise total, k-means sums/counts) allreduce them
over NCCL on the runtime stream.  Kernel and collective time are reported
separately.

``--impl reference`` times the reference CPU path instead: the same NumPy
program (eager evaluation) over a blocked partition of the same
full named shape on all host cores, rank 0 only; it never
imports the product package (oracle/programs.py loads the program file by
path), so libgrumpy_rt.so is not mapped into that process.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

BASE = json.load(open(os.path.join(REPO, "BASELINE.json")))
METRIC = BASE["metric"]


# ---------------------------------------------------------------------------
# distributed plumbing (timing, parity sums)
# ---------------------------------------------------------------------------
class Dist:
    def __init__(self, gloo: bool = True):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local_rank = int(os.environ.get("LOCAL_RANK", "0"))
        self.td = None
        if self.world > 1 and gloo:
            import torch.distributed as td
            td.init_process_group("gloo")
            self.td = td

    def barrier(self):
        if self.td is not None:
            self.td.barrier()

    def _reduce(self, vec, op):
        v = np.asarray(vec, dtype=np.float64)
        if self.td is None:
            return v
        import torch
        t = torch.from_numpy(np.array(v, copy=True).reshape(-1))
        self.td.all_reduce(t, op=op)
        return t.numpy().reshape(v.shape)

    def max(self, x: float) -> float:
        if self.td is None:
            return x
        return float(self._reduce([x], self.td.ReduceOp.MAX)[0])

    def sum_f64(self, vec):
        if self.td is None:
            return np.asarray(vec, dtype=np.float64)
        return self._reduce(vec, self.td.ReduceOp.SUM)

    def all_ok(self, ok: bool) -> bool:
        if self.td is None:
            return ok
        return float(self._reduce([0.0 if ok else 1.0], self.td.ReduceOp.MAX)[0]) == 0.0

    def close(self):
        if self.td is not None:
            self.td.destroy_process_group()


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------
class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def wait_first(self, timeout):
        t0 = time.time()
        while self.proc is not None and not self.lines and time.time() - t0 < timeout:
            time.sleep(0.02)

    def mark(self):
        self.mark_at = len(self.lines)

    def since_mark(self):
        return len(self.lines) - getattr(self, "mark_at", 0) if self.proc is not None else 99

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines[getattr(self, "mark_at", 0):]:
            parts = [p.strip() for p in l.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def bf16_peak():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        return float(json.load(open(p))["bf16_tflops"])
    return 2250.0


def peaks():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


# ---------------------------------------------------------------------------
# workloads
# ---------------------------------------------------------------------------
def _programs():
    """The NumPy-over-xp config programs without importing the product package
    (oracle/programs.py loads paper_1901_03771_b200/workloads.py by path)."""
    from oracle import programs
    return programs.load()


MLP_H = 1024   # hidden width (unpinned by BASELINE.json; SURVEY.md §8(d) C4 recommends 1024)
KM_D = 4       # k-means dimensionality (SURVEY.md §8(d) C5 recommends 4)

# elements(rows): iteration-space points for `rows` leading rows;
# bytes(rows): algorithmic HBM bytes of the dominant fused kernel per launch
# (inputs read once, outputs written once).  collective: the region has
# reduction partials over the sharded axis (allreduced over NCCL at N > 1).
WORKLOADS = {
    "blackscholes-f32": dict(
        label="f32", shape="[2^28] options",
        desc="Black-Scholes call+put, 2^28 options, fp32 (BASELINE configs[1]); put = X e (1-N(d2)) - S (1-N(d1)): "
             "2 erf per option",
        program=lambda xp, a: _programs().blackscholes(xp, *a),
        elements=lambda n: n, bytes=lambda n: 5 * 4 * n, bound="hbm"),
    "blackscholes-f64": dict(
        label="f64", shape="[2^28] options",
        desc="Black-Scholes call+put, 2^28 options, fp64 (BASELINE configs[1]); 2 erf per option",
        program=lambda xp, a: _programs().blackscholes(xp, *a),
        elements=lambda n: n, bytes=lambda n: 5 * 8 * n, bound="hbm (fp64 pipe limits)",
        compute=dict(pipe="fp64", ops=171, lanes_per_sm_clk=64,
                     note="DFMA+DMUL+DADD per option of the libdevice exp/log/erf/div/sqrt code (ncu dynamic count)")),
    "listing1": dict(
        label="f64", shape="[2^24]",
        desc="paper Listing 1 chain (4 mul + 2 add), 2^24 fp64 (BASELINE configs[0])",
        program=lambda xp, a: (_programs().listing1(xp, *a),),
        elements=lambda n: n, bytes=lambda n: 4 * 8 * n, bound="hbm"),
    "rownorm": dict(
        label="f32", shape="[65536, 4096]",
        desc="row-normalise 65536x4096 fp32 then sum; total forced (BASELINE configs[2])",
        program=lambda xp, a: (_programs().rownorm(xp, *a)[1],),
        elements=lambda n: n * 4096, bytes=lambda n: n * 4096 * 4 + 4, bound="hbm", collective=True),
    "rownorm-y": dict(
        label="f32", shape="[65536, 4096]",
        desc="row-normalise 65536x4096 fp32, y and total forced",
        program=lambda xp, a: _programs().rownorm(xp, *a),
        elements=lambda n: n * 4096, bytes=lambda n: 2 * n * 4096 * 4 + 4, bound="hbm", collective=True),
    "mlp": dict(
        label="f32", shape=f"batch 65536, 784-{MLP_H}-10",
        desc=f"MNIST-style MLP inference batch 65536, 784-{MLP_H}-10, cuBLAS GEMMs + fused epilogues (BASELINE configs[3])",
        program=lambda xp, a: _programs().mlp(xp, *a),
        elements=lambda n: n * (MLP_H + 10), bytes=lambda n: 2 * n * MLP_H * 4 + MLP_H * 4,
        # the dominant launch is layer 1 as one cuBLASLt call: X@W1 in FP32
        # emulated with BF16x9 tensor-core products + the bias/ReLU epilogue
        # (the R1 region absorbed)
        library_flops={"Gemm+relu_bias": lambda n: 2.0 * n * 784 * MLP_H, "Gemm": lambda n: 2.0 * n * 784 * MLP_H},
        # the repo's own kernels of the step (HBM rooflines): layer 2 + b2 +
        # softmax + argmax as the skinny-product row kernel, and the R1
        # bias+ReLU map when the cuBLASLt epilogue is off (GRUMPY_GEMM_EPILOGUE=0)
        repo_bytes={"rows:gr_region": lambda n: n * MLP_H * 4 + n * 10 * 4 + n * 8 + MLP_H * 10 * 4 + 40,
                    "map:gr_region": lambda n: 2 * n * MLP_H * 4 + MLP_H * 4},
        bound="tensor (cuBLASLt BF16x9-emulated FP32 GEMM + fused bias/ReLU epilogue)"),
    "kmeans": dict(
        label="f32", shape=f"[2^26, {KM_D}] points x 64 centroids",
        desc=f"k-means assignment, 2^26 points x 64 centroids, D={KM_D} (BASELINE configs[4])",
        program=lambda xp, a: _km_step(xp, a),
        elements=lambda n: n, bytes=lambda n: n * (KM_D * 4 + 8) + 64 * KM_D * 4,
        bound="issue (certified nearest-centre search: FFMA2 keys + FMNMX top-2, NumPy-order scan for uncertified rows)",
        # per point, the program as NumPy states it: 64 centroids x (D sub +
        # D square + (D-1) add + 1 compare of the argmin) — algorithmic
        # lane-ops; the kernel's expanded-key search executes fewer
        compute=dict(pipe="fp32", ops=64 * (3 * KM_D), lanes_per_sm_clk=128,
                     note="algorithmic: 64 x (4 sub + 4 mul + 3 add + 1 argmin compare) lane-ops per point "
                          "(the NumPy formulation; the certified key search executes 64 x ~2.5 FP32-pipe "
                          "instructions + ~3.5 ALU instructions per point)"),
        collective=True),
    "cumsum": dict(
        label="f32", shape="[2^28]",
        desc="map-scan cumsum(x*0.5+1) over 2^28 fp32 (SURVEY.md §8(f))",
        program=lambda xp, a: (_programs().scan(xp, *a),),
        elements=lambda n: n, bytes=lambda n: 2 * 4 * n, bound="hbm", shardable=False),
    "cumsum-rows": dict(
        label="f32", shape="[65536, 4096]",
        desc="map-scan cumsum(x*0.5+1, axis=1) over 65536x4096 fp32 rows (SURVEY.md §8(f), scan along the contiguous axis)",
        program=lambda xp, a: (_programs().scan_rows(xp, *a),),
        elements=lambda n: n * 4096, bytes=lambda n: 2 * 4 * n * 4096, bound="hbm"),
    "transpose": dict(
        label="f32", shape="[16384, 16384]",
        desc="x.T + y, 16384x16384 fp32: transposed leaf staged through shared-memory tiles (north_star K1 staging)",
        program=lambda xp, a: (_programs().transpose_add(xp, *a),),
        elements=lambda n: n * 16384, bytes=lambda n: 3 * 4 * n * 16384, bound="hbm", shardable=False),
    "jacobi": dict(
        label="f32", shape="[16384, 16384]",
        desc="5-point Jacobi sweep (slice-assign), 16384x16384 fp32 (SURVEY.md §8(f))",
        program=lambda xp, a: (_programs().jacobi(xp, *a),),
        elements=lambda n: n * 16384, bytes=lambda n: 2 * 4 * n * 16384, bound="hbm", shardable=False),
}


def _km_step(xp, a):
    """k-means step on this shard: labels + per-cluster fp64 partial sums and
    counts (one fused kernel); sharded runs allreduce sums/counts over NCCL."""
    lab, sums, counts = _programs().kmeans_partials(xp, *a)
    return (lab, *sums, counts)


def global_rows(name):
    return _programs().NAMED[name][0]


def split(n, world, rank):
    base, rem = divmod(n, world)
    off = rank * base + min(rank, rem)
    return off, off + base + (1 if rank < rem else 0)


def rows_of(name, scaling, world, rank):
    """[lo, hi) of the named shape owned by ``rank`` (global extent, lo, hi)."""
    n = global_rows(name)
    if not WORKLOADS[name].get("shardable", True):
        return n, 0, n                      # replicas: every rank runs the whole shape
    if scaling == "weak":
        return n * world, rank * n, (rank + 1) * n
    lo, hi = split(n, world, rank)
    return n, lo, hi


def config_of(name, scaling, world):
    """The `config` dict, identical for the GPU arm and the reference arm."""
    w = WORKLOADS[name]
    n = global_rows(name)
    shard = w.get("shardable", True)
    total = n * world if (scaling == "weak" and shard) else n
    return {"workload": w["desc"], "shape": w["shape"], "leading_rows": total,
            "elements": w["elements"](total),
            "parallelism": (f"shard{world} (leading axis, {scaling} scaling)" if shard else f"replicas{world}"),
            "l2": "inputs larger than the 126 MB L2 (no flush): the dominant kernel streams %.2f GiB per launch"
                  % (w["bytes"](total // (world if shard and scaling == 'strong' else 1)) / 2 ** 30)}


def host_inputs(name, lo, hi):
    return _programs().named_inputs(name, lo, hi)


def cpu_sample_n(name):
    """Leading extent of the bounded single-thread CPU sample (~5-20 s)."""
    return {"blackscholes-f32": 1 << 24, "blackscholes-f64": 1 << 24, "listing1": 1 << 24,
            "rownorm": 16384, "rownorm-y": 16384, "mlp": 16384, "kmeans": 1 << 20, "jacobi": 4096, "transpose": 4096,
            "cumsum": 1 << 24, "cumsum-rows": 4096}[name]


# ---------------------------------------------------------------------------
# CPU reference path: the NumPy program over a blocked partition
# ---------------------------------------------------------------------------
class BlockedNumpy:
    """One step = the NumPy program over the whole input, evaluated on row
    blocks by a thread pool (NumPy releases the GIL in ufunc loops and
    OpenBLAS calls); reduction partials of the blocks are combined."""

    def __init__(self, name, inputs, threads):
        from concurrent.futures import ThreadPoolExecutor
        self.name = name
        self.inputs = inputs
        self.threads = threads
        self.rows = inputs[0].shape[0]
        self.pool = ThreadPoolExecutor(max_workers=threads)
        nb = min(self.rows, threads * 4)
        e = np.linspace(0, self.rows, nb + 1).astype(np.int64)
        self.blocks = [(int(e[i]), int(e[i + 1])) for i in range(nb)]
        self.prog = WORKLOADS[name]["program"]

    def _part(self, lo, hi):
        return [x[lo:hi] if x.shape and x.shape[0] == self.rows else x for x in self.inputs]

    def step(self):
        name = self.name
        if name == "jacobi":
            def f(b):
                lo, hi = b
                s, e = max(lo - 1, 0), min(hi + 1, self.rows)
                return self.prog(np, [self.inputs[0][s:e]])[0][lo - s:lo - s + (hi - lo)]
            return list(self.pool.map(f, self.blocks))
        if name == "transpose":
            x, y = self.inputs
            return list(self.pool.map(lambda b: _programs().transpose_add(np, x[:, b[0]:b[1]], y[b[0]:b[1]]),
                                      self.blocks))
        if name == "cumsum":
            parts = list(self.pool.map(lambda b: self.prog(np, self._part(*b))[0], self.blocks))
            offs = np.cumsum([np.float32(0)] + [p[-1] for p in parts[:-1]]).astype(np.float32)

            def add(i):
                parts[i] += offs[i]
            list(self.pool.map(add, range(len(parts))))
            return parts
        outs = list(self.pool.map(lambda b: self.prog(np, self._part(*b)), self.blocks))
        if name in ("rownorm", "rownorm-y"):
            total = sum(o[-1] for o in outs)   # combine block partials
            return outs, total
        if name == "kmeans":
            sums = [sum(o[1 + d] for o in outs) for d in range(KM_D)]
            counts = sum(o[-1] for o in outs)
            return outs, sums, counts
        return outs

    def close(self):
        self.pool.shutdown()


def run_reference(args, dist):
    """--impl reference: the reference's CPU path on all host cores, rank 0,
    on the full named shape of the GPU arm's config."""
    if dist.rank != 0:
        return
    name = args.workload
    w = WORKLOADS[name]
    cores = len(os.sched_getaffinity(0))
    n_glob = rows_of(name, args.scaling, dist.world, 0)[0]
    inputs = host_inputs(name, 0, n_glob)
    ref = BlockedNumpy(name, inputs, cores)
    for _ in range(args.warmup):
        ref.step()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        ref.step()
        times.append(time.perf_counter() - t0)
    ref.close()
    t = sum(times) / len(times)
    value = w["elements"](n_glob) / t
    from oracle import programs
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "elements/s",
        "n_gpus": dist.world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": w["label"],
        "data": "synthetic (numpy default_rng, row blocks seeded [42, block])",
        "config": config_of(name, args.scaling, dist.world),
        "cpu_baseline": {"value": value, "unit": "elements/s", "cores": cores, "kind": "port",
                         "cpu_model": cpu_model(),
                         "sample": f"the full named shape ({n_glob} leading rows) per step: eager NumPy program "
                                   f"(+scipy erf) over {len(ref.blocks)} row blocks on {cores} threads"},
        "e2e": {"value": value, "unit": "elements/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "native_shim_mapped": programs.native_shim_mapped(),
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU leg
# ---------------------------------------------------------------------------
def run_grumpy(args, dist):
    import paper_1901_03771_b200 as gp
    from paper_1901_03771_b200 import runtime

    rt = runtime.get()
    name = args.workload
    w = WORKLOADS[name]
    n_glob, lo, hi = rows_of(name, args.scaling, dist.world, dist.rank)
    rows = hi - lo
    prog = w["program"]
    sess = gp.Session()
    gp.set_default_session(sess)

    host = host_inputs(name, lo, hi)
    order = _programs().NAMED[name][4]
    sharded = dist.world > 1 and w.get("collective", False) and w.get("shardable", True)
    if sharded:
        # leading-axis sharding with reduction partials allreduced over NCCL
        import paper_1901_03771_b200.distributed as D
        D.init(backend="nccl", session=sess)

        def inputs_of(arrs):
            return [D.local_input(x, n_glob, lo, session=sess) if c == "S" else gp.asarray(x)
                    for c, x in zip(order, arrs)]
    else:
        # row-local regions: each rank's shard is an independent problem
        def inputs_of(arrs):
            return [gp.asarray(x) for x in arrs]
    dev = inputs_of(host)
    for d in dev:  # upload once (not timed)
        d.node.data.device = rt.upload(d.node.data.host)

    # clocks sampler runs from before warm-up so it has samples under load
    clocks = Clocks(rt.device)
    clocks.start()
    clocks.wait_first(3.0)

    # warmup (includes NVRTC compile on the first step).  The warm-up keeps the
    # same number of step outputs alive as the timed loop, so the caching pool
    # reaches its steady state (no cuMemAlloc inside the timed region).
    t0 = time.perf_counter()
    keep = [prog(gp, dev)]
    gp.force(*keep[0])
    rt.sync()
    cold_s = time.perf_counter() - t0
    for _ in range(max(args.warmup - 1, 3)):
        outs = prog(gp, dev)
        gp.force(*outs)
        keep.append(outs)
        if len(keep) > 2:
            keep.pop(0)
    rt.sync()
    del outs

    # timed region: exactly K steps; per-launch events inside the executor
    k0 = sess.stats.kernels_executed
    c0 = sess.stats.collectives
    e_all0, e_all1 = rt.event(), rt.event()
    sess.executor.enable_profile()
    dist.barrier()
    rt.sync()
    clocks.mark()
    a0 = rt.pool_stats()["cuMemAlloc_calls"]
    h0 = time.perf_counter()
    rt.record(e_all0)
    for i in range(args.steps):
        outs = prog(gp, dev)
        gp.force(*outs)
        keep.append(outs)
        if len(keep) > 2:
            keep.pop(0)
    rt.record(e_all1)
    host_issue_s = time.perf_counter() - h0
    rt.sync()
    allocs_in_timed = rt.pool_stats()["cuMemAlloc_calls"] - a0
    launches = sess.stats.kernels_executed - k0
    collectives = sess.stats.collectives - c0
    prof = sess.executor.take_profile()
    sess.executor.profile = None
    last = keep[-1]
    # keep the GPU loaded (untimed) until the sampler has enough points; the
    # iteration count is agreed over ranks (a step may run a collective, so
    # every rank must run the same number of them)
    step_s = rt.elapsed_ms(e_all0, e_all1) / 1e3 / max(args.steps, 1)
    # (nvidia-smi samples every 100 ms: ~0.8 s of steps covers 5 samples)
    want = 0 if clocks.since_mark() >= 5 else min(int(0.8 / max(step_s, 1e-6)) + 1, 2000)
    for _ in range(int(dist.max(float(want)))):
        outs = prog(gp, dev)
        gp.force(*outs)
    rt.sync()
    clk = clocks.stop()
    dist.barrier()
    my_ms = rt.elapsed_ms(e_all0, e_all1)
    total_ms = dist.max(my_ms)
    del keep
    # dominant launch = largest share of device time in the timed region
    by_label = {}
    for fam, lab, ms in prof:
        by_label.setdefault((fam, lab), []).append(ms)
    work = {k: v for k, v in by_label.items() if k[0] != "collective"}
    dom = max(work.items(), key=lambda kv: sum(kv[1]))
    kmean = statistics.mean(dom[1])
    share = sum(dom[1]) / max(my_ms, 1e-9)
    kernel_ms_step = sum(ms for f, _l, ms in prof if f != "collective") / args.steps
    coll_ms_step = sum(ms for f, _l, ms in prof if f == "collective") / args.steps
    elements = w["elements"](n_glob) * (1 if w.get("shardable", True) else dist.world)
    value = elements * args.steps / (total_ms / 1e3)
    peak, peak_src = peaks()
    alg_bytes = w["bytes"](rows)
    achieved = alg_bytes / (kmean / 1e3) / 1e9
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": _traffic(name), "peak_source": peak_src}
    if dom[0][0] == "library" and dom[0][1] in w.get("library_flops", {}):
        # a library GEMM dominates: tensor-pipe roofline.  FP32 emulated with
        # BF16x9 issues 9 BF16 products per FP32 multiply-add, so its peak is
        # the measured dense BF16 rate / 9
        fl = w["library_flops"][dom[0][1]](rows)
        tf = fl / (kmean / 1e3) / 1e12
        bf = bf16_peak()
        emu = rt.gemm_math == "bf16x9"
        pk = bf / 9 if emu else 148 * 128 * 2 * 1.965e9 / 1e12
        roof = {"bound": "tensor", "achieved": tf, "peak": pk, "unit": "TFLOP/s", "frac": tf / pk,
                "traffic": None,
                "peak_source": ("MEASURED_PEAKS.json bf16_tflops / 9 (BF16x9 emulated FP32)" if emu
                                else "FP32 FMA datasheet: 148 SM x 128 lanes x 2 x 1.965 GHz"),
                "flops_per_launch": fl}

    # parity of the last timed step at the full size
    from oracle import fullsize
    t_par = time.perf_counter()
    got = [np.asarray(o) for o in last]
    del last
    parity = fullsize.check(name, host, got, comm_sum=dist.sum_f64 if sharded else None,
                            world=dist.world if sharded else 1)
    parity["seconds"] = round(time.perf_counter() - t_par, 2)
    parity_ok_all = dist.all_ok(parity["ok"])
    del got

    e2e = _e2e(args, dist, gp, rt, sess, prog, host, inputs_of, elements, pinned=True)
    e2e_pg = _e2e(args, dist, gp, rt, sess, prog, host, inputs_of, elements, pinned=False)

    line = {
        "metric": METRIC, "value": value, "unit": "elements/s", "n_gpus": dist.world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": w["label"],
        "data": "synthetic (numpy default_rng, row blocks seeded [42, block])",
        "config": config_of(name, args.scaling, dist.world),
        "parity": parity,
        "e2e": e2e,
        "e2e_pageable": e2e_pg,
        "roofline": {**roof, "kernel_ms": kmean, "kernel": f"{dom[0][0]}:{dom[0][1]}",
                     "kernel_share_of_step": share, "launches_per_step": len(prof) / args.steps,
                     "algorithmic_bytes_per_launch": alg_bytes, "limiter": w["bound"],
                     "compute": _compute_roofline(w, rows, kmean, clk)},
        "step_breakdown_ms": {"kernels": kernel_ms_step, "collectives": coll_ms_step,
                              "device_step": my_ms / args.steps,
                              "host_issue": host_issue_s * 1e3 / args.steps,
                              "per_launch": {f"{f}:{l}": statistics.mean(v) for (f, l), v in by_label.items()}},
        "repo_kernel_rooflines": [
            {"kernel": k, "kernel_ms": statistics.mean(by_label[tuple(k.split(":", 1))]),
             "algorithmic_bytes": fb(rows),
             "achieved_gbs": fb(rows) / (statistics.mean(by_label[tuple(k.split(":", 1))]) / 1e3) / 1e9,
             "frac": fb(rows) / (statistics.mean(by_label[tuple(k.split(":", 1))]) / 1e3) / 1e9 / peak}
            for k, fb in w.get("repo_bytes", {}).items() if tuple(k.split(":", 1)) in by_label],
        "rows_per_gpu": rows,
        "gpu_launches": launches,
        "collectives_in_timed_region": collectives,
        "cuMemAlloc_in_timed_region": allocs_in_timed,
        "clocks": clk,
        "cold_first_step_s": cold_s,
        "device": rt.name,
        "device_index": rt.device,
        "comm": type(sess.comm).__name__ if sess.comm is not None else None,
    }
    if dist.rank == 0 and dist.world == 1 and not args.no_cpu_baseline:
        sample = min(args.cpu_sample or cpu_sample_n(name), rows)
        sample_in = host_inputs(name, 0, sample)
        sample_elems = w["elements"](sample)
        if name == "transpose":
            # x.T + y needs square blocks: the leading sample x sample corner
            sample_in = [np.ascontiguousarray(a[:, :sample]) for a in sample_in]
            sample_elems = sample * sample
        t = _cpu_time(name, sample_in, 2)
        line["cpu_baseline"] = {"value": sample_elems / t, "unit": "elements/s", "cores": 1,
                                "kind": "port", "cpu_model": cpu_model(),
                                "sample": f"leading extent {sample} (of {n_glob}), eager NumPy program single "
                                          f"thread, best of 2"}
    if dist.rank == 0:
        print(json.dumps(line), flush=True)
    if not parity_ok_all:
        print(f"VerificationFailed: rank {dist.rank} parity {json.dumps(parity)}", file=sys.stderr, flush=True)
        return 1
    return 0


def _cpu_time(name, inputs, reps):
    prog = WORKLOADS[name]["program"]
    best = float("inf")
    for _ in range(reps):
        t0 = time.perf_counter()
        prog(np, inputs)
        best = min(best, time.perf_counter() - t0)
    return best


def _e2e(args, dist, gp, rt, sess, prog, host, inputs_of, elements, pinned):
    """The metric through the public API: host inputs -> program -> every
    output back in host memory, each step (streamed when eligible)."""
    if pinned:
        src = []
        for x in host:
            p = rt.pinned_empty(x.shape, x.dtype)
            p[...] = x
            src.append(p)
    else:
        src = host
    outs0 = prog(gp, inputs_of(src))
    shapes = [(o.shape, o.dtype) for o in outs0]
    del outs0
    dst = [rt.pinned_empty(s, d) if pinned else np.empty(s, d) for s, d in shapes]
    h2d = sum(x.nbytes for x in src)
    d2h = sum(x.nbytes for x in dst)
    steps = max(1, min(args.steps, args.e2e_steps))
    sc0 = sess.stats.streamed_chunks
    # the first call compiles the chunk kernels, the next two reach the
    # pool's and the copy engines' steady state (tools/e2e_probe.py: 11, 5.6,
    # then 4.8 ms per MLP step)
    WARM = 3
    per_step = []
    for it in range(WARM + steps):
        if it == WARM:
            dist.barrier()
            rt.sync()
            t0 = time.perf_counter()
        ts = time.perf_counter()
        outs = prog(gp, inputs_of(src))
        # to_external of every output into host buffers; regions reading host
        # inputs row-locally stream (H2D / kernel / D2H overlap)
        gp.materialize(*outs, out=dst)
        if it >= WARM:
            per_step.append(time.perf_counter() - ts)
    rt.sync()
    s = dist.max(time.perf_counter() - t0)
    return {"value": elements * steps / s, "unit": "elements/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "steps": steps, "host_memory": "page-locked" if pinned else "pageable",
            "streamed_chunks_per_step": (sess.stats.streamed_chunks - sc0) / (WARM + steps),
            "step_ms": {"mean": 1e3 * s / steps, "median": 1e3 * float(np.median(per_step)),
                        "max": 1e3 * max(per_step)}}


def _compute_roofline(w, n, kernel_ms, clk):
    """For kernels bound by an arithmetic pipe rather than HBM: lane-ops per
    second of the dominant kernel against the pipe's peak at the measured SM
    clock (SMs x lanes per SM per clock)."""
    c = w.get("compute")
    if not c:
        return None
    mhz = (clk or {}).get("sm_mhz") or 1965.0
    peak = 148 * c["lanes_per_sm_clk"] * mhz * 1e6
    achieved = w["elements"](n) * c["ops"] / (kernel_ms / 1e3)
    return {"pipe": c["pipe"], "lane_ops_per_element": c["ops"], "achieved_lane_ops_s": achieved,
            "peak_lane_ops_s": peak, "frac": achieved / peak, "peak_clock_mhz": mhz, "note": c["note"]}


def _traffic(workload):
    p = os.path.join(REPO, "profiles", "traffic.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get(workload)
    return None


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="grumpy", choices=["grumpy", "reference"])
    ap.add_argument("--workload", default="blackscholes-f32", choices=sorted(WORKLOADS))
    ap.add_argument("--scaling", default="strong", choices=["weak", "strong"])
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--cpu-sample", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torchrun on this node
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
               os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl != "reference":
        # the native shim (and with it cuBLAS 12.9) loads before anything
        # imports PyTorch (torch.distributed below), whose wheel carries an
        # older libcublas.so.12
        import paper_1901_03771_b200  # noqa: F401
        from paper_1901_03771_b200 import runtime
        # one GPU per rank; a box with fewer GPUs than ranks (the 1-GPU test
        # box) shares devices, and partials then combine through the host
        # (distributed.HostStagedComm) because NCCL needs distinct devices
        ndev = max(runtime.device_count(), 1)
        os.environ.setdefault("GRUMPY_DEVICE", str(int(os.environ.get("LOCAL_RANK", "0")) % ndev))
    # the reference arm runs on rank 0 only: no collectives, no process group
    dist = Dist(gloo=args.impl != "reference")
    rc = 0
    try:
        if args.impl == "reference":
            run_reference(args, dist)
        else:
            rc = run_grumpy(args, dist)
    finally:
        dist.close()
    sys.exit(rc or 0)


if __name__ == "__main__":
    main()
