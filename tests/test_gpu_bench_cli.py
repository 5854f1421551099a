"""The bench CLI's SPEC examples and npy stores of
lazy results, on the GPU."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_1901_03771_b200 as gp
from paper_1901_03771_b200 import bench_cli, npyio, workloads as wl

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_blackscholes_example():
    rep = bench_cli.run("blackscholes", 10 ** 5, seed=42, dtype="f64")
    assert rep["status"] == "PASSED", rep
    assert rep["kernels_executed"] == 1 and rep["library_calls"] == 0
    assert rep["max_abs_err"] <= 1e-10 * 100


def test_jacobi_example():
    rep = bench_cli.run("jacobi", 512, iters=10, seed=42, dtype="f64")
    assert rep["status"] == "PASSED", rep
    assert rep["kernels_executed"] == 10          # one fused kernel per sweep


def test_innerproduct_example():
    rep = bench_cli.run("innerproduct", 10 ** 6, seed=42)
    assert rep["status"] == "PASSED", rep
    assert rep["kernels_executed"] == 1


def test_kmeans_and_cumsum_reports():
    rep = bench_cli.run("kmeans", 1 << 14, iters=3, seed=3)
    assert rep["status"] == "PASSED", rep
    rep = bench_cli.run("cumsum", 1 << 20, seed=3)
    assert rep["status"] == "PASSED", rep
    assert set(rep) == set(bench_cli.REPORT_KEYS)


def test_cli_process_cold_exceeds_warm(tmp_path):
    """A fresh process with an empty cubin cache: cold (plan + NVRTC compile
    + run) exceeds warm; exit code 0, JSON report and npy
    outputs written."""
    env = dict(os.environ, GRUMPY_CACHE_DIR=str(tmp_path / "cache"), PYTHONPATH=ROOT)
    out = tmp_path / "r.json"
    p = subprocess.run([sys.executable, "-m", "paper_1901_03771_b200.bench_cli", "run", "blackscholes",
                        "--size", "1000", "--iters", "1", "--seed", "42", "--json", str(out),
                        "--outputs-npy", str(tmp_path / "o")], env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr
    rep = json.loads(out.read_text())
    g = rep["engines"]["grumpy_b200"]
    assert g["cold_s"] > g["warm_s"] and g["compile_ms"] > 0
    call = np.load(tmp_path / "o" / "blackscholes_out0.npy")
    S, X, T = wl.blackscholes_inputs(1000, 42, np.float64)
    ec, _ = wl.blackscholes(np, S, X, T)
    assert np.max(np.abs(call - ec)) <= 1e-12 * 100


def test_save_lazy_result_and_reload(tmp_path):
    s = gp.Session()
    old = gp.set_default_session(s)
    try:
        x = np.random.default_rng(0).standard_normal((64, 33))
        y = gp.asarray(x) * 2.0 + 1.0                   # pending: the store forces it
        gp.save(tmp_path / "y.npy", y)
        assert s.stats.kernels_executed == 1
        assert np.array_equal(np.load(tmp_path / "y.npy"), x * 2.0 + 1.0)
        z = gp.load(tmp_path / "y.npy")
        assert np.array_equal(np.asarray(z.sum(axis=1)), (x * 2.0 + 1.0).sum(axis=1))
    finally:
        gp.set_default_session(old)


def test_jit_pipelining_multi_step_cold(tmp_path):
    """A cold multi-step plan compiles its kernels on worker threads
    (GRUMPY_PRECOMPILE) and still produces the right results."""
    env = dict(os.environ, GRUMPY_CACHE_DIR=str(tmp_path / "c"), PYTHONPATH=ROOT)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "jit_pipeline_probe.py")], env=env,
                       capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr
    lines = [json.loads(l.split(" ", 1)[1]) for l in p.stdout.splitlines() if l.startswith("precompile=")]
    assert len(lines) == 4 and all(l["ok"] for l in lines)
    assert len({l["kernels"] for l in lines}) == 1 and lines[0]["kernels"] >= 4
