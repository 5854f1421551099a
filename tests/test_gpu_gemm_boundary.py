"""np.dot boundary: BF16x9-emulated FP32 GEMMs and
the cuBLASLt BIAS / RELU_BIAS epilogues that absorb the R1 region."""
import numpy as np
import pytest

import paper_1901_03771_b200 as gp
from paper_1901_03771_b200 import runtime, session as gsession, workloads as wl

pytestmark = pytest.mark.gpu


@pytest.fixture
def sess():
    s = gp.Session()
    old = gp.set_default_session(s)
    yield s
    gp.set_default_session(old)


def _scale(X, W, b):
    return np.abs(X).astype(np.float64) @ np.abs(W).astype(np.float64) + np.abs(b)


def test_emulation_active():
    # this process loaded the shim before any PyTorch import
    assert runtime.get().gemm_math == gsession.GEMM_MATH == "bf16x9"


@pytest.mark.parametrize("shape", [(257, 131, 67), (1024, 784, 256), (5, 3, 1)])
def test_relu_bias_layer(sess, shape):
    m, k, n = shape
    rng = np.random.default_rng(m)
    X = rng.standard_normal((m, k)).astype(np.float32)
    W = rng.standard_normal((k, n)).astype(np.float32)
    b = rng.standard_normal(n).astype(np.float32)
    h = gp.maximum(gp.asarray(X) @ gp.asarray(W) + gp.asarray(b), 0)
    steps = sess.plan([h.node])
    assert len(steps) == 1 and steps[0].kind == "Library" and steps[0].epilogue[0] == "relu_bias"
    got = np.asarray(h)
    assert sess.stats.library_calls == 1 and sess.stats.kernels_executed == 0
    ref = np.maximum(X.astype(np.float64) @ W.astype(np.float64) + b, 0)
    # FP32-accurate: within a few ulps of the float64 result, relative to sum|x||w|
    assert np.max(np.abs(got - ref) / _scale(X, W, b)) < 4 * np.finfo(np.float32).eps
    assert np.array_equal(got == 0, ref == 0) or np.mean((got == 0) != (ref == 0)) < 1e-3


def test_bias_only_and_transposed_operand(sess):
    rng = np.random.default_rng(3)
    X = rng.standard_normal((300, 96)).astype(np.float32)
    W = rng.standard_normal((40, 96)).astype(np.float32)
    b = rng.standard_normal((1, 40)).astype(np.float32)
    z = gp.asarray(X) @ gp.asarray(W).T + gp.asarray(b)       # transpose absorbed into the op flag
    t = z.sum()                                                 # z has two consumers: no ReLU absorbed
    steps = sess.plan([z.node, t.node])
    lib = [s for s in steps if s.kind == "Library"]
    assert len(lib) == 1 and lib[0].epilogue[0] == "bias" and lib[0].trans_flags == (False, True)
    gp.force(z, t)
    ref = X.astype(np.float64) @ W.T.astype(np.float64) + b
    assert np.max(np.abs(np.asarray(z) - ref) / _scale(X, W.T, b)) < 4 * np.finfo(np.float32).eps


def test_nan_and_signed_zero_follow_numpy(sess):
    """NaN rows stay NaN through the fused ReLU (np.maximum propagates NaN)."""
    rng = np.random.default_rng(4)
    X = rng.standard_normal((64, 32)).astype(np.float32)
    W = rng.standard_normal((32, 16)).astype(np.float32)
    b = rng.standard_normal(16).astype(np.float32)
    X[5, 3] = np.nan
    X[9] = 0.0
    b[2] = -1.0
    got = np.asarray(gp.maximum(gp.asarray(X) @ gp.asarray(W) + gp.asarray(b), 0))
    exp = np.maximum(X @ W + b, 0)
    assert np.array_equal(np.isnan(got), np.isnan(exp))
    fin = ~np.isnan(exp)
    np.testing.assert_allclose(got[fin], exp[fin], rtol=1e-5, atol=1e-5)


def test_mlp_plan_two_library_steps_one_kernel(sess):
    X, W1, b1, W2, b2 = wl.mlp_inputs(batch=2048, hidden=256)
    p, lab = wl.mlp(gp, *[gp.asarray(a) for a in (X, W1, b1, W2, b2)])
    gp.force(p, lab)
    assert sess.stats.library_calls == 2 and sess.stats.kernels_executed == 1
    ep, elab = wl.mlp(np, X, W1, b1, W2, b2)
    np.testing.assert_allclose(np.asarray(p), ep, rtol=1e-4, atol=1e-6)
    assert np.mean(np.asarray(lab) == elab) >= 0.999


def test_emulated_gemm_special_values(sess):
    """BF16x9-emulated FP32 keeps IEEE special values: +-inf rows, NaN rows,
    results near the overflow threshold and subnormal results (tools/gemm_special_values.py)."""
    rng = np.random.default_rng(0)
    X = rng.random((64, 32)).astype(np.float32)
    W = rng.random((32, 16)).astype(np.float32)
    X[3, 5], X[7, 1], X[9, 2], X[11, 0] = np.inf, -np.inf, 3e38, np.nan
    X[10, :] = 1e-40
    got = np.asarray(gp.asarray(X) @ gp.asarray(W))
    with np.errstate(all="ignore"):
        exp = X.astype(np.float64) @ W.astype(np.float64)
    assert np.array_equal(np.isnan(got), np.isnan(exp))
    assert np.array_equal(np.isinf(got), np.isinf(exp)) and np.array_equal(got[np.isinf(exp)], exp[np.isinf(exp)])
    fin = np.isfinite(exp) & (np.abs(exp) > 1e-37)
    assert np.max(np.abs(got[fin] - exp[fin]) / np.abs(exp[fin])) < 4 * np.finfo(np.float32).eps
    sub = np.isfinite(exp) & (np.abs(exp) <= 1e-37)
    assert np.max(np.abs(got[sub] - exp[sub])) < 1e-44 * 32    # a few subnormal ulps


def _skinny_ref(A, B):
    """float64 product and its |A||B| scale (the tolerance's sum of |terms|)."""
    return A.astype(np.float64) @ B.astype(np.float64), np.abs(A).astype(np.float64) @ np.abs(B).astype(np.float64)


@pytest.mark.parametrize("R,K,N", [(8192, 256, 10), (4096 + 37, 32, 16), (5000, 1024, 1), (65536, 1024, 10)])
def test_skinny_product_forced(sess, R, K, N):
    """z = A @ B with B small: one row kernel (TMA-streamed A, constant-bank
    B), no library call; |z - z64| <= 2K eps32 sum|a||b| (fp32 FMA chains)."""
    rng = np.random.default_rng(R + K + N)
    A = rng.standard_normal((R, K)).astype(np.float32)
    B = rng.standard_normal((K, N)).astype(np.float32)
    z = gp.asarray(A) @ gp.asarray(B)
    got = np.asarray(z)
    assert sess.stats.library_calls == 0 and sess.stats.kernels_executed == 1
    e, sc = _skinny_ref(A, B)
    assert np.all(np.abs(got - e) <= 2 * K * 6e-8 * sc)


def test_skinny_product_with_row_consumers(sess):
    rng = np.random.default_rng(5)
    A = rng.standard_normal((8192, 128)).astype(np.float32)
    B = rng.standard_normal((128, 7)).astype(np.float32)
    b = rng.standard_normal(7).astype(np.float32)
    ga = gp.asarray(A)
    z = ga @ gp.asarray(B) + gp.asarray(b)
    m = z.max(1)
    y = gp.maximum(z, 0) * 2.0
    am = z.argmax(1)
    gp.force(m, y, am)
    assert sess.stats.library_calls == 0
    e = A.astype(np.float64) @ B.astype(np.float64) + b
    _, sc = _skinny_ref(A, B)
    tol = 2 * 128 * 6e-8 * (sc + np.abs(b))
    assert np.all(np.abs(np.asarray(m) - e.max(1)) <= tol.max(1))
    assert np.all(np.abs(np.asarray(y) - np.maximum(e, 0) * 2) <= 2 * tol)
    lab = np.asarray(am)
    srt = np.sort(e, axis=1)
    clear = (srt[:, -1] - srt[:, -2]) > 2 * tol.max(1)
    assert np.array_equal(lab[clear], e.argmax(1)[clear])


def test_mlp_layer2_fused(sess):
    """C4 at batch 8192: layer 1 = one cuBLASLt GEMM with the RELU_BIAS
    epilogue, layer 2 + b2 + softmax + argmax = one hand-written row kernel."""
    X, W1, b1, W2, b2 = wl.mlp_inputs(batch=8192, hidden=1024)
    p, lab = wl.mlp(gp, *[gp.asarray(a) for a in (X, W1, b1, W2, b2)])
    gp.force(p, lab)
    assert sess.stats.library_calls == 1 and sess.stats.kernels_executed == 1
    ep, elab = wl.mlp(np, X, W1, b1, W2, b2)
    assert np.max(np.abs(np.asarray(p) - ep)) <= 1e-5
    assert np.array_equal(np.asarray(lab), elab)


def test_skinny_disabled_matches(sess, monkeypatch):
    from paper_1901_03771_b200 import codegen_rows
    rng = np.random.default_rng(9)
    A = rng.standard_normal((8192, 64)).astype(np.float32)
    B = rng.standard_normal((64, 3)).astype(np.float32)
    z1 = np.asarray(gp.asarray(A) @ gp.asarray(B))
    monkeypatch.setattr(codegen_rows, "SKINNY", False)
    s2 = gp.Session()
    z2 = np.asarray(gp.asarray(A, session=s2) @ gp.asarray(B, session=s2))
    assert s2.stats.library_calls == 1
    e, sc = _skinny_ref(A, B)
    assert np.all(np.abs(z1 - e) <= 2 * 64 * 6e-8 * sc) and np.all(np.abs(z2 - e) <= 2 * 64 * 6e-8 * sc)
