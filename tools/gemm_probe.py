"""np.dot boundary study on the MLP's first layer,
X[65536,784] @ W1[784,1024] + b1 -> ReLU:

  sgemm        cublasSgemm FP32 (CUDA cores) + the fused R1 bias+ReLU kernel
  sgemm-bf16x9 the same GEMM with FP32 emulated by BF16x9 tensor-core products
  lt-epi       cuBLASLt FP32 GEMM with the RELU_BIAS epilogue (no R1 kernel)
  lt-epi-x9    cuBLASLt emulated FP32 with the RELU_BIAS epilogue

Times: CUDA events, mean of 20 after 3 warm-ups.  Accuracy: error of h
against a float64 reference on 2048 sampled rows, relative to sum|x||w|.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1901_03771_b200 as gp  # noqa: E402
from paper_1901_03771_b200 import runtime, workloads as wl  # noqa: E402
from paper_1901_03771_b200.tensor import DType  # noqa: E402


def timed(rt, fn, reps=20):
    for _ in range(3):
        fn()
    ev = []
    for _ in range(reps):
        a, b = rt.event(), rt.event()
        rt.record(a)
        fn()
        rt.record(b)
        ev.append((a, b))
    return float(np.mean([rt.elapsed_ms(a, b) for a, b in ev]))


def main():
    rt = runtime.get()
    X, W1, b1, _, _ = wl.mlp_inputs()
    B, K = X.shape
    H = W1.shape[1]
    dX, dW, db = rt.upload(X), rt.upload(W1), rt.upload(b1)
    C = rt.alloc(B * H * 4)
    rows = np.random.default_rng(0).choice(B, 2048, replace=False)
    ref = np.maximum(X[rows].astype(np.float64) @ W1.astype(np.float64) + b1, 0)
    scale = np.abs(X[rows]).astype(np.float64) @ np.abs(W1).astype(np.float64) + np.abs(b1)

    def err(h):
        d = np.abs(h[rows].astype(np.float64) - ref) / scale
        return float(d.max()), float(np.sqrt(np.mean(d * d)))

    # the grumpy R1 region kernel (bias + ReLU over the GEMM output)
    sess = gp.Session()
    gp.set_default_session(sess)
    hg = gp.asarray(np.zeros((B, H), np.float32))
    hg.node.data.device = C
    r1 = gp.maximum(hg + gp.asarray(b1), 0)
    gp.force(r1)
    st = sess.executor.last_steps[0]
    k, grid = st.cache["kernel"], st.cache["grid"]
    out = sess.graph  # noqa: F841
    R = rt.alloc(B * H * 4)
    params = runtime.pack_params([sess.executor.device_ptr(l) for l in [st.leaves[i] for i in st.cache["perm"]]]
                                 + [R.ptr])
    r1_ms = timed(rt, lambda: rt.launch(k, grid, k.block, params))

    res = {}
    for mode in ("fp32", "bf16x9"):
        rt.set_gemm_math(mode)
        ms = timed(rt, lambda: rt.gemm(False, False, B, H, K, DType.f32, dX.ptr, K, dW.ptr, H, C.ptr, H))
        rt.launch(k, grid, k.block, params)
        rt.sync()
        h = R.to_numpy(DType.f32, (B, H))
        res["sgemm" if mode == "fp32" else "sgemm-bf16x9"] = (ms, ms + r1_ms, err(h))
    rt.set_gemm_math("fp32")
    for name, emu in (("lt-epi", False), ("lt-epi-x9", True)):
        ms = timed(rt, lambda: rt.gemm_epilogue(False, False, B, H, K, dX.ptr, K, dW.ptr, H, C.ptr, H,
                                               bias=db.ptr, epilogue="relu_bias", emulate=emu))
        rt.sync()
        h = C.to_numpy(DType.f32, (B, H))
        res[name] = (ms, ms, err(h))
    flops = 2.0 * B * K * H
    print(f"R1 bias+ReLU kernel: {r1_ms:.4f} ms")
    for name, (g, tot, (emax, erms)) in res.items():
        print(f"{name:13s} gemm {g:.4f} ms ({flops / g / 1e9:.0f} GFLOP/s)  gemm+epilogue {tot:.4f} ms  "
              f"err max {emax:.3e} rms {erms:.3e} (relative to sum|x||w|)", flush=True)


if __name__ == "__main__":
    main()
