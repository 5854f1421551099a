#!/usr/bin/env python
"""Generate the committed golden fixtures (run from the repo root).

spec_kats.json   — every known-answer example the reference spec states for
                   this path (/root/reference/SPEC.md, cited per entry).  The
                   reference ships no tests or executable engine (SURVEY.md §0,
                   §8(c)), so these prose KATs are its golden vectors.
configs_small.npz — inputs and NumPy/SciPy outputs of the five BASELINE.json
                   configs at small sizes, computed with the reference's own
                   arithmetic dependencies (numpy 2.3.5, scipy 1.18.1;
                   pkg/pyproject.toml:10-14) by the user programs of
                   paper_1901_03771_b200/workloads.py run with xp = numpy.
"""

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

from paper_1901_03771_b200 import workloads as wl  # noqa: E402

SPEC_KATS = [
    # tensor-core
    {"name": "broadcast_equal", "ref": "SPEC.md:51", "op": "broadcast_shapes", "a": [2, 3], "b": [2, 3], "expect": [2, 3]},
    {"name": "broadcast_col_row", "ref": "SPEC.md:52", "op": "broadcast_shapes", "a": [1024, 1], "b": [1024], "expect": [1024, 1024]},
    {"name": "broadcast_incompatible", "ref": "SPEC.md:53", "op": "broadcast_shapes", "a": [3, 4], "b": [2, 4], "raises": "IncompatibleShapes"},
    {"name": "delinearize_0", "ref": "SPEC.md:60", "op": "delinearize", "linear": 0, "shape": [4, 5], "expect": [0, 0]},
    {"name": "delinearize_7", "ref": "SPEC.md:61", "op": "delinearize", "linear": 7, "shape": [4, 5], "expect": [1, 2]},
    {"name": "delinearize_19", "ref": "SPEC.md:62", "op": "delinearize", "linear": 19, "shape": [4, 5], "expect": [3, 4]},
    {"name": "delinearize_oob", "ref": "SPEC.md:58", "op": "delinearize", "linear": 20, "shape": [4, 5], "raises": "OutOfBounds"},
    # expr-dag inference
    {"name": "infer_mul_broadcast", "ref": "SPEC.md:146", "op": "infer_map_mul", "shapes": [[1024, 1], [1024]], "expect": [1024, 1024]},
    {"name": "infer_matvec", "ref": "SPEC.md:147", "op": "infer_matvec", "shapes": [[10, 784], [784]], "expect": [10]},
    {"name": "infer_reduce_all", "ref": "SPEC.md:148", "op": "infer_reduce_all", "shapes": [[4, 5]], "expect": []},
    {"name": "infer_transpose", "ref": "SPEC.md:153", "op": "infer_transpose", "shapes": [[3, 7]], "perm": [1, 0], "expect": [7, 3]},
    {"name": "infer_slice_interior", "ref": "SPEC.md:154", "op": "infer_slice", "shapes": [[66, 66]], "expect": [64, 64]},
    {"name": "infer_scan", "ref": "SPEC.md:155", "op": "infer_scan", "shapes": [[5]], "expect": [5]},
    # executor
    {"name": "run_map_identity", "ref": "SPEC.md:370", "op": "map_identity", "x": [1, 2, 3, 4], "expect": [1, 2, 3, 4]},
    {"name": "run_map_reduce_sum", "ref": "SPEC.md:379", "op": "sum", "x": [1, 2, 3, 4], "expect": 10},
    {"name": "run_map_reduce_inner", "ref": "SPEC.md:380", "op": "inner", "a": [1, 2, 3], "b": [4, 5, 6], "expect": 32},
    {"name": "run_map_scan_cumsum", "ref": "SPEC.md:388", "op": "cumsum", "x": [1, 2, 3], "expect": [1, 3, 6]},
    {"name": "run_map_scan_zeros", "ref": "SPEC.md:389", "op": "cumsum", "x": [0, 0, 0, 0], "expect": [0, 0, 0, 0]},
    {"name": "run_map_scan_max", "ref": "SPEC.md:390", "op": "cummax", "x": [3, 1, 4, 1, 5], "expect": [3, 3, 4, 4, 5]},
    {"name": "gemv_identity", "ref": "SPEC.md:397", "op": "gemv", "A": [[1, 0, 0], [0, 1, 0], [0, 0, 1]], "x": [7, 8, 9], "trans": False, "expect": [7, 8, 9]},
    {"name": "gemv_trans", "ref": "SPEC.md:398", "op": "gemv", "A": [[1, 2], [3, 4]], "x": [1, 1], "trans": True, "expect": [4, 6]},
    # lowering
    {"name": "eval_point_const", "ref": "SPEC.md:316", "op": "const3", "shape": [4], "expect": [3.0, 3.0, 3.0, 3.0]},
    {"name": "eval_point_inner_i2", "ref": "SPEC.md:317", "op": "inner_point", "a": [1, 2, 3], "b": [4, 5, 6], "i": 2, "expect": 18},
]


def main():
    with open(os.path.join(HERE, "spec_kats.json"), "w") as f:
        json.dump(SPEC_KATS, f, indent=1)
    from scipy.special import erf  # noqa: F401  (SciPy is the reference's erf)
    out = {}
    W, a, b = wl.listing1_inputs(n=4099, seed=1)
    out.update(l1_W=W, l1_a=a, l1_b=b, l1_out=wl.listing1(np, W, a, b))
    for dt, tag in ((np.float32, "f32"), (np.float64, "f64")):
        S, X, T = wl.blackscholes_inputs(n=4099, seed=2, dtype=dt)
        c, p = wl.blackscholes(np, S, X, T)
        out.update({f"bs{tag}_S": S, f"bs{tag}_X": X, f"bs{tag}_T": T, f"bs{tag}_call": c, f"bs{tag}_put": p})
    (x,) = wl.rownorm_inputs(rows=64, cols=512, seed=3)
    y, tot = wl.rownorm(np, x)
    out.update(rn_x=x, rn_y=y, rn_total=np.asarray(tot))
    X, W1, b1, W2, b2 = wl.mlp_inputs(batch=256, hidden=64, seed=4)
    pr, lab = wl.mlp(np, X, W1, b1, W2, b2)
    out.update(mlp_X=X, mlp_W1=W1, mlp_b1=b1, mlp_W2=W2, mlp_b2=b2, mlp_p=pr, mlp_lab=lab)
    P, C = wl.kmeans_inputs(n=4096, k=64, d=4, seed=5)
    klab, ksums, kcounts = wl.kmeans_partials(np, P, C)
    out.update(km_P=P, km_C=C, km_lab=klab, km_sums=np.stack(ksums, 1), km_counts=kcounts)
    np.savez_compressed(os.path.join(HERE, "configs_small.npz"), **out)
    print("wrote", len(SPEC_KATS), "KATs and", len(out), "arrays")


if __name__ == "__main__":
    main()
