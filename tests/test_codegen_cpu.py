"""Code generation on CPU: every kernel family is generated and compiled by
NVRTC for sm_100a (no GPU needed), and the generated source keeps the
properties the design relies on (vector loads, no FMA contraction, NumPy-order
reductions, one kernel per region)."""
import re
import subprocess

import numpy as np
import pytest

import paper_1901_03771_b200 as gp
from paper_1901_03771_b200 import codegen, planner, runtime, workloads as wl
from paper_1901_03771_b200.codegen_rows import tree_chunks


@pytest.fixture
def sess():
    s = gp.Session()
    old = gp.set_default_session(s)
    yield s
    gp.set_default_session(old)


def kernels(outs):
    steps = planner.plan_regions([o.node for o in outs], row_fusion=codegen.row_fusable, check=codegen.check_step)
    res = []
    for st in steps:
        if st.kind != "Fused":
            continue
        ks = codegen.cached_generate(codegen.canonicalize(codegen.Region(st.roots, st.leaves, st.nodes)))
        res.append((ks, runtime.compile_cubin(ks.source)))
    return res


def sass(cubin, tmp_path):
    p = tmp_path / "k.cubin"
    p.write_bytes(cubin)
    return subprocess.run(["cuobjdump", "-sass", str(p)], capture_output=True, text=True).stdout


def test_map_family_vectorised_no_fma(sess, tmp_path):
    W, a, b = (gp.asarray(x) for x in wl.listing1_inputs(n=1 << 12))
    (ks, cub), = kernels([wl.listing1(gp, W, a, b)])
    assert ks.family == "map" and ks.vec == 2
    s = sass(cub, tmp_path)
    assert "LDG.E.128" in s and "STG.E.128" in s
    assert "DFMA" not in s            # --fmad=false: NumPy never contracts a*b+c


def test_blackscholes_single_multiroot_kernel(sess):
    S, X, T = (gp.asarray(x) for x in wl.blackscholes_inputs(n=1 << 12))
    ks = kernels(list(wl.blackscholes(gp, S, X, T)))
    assert len(ks) == 1 and ks[0][0].family == "map" and len(ks[0][0].root_slots) == 2


@pytest.mark.parametrize("C", [256, 4096])
def test_rownorm_coop(sess, C, tmp_path):
    (x,) = wl.rownorm_inputs(rows=64, cols=C)
    (ks, cub), = kernels(list(wl.rownorm(gp, gp.asarray(x))))
    assert ks.family == "coop"
    assert "gr::row_sum" in ks.source
    assert ks.source.count("gr::row_sum") == 3   # mean (shared by std via CSE), var, total


def test_rows_tile_pairwise():
    from paper_1901_03771_b200.codegen_rows import rows_tile_pairwise
    assert rows_tile_pairwise(65536, 4096) and rows_tile_pairwise(64, 256) and rows_tile_pairwise(1, 7)
    assert not rows_tile_pairwise(58, 4096)      # 29 rows split mid-row
    assert not rows_tile_pairwise(64, 1)         # 8-accumulator leaves, not a row tree
    assert not rows_tile_pairwise(4, 16)         # 32-element nodes do not split


def test_rownorm_total_non_power_of_two_rows(sess):
    """58 rows: np.sum's pairwise tree over the flattened y is not a tree of
    rows, so the total leaves the row region (row stats become their own step
    and the total runs in flattened-tree mode) instead of a wrong fold."""
    (x,) = wl.rownorm_inputs(rows=58, cols=4096)
    ks = kernels(list(wl.rownorm(gp, gp.asarray(x))))
    assert len(ks) >= 2
    (x,) = wl.rownorm_inputs(rows=64, cols=4096)
    assert len(kernels(list(wl.rownorm(gp, gp.asarray(x))))) == 1


def test_row_families(sess):
    rng = np.random.default_rng(0)
    z = gp.asarray(rng.standard_normal((100, 10)).astype(np.float32))
    p = gp.exp(z - z.max(1)[:, None])
    p = p / p.sum(1)[:, None]
    (ks, _), = kernels([p, p.argmax(1)])
    assert ks.family == "rows"
    x = gp.asarray(rng.standard_normal((300, 50)))
    for outs in ([x.sum(0)], [x.sum()], [x.argmax()], [x.max(1), x.min(1)], [x.std(1)]):
        assert all(k[1] for k in kernels(outs))


def test_kmeans_keyed(sess):
    P, C = (gp.asarray(v) for v in wl.kmeans_inputs(n=1024, k=16, d=4))
    lab, sums, counts = wl.kmeans_partials(gp, P, C)
    (ks, _), = kernels([lab, *sums, counts])
    assert ks.meta["keyed"] == 5 and "__shfl_sync" in ks.source


def test_kmeans_constant_bank_and_match_any(sess):
    """Centroids (row-invariant, 4 KB) go to the constant bank; the keyed sums
    use warp groups of equal keys; the 64-way argmin is unrolled."""
    P, C = (gp.asarray(v) for v in wl.kmeans_inputs(n=8192, k=64, d=4))
    lab, sums, counts = wl.kmeans_partials(gp, P, C)
    (ks, _), = kernels([lab, *sums, counts])
    assert ks.meta["cbank"] and "__constant__ float gr_cin1[256];" in ks.source
    assert "__match_any_sync" in ks.source and "__popc(kpeers)" in ks.source
    # a leaf read per row is never staged in the constant bank
    x = gp.asarray(np.ones((8192, 8), np.float32))
    (ks2, _), = kernels([(x * 2.0).argmax(1)])
    assert not ks2.meta["cbank"]


def test_paired_argmin_loop_compiles(sess, monkeypatch):
    from paper_1901_03771_b200 import codegen_rows
    monkeypatch.setattr(codegen_rows, "PAIR_LOOPS", True)
    monkeypatch.setattr(codegen_rows, "NEAREST", False)     # the exact paired scan itself
    codegen._GEN_CACHE.clear()
    P, C = (gp.asarray(v) for v in wl.kmeans_inputs(n=8192, k=64, d=4))
    lab = wl.kmeans_assign(gp, P, C)
    (ks, cubin), = kernels([lab])
    assert "gr::p2::square_nc" in ks.source and "2 * i" in ks.source and cubin
    codegen._GEN_CACHE.clear()


def test_views_and_slice_assign(sess):
    rng = np.random.default_rng(1)
    a = gp.asarray(rng.standard_normal((66, 66)))
    b = gp.asarray(rng.standard_normal((66, 66)))
    # one Jacobi sweep in slice-assign form
    b[1:-1, 1:-1] = 0.2 * (a[1:-1, 1:-1] + a[1:-1, :-2] + a[1:-1, 2:] + a[:-2, 1:-1] + a[2:, 1:-1])
    ks = kernels([b])
    assert len(ks) == 1
    t = gp.asarray(rng.standard_normal((8, 6, 4)))
    ks = kernels([t.transpose(2, 0, 1).reshape(4, 48)[:, ::3] * 2])
    assert len(ks) == 1


def test_tree_chunks_match_numpy_split():
    def leaves(n, depth):
        if depth == 0:
            return [n]
        h = n // 2
        h -= h % 8
        return leaves(h, depth - 1) + leaves(n - h, depth - 1)
    for n in (3000, 10 ** 6, 1 << 20, 123457):
        D, sizes = tree_chunks(n)
        got = leaves(n, D)
        assert len(got) == 1 << D and sorted(set(got)) == sizes and sum(got) == n


def test_literals_bit_exact():
    assert codegen.c_literal(0.1, gp.DType.f32) == "gr::f32_bits(0x3dcccccdu)"
    assert codegen.c_literal(-0.0, gp.DType.f64) == "gr::f64_bits(0x8000000000000000ull)"
    assert codegen.c_literal(-(2 ** 31), gp.DType.i32) == "(-2147483647 - 1)"
