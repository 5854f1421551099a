"""Code-generation choices of round 2, checked on CPU (sources and NVRTC
builds, no GPU): DAG-determined product fusion in inexact regions, the
nearest-centre pattern, row prefetch and 32-bit bincount keys, the TMA scan
and warp-per-row generators."""
import numpy as np
import pytest

import paper_1901_03771_b200 as gp
from paper_1901_03771_b200 import codegen, codegen_rows, codegen_scan, runtime, workloads as wl


def _source(roots):
    sess = gp.session.default_session()
    st = sess.plan([r.node for r in roots])[0]
    return codegen.generate(codegen.canonicalize(codegen.Region(st.roots, st.leaves, st.nodes)))


def test_fusion_same_in_packed_body_and_tail():
    """An inexact f32 region with a tail: the packed body fuses with explicit
    FFMA2 and the scalar tail with FMA — never ptxas's own contraction (whose
    choice follows the emission order)."""
    S, X, T = wl.blackscholes_inputs(n=(1 << 12) + 3)
    ks = _source(list(wl.blackscholes(gp, *map(gp.asarray, (S, X, T)))))
    body, tail = ks.source.split("void tail(")
    assert "gr::p2::fma(" in body and "gr::fma_(" in tail
    assert "ldv_part" not in ks.source                # the ptxas-contraction experiment is off
    assert "gr::p2::mul_nc" in body                  # unfused products stay uncontractable


def test_fusion_picks_by_operand_position():
    """a*b - c*d: the product fused is fixed by the DAG (the last operand by
    default), the other is formed uncontractably."""
    rng = np.random.default_rng(1)
    a, b, c, d = (gp.asarray(rng.standard_normal(4096).astype(np.float32)) for _ in range(4))
    ks = _source([a * b - gp.exp(c) * d])
    assert "gr::p2::fma(" in ks.source and "gr::p2::mul_nc(" in ks.source
    assert codegen.FMA_PICK in ("first", "last")


def test_exact_regions_never_fuse():
    rng = np.random.default_rng(2)
    a, b = (gp.asarray(rng.standard_normal(4096).astype(np.float32)) for _ in range(2))
    ks = _source([a * b + 1.0])
    assert "fma(" not in ks.source.replace("mul_nc", "")


@pytest.mark.parametrize("form", ["square", "mul", "reversed"])
def test_nearest_pattern_forms(form):
    P, C = wl.kmeans_inputs(n=4096, k=16, d=3)
    gP, gC = gp.asarray(P), gp.asarray(C)
    if form == "square":
        d = ((gP[:, None, :] - gC[None]) ** 2).sum(-1)
    elif form == "mul":
        t = gP[:, None, :] - gC[None]
        d = (t * t).sum(-1)
    else:
        d = ((gC[None] - gP[:, None, :]) ** 2).sum(-1)
    assert codegen_rows.match_nearest(d.node, (1,)) is not None
    ks = _source([d.argmin(1)])
    assert "gr::nearest_centre<16, 3>" in ks.source and "gr_nnpack" in ks.source
    assert ks.meta["cbank_pair"]
    runtime.compile_cubin(ks.source)


def test_nearest_not_for_other_programs():
    P, C = wl.kmeans_inputs(n=4096, k=15, d=3)            # odd centre count
    gP, gC = gp.asarray(P), gp.asarray(C)
    d = ((gP[:, None, :] - gC[None]) ** 2).sum(-1)
    assert codegen_rows.match_nearest(d.node, (1,)) is None
    P2, C2 = wl.kmeans_inputs(n=4096, k=16, d=3)
    d2 = ((gp.asarray(P2)[:, None, :] - gp.asarray(C2)[None]) ** 2).sum(-1)
    assert "nearest_centre" not in _source([d2.argmax(1)]).source      # argmax: the plain scan


def test_kmeans_row_prefetch_and_match32():
    P, C = wl.kmeans_inputs(n=1 << 14)
    lab, sums, counts = wl.kmeans_partials(gp, gp.asarray(P), gp.asarray(C))
    ks = _source([lab] + sums + [counts])
    assert "gr::prefetch_l1(p.in0 + (r + stride) * 4LL)" in ks.source
    assert "(unsigned)kkey : 0xffffffffu" in ks.source
    assert "const float kw0 = L" in ks.source                  # weights reuse the row's vector load
    assert "gr::nearest_exact<64, 4>(" in ks.source             # the exact scan out of line
    runtime.compile_cubin(ks.source)


def test_scan_tma_generator_builds(monkeypatch):
    monkeypatch.setattr(codegen_scan, "SCAN_TMA", True)
    x = gp.asarray(np.arange(1 << 20, dtype=np.float32))
    ks = _source([gp.cumsum(x * 0.5 + 1.0)])
    assert ks.meta["label"] == "scan-tma"
    assert len(ks.meta["tmaps"]) == 2 and ks.meta["tmaps"][-1][0] == 1     # leaf map + output map
    # look-back by rounds: the round's aggregates as a warp tree, one warp
    assert "gr::round_tree<" in ks.source and "mbar_wait(&own_bar" not in ks.source
    runtime.compile_cubin(ks.source)
    # the left-fold alternative: two warps handing the CTA's prefix over
    monkeypatch.setattr(codegen_scan, "SCAN_TMA_TREE", False)
    monkeypatch.setattr(codegen_scan, "SCAN_TMA_LBW", 2)
    two = _source([gp.cumsum(x * 0.5 + 1.0 + 0.0)]).source
    assert "gr::round_stage<" in two and "gr::round_fold<" in two and "mbar_wait(&own_bar" in two
    runtime.compile_cubin(two)
    monkeypatch.setattr(codegen_scan, "SCAN_TMA_LBW", 1)
    one = _source([gp.cumsum(x * 0.5 + 2.0)]).source
    assert "gr::tile_lookback_round<" in one and "mbar_wait(&own_bar" not in one
    runtime.compile_cubin(one)
    odd = gp.asarray(np.arange((1 << 20) + 7, dtype=np.float32))
    tail = _source([gp.cumsum(odd)])
    assert tail.meta["label"] == "scan-tma" and "K::tail_value(p, ix)" in tail.source   # tail past the last line
    assert tail.meta["tmaps"][0][2] == ((1 << 20) + 7) // 32
    runtime.compile_cubin(tail.source)


def test_wrow_generator_paired_two_pass(monkeypatch):
    monkeypatch.setattr(codegen, "ROW_FAMILY", "wrow")
    (x,) = wl.rownorm_inputs(rows=256, cols=4096)
    y, t = wl.rownorm(gp, gp.asarray(x))
    ks = _source([t])
    assert ks.family == "wrow"
    assert "gr::p2::div_shr<FAST>" in ks.source and "K::rows<false>" in ks.source
    runtime.compile_cubin(ks.source)


def test_kmeans_two_rows_per_search_builds(monkeypatch):
    monkeypatch.setattr(codegen_rows, "NEAREST_PAIR_ROWS", True)
    P, C = wl.kmeans_inputs(n=1 << 14)
    lab, sums, counts = wl.kmeans_partials(gp, gp.asarray(P), gp.asarray(C))
    ks = _source([lab] + sums + [counts])
    assert "gr::nearest_centre_n<64, 4, 2>" in ks.source and "K::nn_labels(" in ks.source
    runtime.compile_cubin(ks.source)


@pytest.mark.parametrize("dt", [np.float32, np.float64, np.int32])
def test_scan_rows_generator_builds(dt):
    """Scans along the last axis go to the warp-per-32-lines kernel (coalesced
    through a padded shared tile; the 48 KB static limit sizes the CTA); other
    axes and short line counts stay thread-per-line."""
    x = gp.asarray(np.ones((1000, 300), dt))
    ks = _source([gp.cumsum(x * 3 + 1, axis=1)])
    assert ks.meta["label"] == "scan-rows" and "K::val(p, r, k)" in ks.source
    runtime.compile_cubin(ks.source)
    assert _source([gp.cumsum(x * 3 + 1, axis=0)]).meta.get("label") is None          # lines
    assert _source([gp.cumsum(gp.asarray(np.ones((31, 300), dt)), axis=1)]).meta.get("label") is None



@pytest.mark.parametrize("shape,label,tiles", [((64, 65536), "scan-tma", 512), ((64, 100003), "scan-lookback", 64 * 13),
                                               ((16, 70001), "scan-lookback", 16 * 9)])
def test_scan_few_long_lines_segmented(shape, label, tiles):
    """Few long lines along the last axis: one look-back scan per line — TMA
    when lines are whole 8192-element tiles, else register-staged with a
    partial last tile per line; the look-back stops at the line's first tile."""
    x = gp.asarray(np.ones(shape, np.float32))
    ks = _source([gp.cumsum(x * 3 + 1, axis=-1)])
    assert ks.meta["label"] == label and ks.meta["tiles"] == tiles
    tpl = -(-shape[-1] // 8192)
    assert f"(t / {tpl}LL) * {tpl}LL" in ks.source
    runtime.compile_cubin(ks.source)


def test_debug_bounds_checks_every_family(monkeypatch):
    """GRUMPY_DEBUG_BOUNDS=1: every leaf read of the
    generated kernels goes through gr::bounds_ok (print + trap); the sources
    still compile.  Staged TMA tiles are exempt (they read zero fill, not
    global memory)."""
    from paper_1901_03771_b200 import codegen_coop
    monkeypatch.setattr(codegen, "DEBUG_BOUNDS", True)
    monkeypatch.setattr(codegen_coop, "COOP_PAIR", False)
    monkeypatch.setattr(codegen_rows, "PAIR_LOOPS", False)
    monkeypatch.setattr(codegen, "_GEN_CACHE", {})
    S, X, T = wl.blackscholes_inputs(n=(1 << 12) + 3)
    (x,) = wl.rownorm_inputs(rows=64, cols=4096)
    P, C = wl.kmeans_inputs(n=1 << 12)
    lab, sums, cnt = wl.kmeans_partials(gp, gp.asarray(P), gp.asarray(C))
    a = gp.asarray(np.ones((256, 256), np.float32))
    progs = [list(wl.blackscholes(gp, *map(gp.asarray, (S, X, T)))), list(wl.rownorm(gp, gp.asarray(x))),
             [lab] + sums + [cnt], [a.T + a], [gp.cumsum(a, axis=1)]]
    for roots in progs:
        ks = _source(roots)
        assert "gr::bounds_ok(" in ks.source, ks.family
        runtime.compile_cubin(ks.source)
    tma = _source([gp.cumsum(gp.asarray(np.ones(1 << 21, np.float32)) * 2)])
    assert tma.meta["label"] == "scan-tma" and "gr::bounds_ok(" not in tma.source

