"""Parity at the BASELINE.json sizes (the sizes bench.py times).

Every config runs at its named shape on one B200 and is checked against the
NumPy program on the same inputs by the chunked full-size checker
(oracle/fullsize.py; tolerances stated there and in SURVEY.md §8(c)).  These
sizes exercise the code paths small tests cannot reach: 2^28-element 64-bit
offsets, the row-normalise total over 65536 row partials, the scan look-back's
slow path (32768 tiles, far more than 512 in flight behind a tile), k-means over
2^26 points and the MLP at batch 65536.
"""

import numpy as np
import pytest

import paper_1901_03771_b200 as gp
from oracle import fullsize, programs

pytestmark = pytest.mark.gpu

wl = programs.load()


def _run(sess, name, prog, expect_kernels=None):
    inp = wl.named_inputs(name)
    dev = [gp.asarray(x) for x in inp]
    outs = prog(dev)
    k0 = sess.stats.kernels_executed
    gp.force(*outs)
    kernels = sess.stats.kernels_executed - k0
    if expect_kernels is not None:
        assert kernels == expect_kernels, (name, kernels)
    got = [np.asarray(o) for o in outs]
    del outs, dev
    return inp, got


def test_listing1_2p24_bitexact(sess):
    inp, got = _run(sess, "listing1", lambda d: [wl.listing1(gp, *d)], expect_kernels=1)
    r = fullsize.check("listing1", inp, got)
    assert r["ok"] and r["mismatches"] == 0, r


@pytest.mark.parametrize("name", ["blackscholes-f32", "blackscholes-f64"])
def test_blackscholes_2p28(sess, name):
    inp, got = _run(sess, name, lambda d: list(wl.blackscholes(gp, *d)), expect_kernels=1)
    r = fullsize.check(name, inp, got)
    assert r["ok"], r


def test_rownorm_65536x4096_y_and_total_bitexact(sess):
    inp, got = _run(sess, "rownorm-y", lambda d: list(wl.rownorm(gp, *d)), expect_kernels=1)
    r = fullsize.check("rownorm-y", inp, got)
    assert r["ok"], r
    assert r["y_bitexact_mismatches"] == 0, r
    assert r["total_bitexact"], r


def test_rownorm_total_only_bitexact(sess):
    inp, got = _run(sess, "rownorm", lambda d: [wl.rownorm(gp, *d)[1]], expect_kernels=1)
    r = fullsize.check("rownorm", inp, got)
    assert r["ok"] and r["total_bitexact"], r


def test_kmeans_2p26_labels_counts_exact(sess):
    def prog(d):
        lab, sums, counts = wl.kmeans_partials(gp, *d)
        return [lab, *sums, counts]
    inp, got = _run(sess, "kmeans", prog, expect_kernels=1)
    r = fullsize.check("kmeans", inp, got)
    assert r["ok"] and r["label_mismatches"] == 0 and r["count_mismatches"] == 0, r


def test_mlp_65536_labels(sess):
    inp, got = _run(sess, "mlp", lambda d: list(wl.mlp(gp, *d)))
    r = fullsize.check("mlp", inp, got)
    assert r["ok"], r
    # no near-ties in the C4 inputs -> labels exact
    assert r["label_mismatches"] == r["near_tie_flips"] == 0, r


def test_cumsum_2p28_f32_lookback_slow_path(sess):
    inp, got = _run(sess, "cumsum", lambda d: [wl.scan(gp, *d)], expect_kernels=1)
    r = fullsize.check("cumsum", inp, got)
    assert r["ok"], r


def test_cumsum_rows_65536x4096_bitexact(sess):
    inp, got = _run(sess, "cumsum-rows", lambda d: [wl.scan_rows(gp, *d)], expect_kernels=1)
    r = fullsize.check("cumsum-rows", inp, got)
    assert r["ok"] and r["mismatches"] == 0, r


def test_cumsum_2p28_int64_exact(sess):
    """Integer prefix sums are exact in any association: any look-back bug at
    32768 tiles (slow path, deep windows) shows as a wrong value."""
    rng = np.random.default_rng(11)
    x = rng.integers(-1000, 1000, 1 << 28, dtype=np.int64)
    got = np.asarray(gp.asarray(x).cumsum())
    ref = np.cumsum(x)
    bad = np.nonzero(got != ref)[0]
    assert len(bad) == 0, (len(bad), bad[:5])


def test_cumsum_2p28_int32_to_int64_exact(sess):
    rng = np.random.default_rng(12)
    x = rng.integers(-(1 << 30), 1 << 30, 1 << 28, dtype=np.int32)
    got = np.asarray((gp.asarray(x) * 3).cumsum())
    assert np.array_equal(got, (x * 3).cumsum())


def test_jacobi_16384_bitexact(sess):
    inp, got = _run(sess, "jacobi", lambda d: [wl.jacobi(gp, *d)], expect_kernels=1)
    r = fullsize.check("jacobi", inp, got)
    assert r["ok"] and r["mismatches"] == 0, r
