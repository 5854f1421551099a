"""Randomised programs on CPU:

* recorder vs NumPy: every seed recorded through grumpy and evaluated by the
  eager oracle over the recorded DAG equals the same program run directly in
  NumPy — bit for bit (equal_nan), so a recorder bug cannot hide behind an
  oracle that reads the same DAG;
* plan simulator over every randomized program, for the
  B200 region pass (with the code generator's verdict) and for Algorithm 1.
"""
import os

import numpy as np
import pytest

import paper_1901_03771_b200 as gp
from paper_1901_03771_b200 import codegen, codegen_rows, planner
from oracle import eager
from random_programs import GP, Numpy, make_program
from test_planner import simulate

NPROG = int(os.environ.get("GRUMPY_RANDOM_PROGRAMS_CPU", "1000"))


@pytest.fixture
def fresh():
    s = gp.Session()
    old = gp.set_default_session(s)
    yield s
    gp.set_default_session(old)


def _same(a, b):
    a, b = np.asarray(a), np.asarray(b)
    if a.shape != b.shape or a.dtype != b.dtype:
        return False
    return np.array_equal(a, b, equal_nan=a.dtype.kind == "f")


@pytest.mark.parametrize("chunk", range(10))
def test_recorder_matches_numpy(fresh, chunk):
    bad = []
    for seed in range(chunk, NPROG, 10):
        outs, inexact, depth = make_program(seed, GP())
        ref, _t2, _d2 = make_program(seed, Numpy())
        mag, _t3, _d3 = make_program(seed, Numpy(absolute=True))
        assert len(outs) == len(ref), seed
        for o, r, m in zip(outs, ref, mag):
            e = eager.evaluate(o.node)
            r = np.asarray(r)
            if _same(e, r):
                continue
            if inexact and e.dtype.kind == "f" and e.shape == r.shape and e.dtype == r.dtype:
                # reassociated (a reduction over a strided view: NumPy walks
                # memory order, which depends on the intermediates' layouts)
                eps = 2.0 ** -24 if e.dtype == np.float32 else 2.0 ** -53
                fin = np.isfinite(r)
                if (np.array_equal(np.isnan(e), np.isnan(r)) and np.array_equal(e[~fin & ~np.isnan(r)], r[~fin & ~np.isnan(r)])
                        and np.all(np.abs(e[fin] - r[fin]) <= 64 * (depth + 2) * eps * np.abs(np.asarray(m, np.float64)[fin]))):
                    continue
            bad.append((seed, o.node, e.dtype, r.dtype))
    assert not bad, bad[:5]


@pytest.mark.parametrize("chunk", range(10))
def test_plan_simulator_random_programs(fresh, chunk):
    for seed in range(chunk, NPROG, 10):
        outs, _t, _d = make_program(seed, GP())
        roots = [o.node for o in outs]
        steps = planner.plan_regions(roots, row_fusion=codegen.row_fusable, check=codegen.check_step,
                                     epilogues=True, skinny=codegen_rows.skinny_ok)
        simulate(steps, roots)
        for st in steps:
            if st.kind == "Fused":
                # every interior node of a fused step is unmaterialized and is
                # not one of its leaves (leaves-only invariant)
                assert all(not n.is_materialized for n in st.nodes), seed
        # Algorithm 1 per root, in force order (the session's algorithm1
        # planner): nodes planned for an earlier root are leaves of later ones
        a1, seen = [], set()
        for r in roots:
            for st in planner.plan(r, fresh.graph):
                if st.root.id not in seen:
                    a1.append(st)
                    seen.add(st.root.id)
        simulate(a1, roots)
