"""Ad-hoc GPU debugging of parity failures (prints, no asserts)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1901_03771_b200 as gp  # noqa: E402
from paper_1901_03771_b200 import codegen  # noqa: E402


def run(fn, x, pair):
    os.environ["GRUMPY_PAIR"] = "1" if pair else "0"
    codegen._GEN_CACHE.clear()
    s = gp.Session()
    return np.asarray(fn(gp.asarray(x, session=s)))


def chain():
    rng = np.random.default_rng(12)
    x = np.concatenate([rng.standard_normal(1 << 16) * 30, rng.uniform(-3, 3, 1 << 16)]).astype(np.float32)
    for name, fn in [("exp*erf", lambda a: gp.exp(a * 0.01) * gp.erf(a)),
                     ("log1", lambda a: gp.log(gp.abs(a) + 1)),
                     ("chain", lambda a: gp.exp(a * 0.01) * gp.erf(a) - gp.log(gp.abs(a) + 1))]:
        p = run(fn, x, True)
        s = run(fn, x, False)
        bad = np.nonzero(~((p == s) | (np.isnan(p) & np.isnan(s))))[0]
        print(name, "mismatches", len(bad))
        for i in bad[:5]:
            print("   x=%r pair=%r scalar=%r" % (x[i], p[i], s[i]))


def views():
    rng = np.random.default_rng(8)
    t = rng.standard_normal((8, 6, 4)).astype(np.float32)
    g1 = np.asarray(gp.asarray(t).transpose(2, 0, 1).reshape(4, 48)[:, ::3] * 2)
    e1 = t.transpose(2, 0, 1).reshape(4, 48)[:, ::3] * 2
    print("transpose-reshape-slice ok", np.array_equal(g1, e1))
    g2 = np.asarray(gp.asarray(t)[::-1, 0, :].T.sum(1))
    e2 = t[::-1, 0, :].T.sum(1)
    print("negstep-T-sum", np.abs(g2 - e2).max(), g2[:3], e2[:3])
    g3 = np.asarray(gp.asarray(t)[::-1, 0, :])
    print("negstep slice ok", np.array_equal(g3, t[::-1, 0, :]))
    g4 = np.asarray(gp.asarray(t)[::-1, 0, :].T)
    print("negstep T ok", np.array_equal(g4, t[::-1, 0, :].T))
    g5 = np.asarray(gp.asarray(t).transpose(2, 0, 1).reshape(4, 48)[:, ::3] * 2 + gp.asarray(t)[::-1, 0, :].T.sum(1)[:, None])
    e5 = e1 + e2[:, None]
    print("combined max err", np.abs(g5 - e5).max())


if __name__ == "__main__":
    chain()
    views()
