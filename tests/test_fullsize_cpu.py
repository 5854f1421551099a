"""The full-size parity checker (oracle/fullsize.py) and the standalone program
loader (oracle/programs.py) on CPU: NumPy's own outputs pass, perturbed ones
fail, and loading the programs never maps the native shim."""

import subprocess
import sys

import numpy as np
import pytest

from oracle import fullsize, programs

wl = programs.load()

SMALL = {"listing1": 1 << 14, "blackscholes-f32": 1 << 14, "blackscholes-f64": 1 << 14, "rownorm": 256,
         "rownorm-y": 256, "mlp": 512, "kmeans": 1 << 14, "cumsum": 1 << 16, "cumsum-rows": 64, "jacobi": 64}


def _outputs(name, inp):
    if name == "listing1":
        return [wl.listing1(np, *inp)]
    if name.startswith("blackscholes"):
        return list(wl.blackscholes(np, *inp))
    if name == "rownorm":
        return [np.asarray(wl.rownorm(np, *inp)[1])]
    if name == "rownorm-y":
        y, t = wl.rownorm(np, *inp)
        return [y, np.asarray(t)]
    if name == "mlp":
        return list(wl.mlp(np, *inp))
    if name == "kmeans":
        lab, sums, counts = wl.kmeans_partials(np, *inp)
        return [lab, *sums, counts]
    if name == "cumsum":
        return [wl.scan(np, *inp)]
    if name == "cumsum-rows":
        return [wl.scan_rows(np, *inp)]
    if name == "jacobi":
        a = inp[0]
        return [wl.jacobi(np, a)]
    raise KeyError(name)


def _inputs(name):
    if name == "jacobi":
        return [np.random.default_rng(3).random((SMALL[name], SMALL[name]), dtype=np.float32)]
    return wl.named_inputs(name, 0, SMALL[name])


@pytest.mark.parametrize("name", sorted(SMALL))
def test_numpy_outputs_pass(name):
    inp = _inputs(name)
    # NumPy's cumsum is one sequential chain: bound it as a chain of 1-element tiles
    kw = {"tile": 1} if name == "cumsum" else {}
    r = fullsize.check(name, inp, _outputs(name, inp), threads=4, **kw)
    assert r["ok"], r
    if name in ("listing1", "jacobi", "kmeans", "cumsum-rows"):
        assert r["mismatches"] == 0
    if name.startswith("rownorm"):
        assert r["total_bitexact"], r


@pytest.mark.parametrize("name", ["listing1", "blackscholes-f32", "rownorm-y", "kmeans", "cumsum", "cumsum-rows", "mlp"])
def test_perturbed_outputs_fail(name):
    inp = _inputs(name)
    out = [np.array(o, copy=True) for o in _outputs(name, inp)]
    o = out[0]
    if o.dtype.kind == "f":
        o.reshape(-1)[o.size // 2] += np.abs(o.reshape(-1)[o.size // 2]) * 1e-2 + 1.0
    else:
        o.reshape(-1)[o.size // 2] = (o.reshape(-1)[o.size // 2] + 1) % 10
    r = fullsize.check(name, inp, out, threads=4)
    assert not r["ok"], r


def test_named_inputs_are_shard_consistent():
    full = wl.named_inputs("kmeans", 0, 1 << 21)
    part = wl.named_inputs("kmeans", 3 << 19, 1 << 21)
    assert np.array_equal(full[0][3 << 19:], part[0])
    assert np.array_equal(full[1], part[1])


def test_total_tree_matches_numpy_sum():
    x = wl.named_inputs("rownorm", 0, 512)[0]
    y, t = wl.rownorm(np, x)
    r = fullsize.check("rownorm", [x], [np.asarray(t)], threads=8)
    assert r["total_bitexact"] and r["total"] == float(t)


def test_programs_loader_does_not_map_the_shim():
    code = ("import sys; sys.path.insert(0, '.'); from oracle import programs; wl = programs.load(); "
            "import numpy as np; wl.blackscholes(np, *wl.named_inputs('blackscholes-f32', 0, 1024)); "
            "assert 'paper_1901_03771_b200' not in sys.modules; assert not programs.native_shim_mapped(); print('ok')")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                         cwd=fullsize.__file__.rsplit("/oracle/", 1)[0])
    assert out.stdout.strip() == "ok", out.stderr


def test_transpose_checker():
    rng = np.random.default_rng(1)
    x = rng.random((300, 300), dtype=np.float32)
    y = rng.random((300, 300), dtype=np.float32)
    out = x.T + y
    assert fullsize.check("transpose", [x, y], [out], threads=4)["ok"]
    out[5, 7] += 1
    assert not fullsize.check("transpose", [x, y], [out], threads=4)["ok"]
