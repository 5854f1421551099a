"""npy v1.0 I/O and DOT dumps on CPU."""
import io
import json
import struct

import numpy as np
import pytest

import paper_1901_03771_b200 as gp
from paper_1901_03771_b200 import bench_cli, npyio
from paper_1901_03771_b200.errors import NpyFormatError


@pytest.fixture
def sess():
    s = gp.Session()
    old = gp.set_default_session(s)
    yield s
    gp.set_default_session(old)


@pytest.mark.parametrize("dt", [np.float32, np.float64, np.int32, np.int64, np.bool_])
@pytest.mark.parametrize("shape", [(), (0,), (7,), (3, 5), (2, 3, 4)])
def test_roundtrip_with_numpy(tmp_path, sess, dt, shape):
    rng = np.random.default_rng(1)
    x = (rng.standard_normal(shape) * 100).astype(dt)
    p = tmp_path / "a.npy"
    npyio.save(p, x)
    # numpy reads what we write, byte for byte the same header format
    y = np.load(p)
    assert y.dtype == x.dtype and y.shape == x.shape and np.array_equal(y, x)
    np.save(tmp_path / "b.npy", x)
    assert (tmp_path / "a.npy").read_bytes() == (tmp_path / "b.npy").read_bytes()
    g = npyio.load(tmp_path / "b.npy")
    assert isinstance(g, gp.ndarray) and g.is_materialized
    assert g.shape == shape and np.dtype(g.dtype) == np.dtype(dt)
    assert np.array_equal(g.node.data.host, x)


def _bytes(x, **kw):
    f = io.BytesIO()
    np.lib.format.write_array(f, x, **kw)
    return f.getvalue()


def test_rejections():
    x = np.arange(6, dtype=np.float32).reshape(2, 3)
    with pytest.raises(NpyFormatError, match="fortran_order"):
        npyio.load(io.BytesIO(_bytes(np.asfortranarray(x))))
    with pytest.raises(NpyFormatError, match="version"):
        npyio.load(io.BytesIO(_bytes(x, version=(2, 0))))
    with pytest.raises(NpyFormatError, match="outside"):
        npyio.load(io.BytesIO(_bytes(x.astype(">f4"))))
    with pytest.raises(NpyFormatError, match="outside"):
        npyio.load(io.BytesIO(_bytes(x.astype(np.uint8))))
    with pytest.raises(NpyFormatError, match="payload"):
        npyio.load(io.BytesIO(_bytes(x)[:-4]))
    with pytest.raises(NpyFormatError, match="trailing"):
        npyio.load(io.BytesIO(_bytes(x) + b"\0"))
    with pytest.raises(NpyFormatError, match="magic"):
        npyio.load(io.BytesIO(b"PK\x03\x04" + b"\0" * 20))
    bad = bytearray(_bytes(np.array([True, False])))
    bad[-1] = 7
    with pytest.raises(NpyFormatError, match="0/1"):
        npyio.load(io.BytesIO(bytes(bad)))
    with pytest.raises(NpyFormatError):
        npyio.save(io.BytesIO(), x.astype(np.uint16))
    with pytest.raises(NpyFormatError):
        npyio.save(io.BytesIO(), x.astype(">f8"))


def test_header_layout():
    f = io.BytesIO()
    npyio.save(f, np.zeros((2, 3), np.float64))
    b = f.getvalue()
    assert b[:8] == b"\x93NUMPY\x01\x00"
    (hlen,) = struct.unpack("<H", b[8:10])
    assert (10 + hlen) % 64 == 0 and b[10 + hlen - 1:10 + hlen] == b"\n"
    assert len(b) == 10 + hlen + 48


def test_dump_dot_dag_and_plan(tmp_path, sess):
    W, a, b = (np.ones(16), np.ones(16) * 2, np.ones(16) * 3)
    gW, ga, gb = gp.asarray(W), gp.asarray(a), gp.asarray(b)
    out = (ga * gW) * (gb * gW) * gW + ga + gb
    dag = gp.dump_dot("dag", tmp_path / "d.dot")
    assert dag.startswith("digraph dag {") and dag.count("->") >= 9
    plan = gp.dump_dot("plan", tmp_path / "p.dot", roots=[out])
    assert plan.count("subgraph cluster_") == 1          # Fig. 1: one fused map
    assert (tmp_path / "p.dot").read_text() == plan
    # pending roots found from the graph when none are given
    assert gp.dump_dot("plan", io.StringIO()).count("subgraph cluster_") == 1


def test_dump_dot_empty_session(tmp_path, sess):
    assert gp.dump_dot("plan", tmp_path / "e.dot") == "digraph plan {\n  compound=true;\n}\n"


def test_cli_dot(tmp_path):
    assert bench_cli.main(["dot", "--target", "plan", "--out", str(tmp_path / "bs.dot"),
                           "--name", "blackscholes", "--size", "1000"]) == 0
    text = (tmp_path / "bs.dot").read_text()
    assert text.count("subgraph cluster_") == 1           # the pricing expression: one kernel
    assert bench_cli.main(["dot", "--target", "dag", "--out", str(tmp_path / "bsd.dot"),
                           "--name", "jacobi", "--size", "64"]) == 0


def test_report_schema_keys():
    assert set(bench_cli.REPORT_KEYS) >= {"engines", "kernels_executed", "library_calls", "max_abs_err", "status"}
    json.dumps({k: None for k in bench_cli.REPORT_KEYS})
