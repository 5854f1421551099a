"""kernel-lowering examples on CPU: iteration spaces, index
maps and the pseudo-C point-program dump.  No GPU needed — lowering is graph
work; compile/run are covered in test_gpu_executor_api.py."""
import numpy as np
import pytest

import paper_1901_03771_b200 as gp
from paper_1901_03771_b200 import lowering, planner
from paper_1901_03771_b200.dag import Graph, Op, OpKind, ReduceOp, ElemCode
from paper_1901_03771_b200.errors import UnsupportedNodeInFusedStep
from paper_1901_03771_b200.tensor import TensorBuffer


def _steps(root):
    return planner.plan(root)


def test_transpose_root_loads_swapped():
    """root Transpose([1,0]) of leaf L: point(i,j) = load L at (j,i)."""
    g = Graph()
    L = g.add_input(TensorBuffer.from_numpy(np.arange(6.0).reshape(2, 3)))
    t = g.add_op(Op(OpKind.TRANSPOSE, attrs=((1, 0),)), [L])
    (st,) = _steps(t)
    k = lowering.lower(st, g)
    assert k.kind == "Map" and k.space.extents == (3, 2) and k.combine is None
    assert k.point.loads == [(L.id, lowering.IndexMap(("i1", "i0")))]
    assert f"load L{L.id}[i1, i0]" in k.point.dump()


def test_broadcast_load_constant_zero():
    """z = x·y, y broadcast along dim 0: load_x(i,j)·load_y(0,j)."""
    g = Graph()
    x = g.add_input(TensorBuffer.from_numpy(np.ones((4, 5))))
    y = g.add_input(TensorBuffer.from_numpy(np.ones((1, 5))))
    z = g.add_op(Op(OpKind.MAP, ElemCode.mul), [x, y])
    (st,) = _steps(z)
    k = lowering.lower(st)
    maps = dict(k.point.loads)
    assert maps[x.id].terms == ("i0", "i1") and maps[y.id].terms == ("0", "i1")
    assert k.point.body[-1].endswith("= mul(ld0, ld1)")


def test_jacobi_interior_select():
    """slice loads become offset maps; SliceAssign becomes select."""
    s = gp.Session()
    a = gp.asarray(np.zeros((66, 66)), session=s)
    b = gp.asarray(np.ones((66, 66)), session=s)
    b[1:-1, 1:-1] = 0.2 * (a[1:-1, 1:-1] + a[1:-1, :-2] + a[1:-1, 2:] + a[:-2, 1:-1] + a[2:, 1:-1])
    (st,) = _steps(b._node)
    k = lowering.lower(st)
    d = k.point.dump()
    assert k.space.extents == (66, 66)
    assert "1 <= i0 < 65 && 1 <= i1 < 65" in d
    terms = sorted(set(m.terms for _, m in k.point.loads))
    # the five-point stencil reads of a and the target-branch read of b
    assert terms == sorted({("i0", "i1"), ("i0", "i1 - 1"), ("i0", "i1 + 1"), ("i0 - 1", "i1"), ("i0 + 1", "i1")})
    assert len(k.point.loads) == 6
    assert "select(" in d


def test_map_reduce_space_is_operand_shape():
    """MapReduce space = shape of the root's operand."""
    g = Graph()
    a = g.add_input(TensorBuffer.from_numpy(np.array([1.0, 2, 3])))
    b = g.add_input(TensorBuffer.from_numpy(np.array([4.0, 5, 6])))
    m = g.add_op(Op(OpKind.MAP, ElemCode.mul), [a, b])
    r = g.add_op(Op(OpKind.REDUCE, attrs=(ReduceOp.sum, (0,), False, None)), [m])
    (st,) = _steps(r)
    k = lowering.lower(st)
    assert k.kind == "MapReduce" and k.space.extents == (3,) and k.combine is ReduceOp.sum
    assert k.reduce_axes == (0,)


def test_reshape_merge_delinearizes():
    s = gp.Session()
    t = gp.asarray(np.zeros((8, 6, 4), np.float32), session=s)
    v = t.transpose(2, 0, 1).reshape(4, 48) * 2
    (st,) = _steps(v._node)
    k = lowering.lower(st)
    (lid, im), = k.point.loads
    # leaf axes (8, 6, 4): axis 0 = i1/6, axis 1 = i1%6, axis 2 = i0
    assert im.terms == ("i1/6", "i1%6", "i0")


def test_row_fused_region_dump_has_fold():
    s = gp.Session()
    x = gp.asarray(np.zeros((4, 8), np.float32), session=s)
    y = x - x.mean(1)[:, None]
    steps = planner.plan_regions([y._node], row_fusion=lambda r, c: True)
    k = lowering.lower(steps[-1])
    assert "fold sum over (r1 < 8)" in k.point.dump()


def test_library_step_is_not_lowered():
    s = gp.Session()
    a = gp.asarray(np.ones((3, 3)), session=s)
    d = gp.dot(a, a)
    steps = _steps(d._node)
    with pytest.raises(ValueError):
        lowering.lower([st for st in steps if st.kind == "Library"][0])


def test_interior_matmul_rejected():
    s = gp.Session()
    a = gp.asarray(np.ones((3, 3)), session=s)
    d = gp.dot(a, a) + 1
    st = planner.PlanStep("Fused", [d._node], [d._node, d._node.preds[0]], [a._node], "Map")
    with pytest.raises(UnsupportedNodeInFusedStep):
        lowering.lower(st)


def test_exec_config_validates():
    from paper_1901_03771_b200.executor import ExecConfig, LibraryCall
    with pytest.raises(ValueError):
        ExecConfig(num_threads=0)
    with pytest.raises(ValueError):
        LibraryCall("Syrk")
