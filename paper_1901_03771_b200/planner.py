"""fusion-planner: from demanded roots to an ordered list of steps.

Two planners share the step vocabulary:

``plan`` — the reference's Algorithm 1,
implemented faithfully with the spec's resolutions: LIFO worklist
(SPEC.md:263), ``set_materialized`` read as a planning-time flag distinct from
has-data, the multiple-use rule, transpose
absorption into library trans-flags, and the greedy
``max_fused_nodes`` split.  Every step it returns is
executable on the B200 path (Map / MapReduce / MapScan kernels, cuBLAS).

``plan_regions`` — the B200 region pass.  Instead of
cutting at every reduction and materializing every multiply-used node, it
partitions the demand set at the points that *must* be in memory (forced
roots, np.dot operands/results, scans, reductions whose consumers cannot share
their iteration space) and recomputes cheap shared producers inside each
region rather than writing them to HBM.  Regions with the same iteration
space and overlapping inputs are merged into one multi-root kernel
(Black-Scholes call+put), and row-local reductions stay inside the region
that consumes them (row-normalise, softmax).
"""

from __future__ import annotations

import dataclasses
from typing import Dict, List, Optional, Sequence, Set, Tuple

from .dag import ElemCode, Node, OpKind
from .tensor import DType

LIBRARY_KINDS = (OpKind.MATMUL, OpKind.MATVEC)
REDUCTION_KINDS = (OpKind.REDUCE, OpKind.ARGREDUCE)


@dataclasses.dataclass
class PlannerLimits:
    """SPEC.md:199-202; default 100."""

    max_fused_nodes: int = 100

    def __post_init__(self):
        if self.max_fused_nodes < 1:
            raise ValueError("max_fused_nodes must be >= 1")


@dataclasses.dataclass
class PlanStep:
    """One element of Algorithm 1's output list.

    kind: "Fused" or "Library"; kernel_kind: "Map" | "MapReduce" | "MapScan"
    for fused steps; call: "Gemm" | "Gemv" and trans_flags for library steps.
    roots: one for Algorithm 1 steps, several for merged B200 regions.
    """

    kind: str
    roots: List[Node]
    nodes: List[Node]            # interior nodes (roots included), creation order
    leaves: List[Node]           # inputs, in kernel parameter order
    kernel_kind: Optional[str] = None
    call: Optional[str] = None
    trans_flags: Tuple[bool, ...] = ()
    operands: List[Node] = dataclasses.field(default_factory=list)
    order_index: int = 0
    # library steps with a fused cuBLASLt epilogue: the GEMM node (the root is
    # then its bias-add or ReLU consumer) and ("bias" | "relu_bias", bias node)
    library_node: Optional[Node] = None
    epilogue: Optional[Tuple[str, Node]] = None
    # executor-owned memo shared by every instantiation of a cached plan
    # (canonical leaf order, generated kernel source)
    cache: dict = dataclasses.field(default_factory=dict)

    @property
    def root(self) -> Node:
        return self.roots[0]

    def describe(self):
        if self.kind == "Library":
            return (f"Library({self.call}, trans={self.trans_flags}, root={self.root.id}, "
                    f"leaves={sorted(l.id for l in self.leaves)})")
        return (f"Fused({self.kernel_kind}, roots={[r.id for r in self.roots]}, "
                f"leaves={sorted(l.id for l in self.leaves)})")


# ---------------------------------------------------------------------------
# Demand traversal and the two predicates
# ---------------------------------------------------------------------------


def demand_set(root: Node, g=None) -> Set[Node]:
    """Nodes reachable backward from root without crossing materialized nodes;
    materialized frontier nodes are included as leaves."""
    seen = {}
    stack = [root]
    while stack:
        n = stack.pop()
        if n.id in seen:
            continue
        seen[n.id] = n
        if n.is_materialized:
            continue
        stack.extend(n.preds)
    return set(seen.values())


def materialize_node(n: Node) -> bool:
    """True iff n is Reduce/Scan/MatMul/MatVec."""
    return n.kind in (OpKind.REDUCE, OpKind.ARGREDUCE, OpKind.SCAN, OpKind.KEYED_SUM) + LIBRARY_KINDS


def _absorbable_transpose(p: Node) -> bool:
    """Rank-2 [1,0] transpose feeding a library op."""
    return (p.kind is OpKind.TRANSPOSE and len(p.shape) == 2 and tuple(p.op.attrs[0]) == (1, 0)
            and not p.is_materialized)


def materialize_pred_of_node(n: Node, p: Node) -> bool:
    """True iff n is a library op, except absorbable transposes."""
    if n.kind not in LIBRARY_KINDS:
        return False
    return not _absorbable_transpose(p)


def library_operands(n: Node):
    """(operand nodes after transpose absorption, trans flags, call name)."""
    ops = []
    flags = []
    for p in n.preds:
        if _absorbable_transpose(p):
            ops.append(p.preds[0])
            flags.append(True)
        else:
            ops.append(p)
            flags.append(False)
    call = "Gemm" if n.kind is OpKind.MATMUL else "Gemv"
    return ops, tuple(flags), call


def _kernel_kind(root: Node) -> str:
    if root.kind is OpKind.SCAN:
        return "MapScan"
    if root.kind in REDUCTION_KINDS or root.kind in (OpKind.KEYED_SUM, OpKind.MATMUL):
        return "MapReduce"
    return "Map"


# ---------------------------------------------------------------------------
# Algorithm 1
# ---------------------------------------------------------------------------


class _A1:
    def __init__(self):
        self.graph_list: List[dict] = []
        self.planned: Set[int] = set()   # set_materialized() planning flag

    def create_subgraph(self, root: Node, visited: Set[int]):
        """Algorithm 1, LIFO worklist."""
        if root.is_materialized or root.id in self.planned:
            return
        new_nodes: Dict[int, Node] = {}
        edges = []
        candidates: List[Node] = []
        visited.add(root.id)
        self.planned.add(root.id)
        candidates.append(root)
        trans = ()
        operands: List[Node] = []
        while candidates:
            node = candidates.pop()
            new_nodes[node.id] = node
            if node.is_materialized:
                continue
            if node is not root and materialize_node(node):
                # becomes its own subgraph; a leaf here
                self.create_subgraph(node, visited)
                continue
            if node is not root and node.id in self.planned:
                continue
            if node.kind in LIBRARY_KINDS:
                operands, trans, _ = library_operands(node)
            for pred in node.preds:
                if node.kind in LIBRARY_KINDS and _absorbable_transpose(pred):
                    # transpose absorption: demand the transpose's operand
                    src = pred.preds[0]
                    if not src.is_materialized:
                        self.create_subgraph(src, visited)
                    new_nodes[src.id] = src
                    edges.append((node.id, src.id))
                    continue
                if pred.id not in visited:
                    if materialize_pred_of_node(node, pred):
                        self.create_subgraph(pred, visited)
                        new_nodes[pred.id] = pred
                    elif not pred.is_materialized:
                        visited.add(pred.id)
                        candidates.append(pred)
                    else:
                        new_nodes[pred.id] = pred
                elif pred.id not in new_nodes:
                    # multiple-use rule
                    if not pred.is_materialized and pred.id not in self.planned:
                        self.create_subgraph(pred, set())
                    new_nodes[pred.id] = pred
                edges.append((node.id, pred.id))
        self.graph_list.append({"root": root, "nodes": new_nodes, "trans": trans, "operands": operands})


def _finalize(root: Node, nodes: Dict[int, Node], planned: Set[int]):
    """Interior = nodes reachable from root without crossing materialized or
    planned-elsewhere nodes; those become leaves (in first-visit order)."""
    interior: Dict[int, Node] = {}
    leaves: Dict[int, Node] = {}
    stack = [root]
    while stack:
        n = stack.pop()
        if n.id in interior or n.id in leaves:
            continue
        if n is not root and (n.is_materialized or n.id in planned):
            leaves[n.id] = n
            continue
        interior[n.id] = n
        if n.kind in LIBRARY_KINDS:
            ops, _, _ = library_operands(n)
            for p in reversed(ops):
                stack.append(p)
        else:
            for p in reversed(n.preds):
                stack.append(p)
    return sorted(interior.values(), key=lambda x: x.id), list(leaves.values())


def _height(n: Node, interior_ids: Set[int], memo: Dict[int, int]) -> int:
    if n.id in memo:
        return memo[n.id]
    h = 0
    for p in n.preds:
        if p.id in interior_ids:
            h = max(h, 1 + _height(p, interior_ids, memo))
    memo[n.id] = h
    return h


def _cone_size(n: Node, interior_ids: Set[int]) -> int:
    seen = set()
    stack = [n]
    while stack:
        x = stack.pop()
        if x.id in seen or x.id not in interior_ids:
            continue
        seen.add(x.id)
        stack.extend(x.preds)
    return len(seen)


def plan(root: Node, g=None, limits: Optional[PlannerLimits] = None) -> List[PlanStep]:
    """Ordered Algorithm 1 plan for ``root``."""
    limits = limits or PlannerLimits()
    if root.is_materialized:
        return []
    extra_planned: Set[int] = set()
    while True:
        a1 = _A1()
        steps = _run_a1(a1, root, extra_planned)
        too_big = None
        for st in steps:
            if st.kind == "Fused" and len(st.nodes) > limits.max_fused_nodes:
                too_big = st
                break
        if too_big is None:
            for i, st in enumerate(steps):
                st.order_index = i
            return steps
        ids = {n.id for n in too_big.nodes}
        memo: Dict[int, int] = {}
        best = None
        for n in too_big.nodes:
            if n is too_big.root:
                continue
            if _cone_size(n, ids) > limits.max_fused_nodes:
                continue
            key = (-_height(n, ids, memo), n.id)
            if best is None or key < best[0]:
                best = (key, n)
        if best is None:  # every interior cone is too large: split just below the root
            best = (None, max((n for n in too_big.nodes if n is not too_big.root), key=lambda x: x.id))
        extra_planned.add(best[1].id)


def _run_a1(a1: _A1, root: Node, split_points: Set[int]) -> List[PlanStep]:
    # split points are planned as their own subgraphs before the root
    for nid in sorted(split_points):
        n = _find(root, nid)
        if n is not None and not n.is_materialized:
            a1.create_subgraph(n, set())
    a1.create_subgraph(root, set())
    steps = []
    for gph in a1.graph_list:
        r = gph["root"]
        nodes, leaves = _finalize(r, gph["nodes"], a1.planned)
        if r.kind in LIBRARY_KINDS:
            ops, trans, call = library_operands(r)
            steps.append(PlanStep("Library", [r], nodes, leaves, call=call, trans_flags=trans, operands=ops))
        else:
            steps.append(PlanStep("Fused", [r], nodes, leaves, kernel_kind=_kernel_kind(r)))
    return steps


def _find(root: Node, nid: int) -> Optional[Node]:
    stack = [root]
    seen = set()
    while stack:
        n = stack.pop()
        if n.id == nid:
            return n
        if n.id in seen:
            continue
        seen.add(n.id)
        stack.extend(n.preds)
    return None


# ---------------------------------------------------------------------------
# B200 region pass
# ---------------------------------------------------------------------------


def _is_view(n: Node) -> bool:
    return n.kind in (OpKind.TRANSPOSE, OpKind.RESHAPE, OpKind.SLICE, OpKind.BROADCAST)


_VIEW_KINDS = (OpKind.SLICE, OpKind.RESHAPE, OpKind.TRANSPOSE, OpKind.BROADCAST)


def _stencil_read(n: Node, consumers) -> bool:
    """Is ``n`` read through two or more distinct slices?"""
    views = {repr(c.op.attrs) for c in consumers.get(n.id, ()) if c.kind is OpKind.SLICE}
    return len(views) >= 2


def _gemm_epilogue(n: Node, consumers, root_ids):
    """(last node, [chain], bias, kind) when the f32 GEMM ``n`` feeds exactly
    one ``+ bias[N]`` (optionally then exactly one ``maximum(., 0)``): the
    pattern a cuBLASLt BIAS / RELU_BIAS epilogue computes in the GEMM."""
    if (n.kind is not OpKind.MATMUL or n.dtype is not DType.f32 or n.id in root_ids
            or 0 in n.shape or 0 in n.preds[0].shape):
        return None
    cons = consumers.get(n.id, [])
    if len(cons) != 1:
        return None
    a = cons[0]
    if not (a.kind is OpKind.MAP and a.op.code is ElemCode.add and len(a.preds) == 2 and a.dtype is DType.f32
            and a.shape == n.shape):
        return None
    bias = a.preds[1] if a.preds[0] is n else a.preds[0] if a.preds[1] is n else None
    N = n.shape[1]
    if bias is None or bias is n or bias.dtype is not DType.f32 or tuple(bias.shape) not in ((N,), (1, N)):
        return None
    cons = consumers.get(a.id, [])
    if a.id not in root_ids and len(cons) == 1:
        r = cons[0]
        z = r.preds[1] if len(r.preds) == 2 and r.preds[0] is a else None
        if (r.kind is OpKind.MAP and r.op.code is ElemCode.maximum and z is not None and z.shape == ()
                and z.op.code is ElemCode.const_splat and z.op.attrs and z.op.attrs[0] == 0 and r.dtype is DType.f32):
            return r, [a, r], bias, "relu_bias"
    return a, [a], bias, "bias"


def plan_regions(roots: Sequence[Node], row_fusion=None, check=None, epilogues: bool = False,
                 skinny=None) -> List[PlanStep]:
    """B200 region planner (module docstring).

    ``row_fusion(reduction, consumer)`` proposes keeping a reduction inside its
    consumer's kernel (None: every reduction is its own step).  ``skinny(n)``
    proposes computing a small-N product inside its consumers' row kernel
    instead of a library step (the code generator may still refuse it).  ``check(step)``
    is the code generator's verdict; when it raises an exception carrying
    ``.node`` that node becomes a materialization point and planning repeats.
    """
    extra: Set[int] = set()
    solo: Set[int] = set()
    for _ in range(256):
        steps = _plan_once(roots, row_fusion, extra, check, solo, epilogues, skinny)
        if check is None:
            return steps
        bad = None
        for st in steps:
            if st.kind != "Fused":
                continue
            try:
                check(st)
            except Exception as e:  # NotFusable
                node = getattr(e, "node", None)
                root_ids = {r.id for r in st.roots}
                if node is None:
                    raise
                if node.id in root_ids:
                    if len(st.roots) == 1 or node.id in solo:
                        raise
                    bad = ("solo", node)      # a root that cannot share this kernel
                elif node.id in extra:
                    raise
                else:
                    bad = ("cut", node)       # an interior node: materialize it
                break
        if bad is None:
            return steps
        (solo if bad[0] == "solo" else extra).add(bad[1].id)
    raise RuntimeError("region planning did not converge")


def _plan_once(roots: Sequence[Node], row_fusion, extra: Set[int], check, solo=frozenset(),
               epilogues: bool = False, skinny=None) -> List[PlanStep]:
    roots = [r for r in dict((r.id, r) for r in roots).values() if not r.is_materialized]
    if not roots:
        return []
    # 1. demand set
    demand: Dict[int, Node] = {}
    stack = list(roots)
    while stack:
        n = stack.pop()
        if n.id in demand:
            continue
        demand[n.id] = n
        if not n.is_materialized:
            stack.extend(n.preds)
    consumers: Dict[int, List[Node]] = {}
    for n in demand.values():
        if n.is_materialized:
            continue
        for p in n.preds:
            consumers.setdefault(p.id, []).append(n)

    # 2. points that must be in memory
    points: Dict[int, Node] = {r.id: r for r in roots}
    root_ids = set(points)
    epi: Dict[int, tuple] = {}          # epilogue root id -> (gemm, chain, bias, kind)
    absorbed: Set[int] = set()
    def is_skinny(n):
        return skinny is not None and n.id not in extra and not n.is_materialized and skinny(n)

    if epilogues:
        for n in demand.values():
            if not n.is_materialized and n.id not in extra and not is_skinny(n):
                e = _gemm_epilogue(n, consumers, root_ids)
                if e is not None and not any(c.id in extra for c in e[1][:-1]):
                    epi[e[0].id] = (n,) + e[1:]
                    absorbed.update([n.id] + [c.id for c in e[1][:-1]])
    for n in demand.values():
        if n.is_materialized:
            continue
        if n.id in epi:
            g = epi[n.id][0]
            points[n.id] = n
            ops, _, _ = library_operands(g)
            for p in ops + [epi[n.id][2]]:
                if not p.is_materialized:
                    points[p.id] = p
            continue
        if n.id in absorbed:
            continue
        if n.kind in LIBRARY_KINDS:
            # operands of a product are in memory (library call or TMA stream)
            ops, _, _ = library_operands(n) if not is_skinny(n) else (list(n.preds), None, None)
            for p in ops:
                if not p.is_materialized:
                    points[p.id] = p
        if n.id in extra:
            points[n.id] = n
            continue
        if n.kind not in _VIEW_KINDS and _stencil_read(n, consumers):
            # read through two or more different slices (a stencil over a
            # computed grid: Jacobi sweep k+1 over sweep k): recomputing it
            # per read multiplies with every chained sweep, so it is
            # materialized — one kernel per sweep
            points[n.id] = n
        if n.kind in LIBRARY_KINDS:
            if not is_skinny(n):
                points[n.id] = n
        elif n.kind in (OpKind.SCAN, OpKind.KEYED_SUM):
            points[n.id] = n
        elif n.kind in REDUCTION_KINDS:
            cons = consumers.get(n.id, [])
            if not cons:
                points[n.id] = n
            elif row_fusion is None or not all(row_fusion(n, c) for c in cons):
                points[n.id] = n

    # 3. one cone per point
    cones = []
    for pid in sorted(points):
        p = points[pid]
        if pid in epi:
            g, chain, bias, kind = epi[pid]
            ops, trans, call = library_operands(g)
            st = PlanStep("Library", [p], [g] + chain, list(dict((o.id, o) for o in ops + [bias]).values()),
                          call=call, trans_flags=trans, operands=ops)
            st.library_node = g
            st.epilogue = (kind, bias)
            cones.append(st)
            continue
        if p.kind in LIBRARY_KINDS and not is_skinny(p):
            ops, trans, call = library_operands(p)
            cones.append(PlanStep("Library", [p], [p], [o for o in ops], call=call, trans_flags=trans, operands=ops))
            continue
        interior: Dict[int, Node] = {}
        leaves: Dict[int, Node] = {}
        st = [p]
        while st:
            n = st.pop()
            if n.id in interior or n.id in leaves:
                continue
            if n is not p and (n.is_materialized or n.id in points):
                leaves[n.id] = n
                continue
            interior[n.id] = n
            for q in reversed(n.preds):
                st.append(q)
        cones.append(PlanStep("Fused", [p], sorted(interior.values(), key=lambda x: x.id),
                              list(leaves.values()), kernel_kind=_kernel_kind(p)))

    # 4. merge map cones with the same iteration space that share inputs or interior
    merged: List[PlanStep] = []
    for c in cones:
        if c.kind == "Fused" and c.kernel_kind == "Map" and c.root.id not in solo:
            for m in merged:
                if (m.kind == "Fused" and m.kernel_kind == "Map" and m.root.shape == c.root.shape
                        and not any(r.id in solo for r in m.roots)
                        and _shares(m, c) and not _depends(m, c) and not _depends(c, m)
                        and not _cyclic([s for s in merged if s is not m] + [_merged_copy(m, c)]
                                        + [s for s in cones if s is not c and s not in merged])):
                    _merge_into(m, c)
                    break
            else:
                merged.append(c)
        else:
            merged.append(c)
    # 4b. fold a reduction step into the step producing its operand (y and
    # y.sum() in one kernel), or fuse cones sharing inputs with a reduction
    # step; each candidate merge is kept only if the code generator accepts it
    if check is not None:
        changed = True
        while changed:
            changed = False
            for a in list(merged):
                if a.kind != "Fused" or a.kernel_kind != "MapReduce" or any(r.id in solo for r in a.roots):
                    continue
                for b in merged:
                    if b is a or b.kind != "Fused" or any(r.id in solo for r in b.roots):
                        continue
                    if not (_depends(a, b) or (_shares(a, b) and not _depends(b, a))):
                        continue
                    if _depends(b, a):
                        continue
                    trial = _merged_copy(b, a)
                    others = [s for s in merged if s is not a and s is not b]
                    if _cyclic(others + [trial]):
                        continue
                    try:
                        check(trial)
                    except Exception:
                        continue
                    b.roots, b.nodes, b.leaves, b.kernel_kind = trial.roots, trial.nodes, trial.leaves, trial.kernel_kind
                    merged.remove(a)
                    changed = True
                    break
                if changed:
                    break

    # 5. topological order over steps
    produced = {}
    for i, s in enumerate(merged):
        for r in s.roots:
            produced[r.id] = i
    order: List[int] = []
    state: Dict[int, int] = {}

    def visit(i):
        if state.get(i) == 2:
            return
        state[i] = 1
        for l in merged[i].leaves:
            j = produced.get(l.id)
            if j is not None and j != i and state.get(j) != 2:
                visit(j)
        state[i] = 2
        order.append(i)

    for i in range(len(merged)):
        visit(i)
    out = [merged[i] for i in order]
    for i, s in enumerate(out):
        s.order_index = i
    return out


def _cyclic(steps: List[PlanStep]) -> bool:
    """True if the steps' leaf -> producing-step dependencies contain a cycle."""
    produced = {}
    for i, s in enumerate(steps):
        for r in s.roots:
            produced[r.id] = i
    deps = [{produced[l.id] for l in s.leaves if l.id in produced and produced[l.id] != i}
            for i, s in enumerate(steps)]
    state = [0] * len(steps)
    for start in range(len(steps)):
        if state[start]:
            continue
        stack = [(start, iter(deps[start]))]
        state[start] = 1
        while stack:
            i, it = stack[-1]
            j = next(it, None)
            if j is None:
                state[i] = 2
                stack.pop()
            elif state[j] == 1:
                return True
            elif state[j] == 0:
                state[j] = 1
                stack.append((j, iter(deps[j])))
    return False


def _shares(a: PlanStep, b: PlanStep) -> bool:
    ia = {n.id for n in a.nodes} | {n.id for n in a.leaves}
    return any(n.id in ia for n in b.nodes) or any(n.id in ia for n in b.leaves)


def _depends(a: PlanStep, b: PlanStep) -> bool:
    """True if a reads any root of b."""
    rb = {r.id for r in b.roots}
    return any(l.id in rb for l in a.leaves)


def _merged_copy(b: PlanStep, a: PlanStep) -> PlanStep:
    """b ∪ a where a may read b's roots (they become interior)."""
    broots = {r.id for r in b.roots}
    ids = {n.id for n in b.nodes}
    nodes = sorted(b.nodes + [n for n in a.nodes if n.id not in ids], key=lambda x: x.id)
    nids = {n.id for n in nodes}
    leaves = [l for l in b.leaves]
    lids = {l.id for l in leaves}
    for l in a.leaves:
        if l.id not in lids and l.id not in broots and l.id not in nids:
            leaves.append(l)
            lids.add(l.id)
    kind = "MapReduce" if "MapReduce" in (a.kernel_kind, b.kernel_kind) else b.kernel_kind
    return PlanStep("Fused", b.roots + a.roots, nodes, leaves, kernel_kind=kind)


def _merge_into(m: PlanStep, c: PlanStep):
    m.roots = m.roots + c.roots
    ids = {n.id for n in m.nodes}
    m.nodes = sorted(m.nodes + [n for n in c.nodes if n.id not in ids], key=lambda x: x.id)
    lids = {n.id for n in m.leaves}
    m.leaves = m.leaves + [l for l in c.leaves if l.id not in lids]


# ---------------------------------------------------------------------------
# Plan cache: structural DAG signatures and step templates
# ---------------------------------------------------------------------------


def dag_signature(roots: Sequence[Node]):
    """Structural key of the demanded DAG plus its nodes in visit order.

    Materialized nodes are leaves keyed by (shape, dtype) only, so a loop that
    rebuilds the same expression on fresh inputs hits the same key; node
    identity inside the DAG (sharing) is captured by local indices."""
    local: Dict[int, int] = {}
    order: List[Node] = []
    items = []
    for r in roots:
        if r.id in local:
            continue
        stack = [r]
        while stack:
            n = stack[-1]
            nid = n.id
            if nid in local:
                stack.pop()
                continue
            if n.data is not None:
                stack.pop()
                local[nid] = len(order)
                order.append(n)
                items.append(("L", n.shape, n.dtype))
                continue
            pending = [p for p in n.preds if p.id not in local]
            if pending:
                stack.extend(reversed(pending))
                continue
            stack.pop()
            local[nid] = len(order)
            order.append(n)
            items.append((n.op, n.shape, n.dtype, tuple([local[p.id] for p in n.preds])))
    return (tuple(items), tuple([local[r.id] for r in roots])), order


def make_template(steps: List[PlanStep], order: List[Node]):
    idx = {n.id: i for i, n in enumerate(order)}
    tmpl = []
    for st in steps:
        tmpl.append({
            "kind": st.kind, "kernel_kind": st.kernel_kind, "call": st.call,
            "trans_flags": st.trans_flags,
            "roots": [idx[n.id] for n in st.roots],
            "nodes": [idx[n.id] for n in st.nodes],
            "leaves": [idx[n.id] for n in st.leaves],
            "operands": [idx[n.id] for n in st.operands],
            "library_node": idx[st.library_node.id] if st.library_node is not None else None,
            "epilogue": (st.epilogue[0], idx[st.epilogue[1].id]) if st.epilogue else None,
            "cache": st.cache,
        })
    return tmpl


def instantiate(tmpl, order: List[Node]) -> List[PlanStep]:
    steps = []
    for i, t in enumerate(tmpl):
        st = PlanStep(t["kind"], [order[j] for j in t["roots"]], [order[j] for j in t["nodes"]],
                      [order[j] for j in t["leaves"]], kernel_kind=t["kernel_kind"], call=t["call"],
                      trans_flags=t["trans_flags"], operands=[order[j] for j in t["operands"]], order_index=i)
        if t.get("library_node") is not None:
            st.library_node = order[t["library_node"]]
        if t.get("epilogue"):
            st.epilogue = (t["epilogue"][0], order[t["epilogue"][1]])
        st.cache = t["cache"]
        steps.append(st)
    return steps
