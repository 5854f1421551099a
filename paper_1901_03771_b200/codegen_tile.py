"""Tile family: map regions that read a leaf transposed (K1 with shared-memory
staging of strided operands).

The reference evaluates index maps point by point (
the paper's transposed predecessors).  On a GPU, a leaf
whose innermost coordinate along the output's fastest axis is not contiguous
(``x.T + y``: output column j reads x[j, i]) turns every warp load into 32
separate sectors.  This family walks the output in TIx32 tiles of its last two
axes (64 rows by default): each staged leaf's tile is loaded with the warp running along the
leaf's own contiguous axis (128-byte coalesced), stored to shared memory,
and read back transposed (rows padded by one element: conflict-free both
ways); every
other leaf and every output move row-wise, coalesced along the output's
contiguous axis.  Points are independent, so results are bit-identical to
the K1 skeleton's.

Staging applies to a leaf access whose offset has coefficient 1 on the
output's second-to-last axis and a coefficient other than 0/1 on its last
axis, with the rest of the offset independent of both (affine index maps:
transposes, slices, broadcasts).  Regions without such a leaf use gr_map.
"""

from __future__ import annotations

import os
from typing import Dict, List, Optional

from .codegen import HEADER, Aff, KernelSource, Region, ValueEmitter, Var, _params_struct
from .dag import OpKind
from .errors import UnsupportedNodeInFusedStep
from .tensor import element_count, row_major_strides

TILE = os.environ.get("GRUMPY_TILE", "1") == "1"
TI = int(os.environ.get("GRUMPY_TILE_TI", "64"))   # output rows per tile (axis -2), one per (warp, r)
TJ = 32          # output columns per tile (axis -1), one per lane
BLOCK = 256      # 8 warps: each thread covers TI / 8 rows of the tile
LEVEL_TILE, LEVEL_ELEM = 1, 2


class TileEmitter(ValueEmitter):
    """Scopes: 0 kernel constants, 1 per tile (batch coordinates), 2 per point."""

    def __init__(self, region: Region, ivar: Var, jvar: Var):
        super().__init__(region)
        self.ivar, self.jvar = ivar, jvar
        self.tile_lines: List[str] = []
        self.elem_lines: List[str] = []
        self.staged: Dict[tuple, tuple] = {}   # key -> (index, leaf, rest Aff, coef on j)

    def emit(self, level, ctype, expr):
        name = self.fresh()
        line = f"const {ctype} {name} = {expr};"
        if level <= 0:
            self.consts.append(line)
        elif level == LEVEL_TILE:
            self.tile_lines.append(line)
        else:
            self.elem_lines.append(line)
        return name

    def derived_var(self, level, expr) -> Var:
        return Var(self.emit(level, "long long", expr), level)

    def load_leaf(self, leaf, off: Aff):
        T = leaf.dtype.ctype
        ptr = f"p.in{self.leaf_index[leaf.id]}"
        ci, cj = off.coef(self.ivar), off.coef(self.jvar)
        rest = off.without(self.ivar).without(self.jvar)
        if ci == 1 and cj not in (0, 1) and rest.level <= LEVEL_TILE:
            key = (leaf.id, rest.key(), cj)
            hit = self.staged.get(key)
            if hit is None:
                hit = self.staged[key] = (len(self.staged), leaf, rest, cj)
            return f"gr_st{hit[0]}[tx][ty + 8 * r]", LEVEL_ELEM
        lvl = max(off.level, 0)
        return self.emit(lvl if lvl > 0 else LEVEL_TILE, T, f"gr::ld<{T}>({ptr} + {off.c()})"), max(lvl, LEVEL_TILE)


def try_generate(region: Region, kname="gr_region") -> Optional[KernelSource]:
    """Tile-family kernel for ``region``, or None when no leaf is read
    transposed (the K1 skeleton is then the right kernel)."""
    if not TILE or any(n.kind is OpKind.SLICE_ASSIGN for n in region.nodes):
        return None
    shape = tuple(region.roots[0].shape)
    if len(shape) < 2 or any(tuple(r.shape) != shape for r in region.roots):
        return None
    I, J = shape[-2], shape[-1]
    if I < 2 or J < 2 or element_count(shape) < 1024:
        return None
    ivar, jvar = Var("i", LEVEL_ELEM), Var("j", LEVEL_ELEM)
    em = TileEmitter(region, ivar, jvar)
    batch = shape[:-2]
    coords: List[Aff] = []
    rest = "bt"
    bcoords: List[Aff] = []
    for d in range(len(batch) - 1, -1, -1):
        ext = batch[d]
        if ext == 1:
            bcoords.append(Aff.of(0))
            continue
        if d == 0:
            bcoords.append(Aff.of(Var(rest, LEVEL_TILE)))
        else:
            c = em.emit(LEVEL_TILE, "long long", f"{rest} % {ext}")
            bcoords.append(Aff.of(Var(c, LEVEL_TILE)))
            rest = em.emit(LEVEL_TILE, "long long", f"{rest} / {ext}")
    bcoords.reverse()
    coords = bcoords + [Aff.of(ivar), Aff.of(jvar)]
    try:
        outs = [em.value(r, coords) for r in region.roots]
    except UnsupportedNodeInFusedStep:
        return None
    if not em.staged:
        return None
    tiles_i, tiles_j = -(-I // TI), -(-J // TJ)
    ntiles = element_count(batch) * tiles_i * tiles_j
    R = TI // (BLOCK // 32)
    lines = ["static __device__ __forceinline__ void tile(const Params& p, const long long t"
             + "".join(f", {l.dtype.ctype} (&gr_st{k})[{TJ}][{TI + 1}]" for k, l, _r, _c in sorted(em.staged.values(),
                                                                                                  key=lambda x: x[0]))
             + ") {",
             "  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;",
             f"  const long long bt = t / {tiles_i * tiles_j}LL, tr = t % {tiles_i * tiles_j}LL;",
             f"  const long long i0 = (tr / {tiles_j}) * {TI}, j0 = (tr % {tiles_j}) * {TJ};",
             "  (void)bt;"]
    lines += ["  " + c for c in em.consts]
    lines += ["  " + l for l in em.tile_lines]
    # load phase: every staged leaf's tile, the warp along the leaf's contiguous axis
    lines.append("#pragma unroll")
    lines.append(f"  for (int r = 0; r < {R}; ++r) {{")
    lines.append(f"    const long long a = tx + {TJ} * (r & {TI // TJ - 1}), b = ty + 8 * (r / {TI // TJ});")
    lines.append(f"    if (i0 + a < {I}LL && j0 + b < {J}LL) {{")
    for k, leaf, rst, cj in sorted(em.staged.values(), key=lambda x: x[0]):
        T = leaf.dtype.ctype
        lines.append(f"      gr_st{k}[b][a] = gr::ld<{T}>(p.in{em.leaf_index[leaf.id]} + ({rst.c()}) + (i0 + a) + "
                     f"{cj}LL * (j0 + b));")
    lines.append("    }")
    lines.append("  }")
    lines.append("  __syncthreads();")
    # compute phase: one point per (warp row, lane), coalesced along j
    lines.append("#pragma unroll")
    lines.append(f"  for (int r = 0; r < {R}; ++r) {{")
    lines.append("    const long long i = i0 + ty + 8 * r, j = j0 + tx;")
    lines.append(f"    if (i < {I}LL && j < {J}LL) {{")
    lines += ["      " + l for l in em.elem_lines]
    st = row_major_strides(shape)
    boff = " + ".join([f"({c.c()}) * {s}LL" for c, s in zip(bcoords, st[:-2])] + ["0LL"])
    for ri, (r, (expr, _lvl)) in enumerate(zip(region.roots, outs)):
        lines.append(f"      gr::st<{r.dtype.ctype}>(p.out{ri} + {boff} + i * {J}LL + j, {expr});")
    lines.append("    }")
    lines.append("  }")
    lines.append("  __syncthreads();")
    lines.append("}")
    params = _params_struct(region)
    smem = "".join(f"  __shared__ {l.dtype.ctype} gr_st{k}[{TJ}][{TI + 1}];\n"
                   for k, l, _r, _c in sorted(em.staged.values(), key=lambda x: x[0]))
    args = "".join(f", gr_st{k}" for k in range(len(em.staged)))
    src = [HEADER, "struct K {", params, f"  static constexpr long long NTILES = {ntiles}LL;",
           "  " + "\n  ".join(lines), "};",
           f'extern "C" __global__ void __launch_bounds__({BLOCK}) {kname}(const K::Params p) {{',
           smem + "  for (long long t = blockIdx.x; t < K::NTILES; t += gridDim.x)",
           f"    K::tile(p, t{args});",
           "}"]
    return KernelSource("tile", "\n".join(src) + "\n", kname,
                        leaf_slots=list(range(len(region.leaves))),
                        root_slots=list(range(len(region.roots))),
                        block=BLOCK, groups=ntiles * BLOCK, vec=1, unroll=1,
                        meta={"shape": shape, "tiles": ntiles, "staged": len(em.staged), "label": "tile-transpose"})
