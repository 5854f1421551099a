"""npy v1.0 tensor I/O and DOT dumps (§8(f) rank 4).

* ``save(file, arr)`` writes an npy v1.0 file: little-endian, C order, dtypes
  {<f4, <f8, <i4, <i8, |b1} only.  A lazy array is materialised
  first (the store is a materialisation trigger).
* ``load(file)`` reads one back as a device-resident leaf; anything else —
  another format version, fortran_order=True, a big-endian or unlisted dtype,
  a truncated payload — raises ``NpyFormatError`` (errors.py:40).
* ``dump_dot(target, out)`` writes the live DAG ("dag") or the plan of the
  pending roots with one cluster per step ("plan") as Graphviz DOT
  (``Graph.dot`` is the DAG form).
"""

from __future__ import annotations

import ast
import os
import struct
from typing import Optional, Sequence

import numpy as np

from .errors import NpyFormatError

MAGIC = b"\x93NUMPY"
_DESCR = {"<f4": np.float32, "<f8": np.float64, "<i4": np.int32, "<i8": np.int64, "|b1": np.bool_}
_DESCR_OF = {np.dtype(v): k for k, v in _DESCR.items()}


def _header(descr: str, shape) -> bytes:
    h = "{" + f"'descr': '{descr}', 'fortran_order': False, 'shape': {tuple(int(d) for d in shape)!r}, " + "}"
    # v1.0: 10-byte preamble + header, padded with spaces and a final newline
    # to a multiple of 64 bytes (numpy's alignment; v1.0 requires 16)
    total = 10 + len(h) + 1
    pad = (-total) % 64
    h = h + " " * pad + "\n"
    if len(h) > 0xFFFF:
        raise NpyFormatError("header too long for npy v1.0")
    return MAGIC + bytes([1, 0]) + struct.pack("<H", len(h)) + h.encode("latin1")


def save(file, arr) -> None:
    """Write ``arr`` (grumpy or NumPy array) as npy v1.0."""
    host = np.asarray(arr)
    descr = _DESCR_OF.get(host.dtype) if host.dtype.byteorder in ("=", "<", "|") else None
    if descr is None:
        raise NpyFormatError(f"dtype {host.dtype} is outside {{<f4, <f8, <i4, <i8, |b1}}")
    host = host if host.flags.c_contiguous else host.copy(order="C")
    own = not hasattr(file, "write")
    f = open(file, "wb") if own else file
    try:
        f.write(_header(descr, host.shape))
        f.write(host.tobytes(order="C"))
    finally:
        if own:
            f.close()


def read_header(f):
    """(descr, shape, data offset) of an npy v1.0 stream positioned at 0."""
    pre = f.read(10)
    if len(pre) < 10 or pre[:6] != MAGIC:
        raise NpyFormatError("not an npy file (bad magic)")
    if (pre[6], pre[7]) != (1, 0):
        raise NpyFormatError(f"npy version {pre[6]}.{pre[7]}, only 1.0 is accepted")
    (hlen,) = struct.unpack("<H", pre[8:10])
    raw = f.read(hlen)
    if len(raw) != hlen:
        raise NpyFormatError("truncated npy header")
    try:
        d = ast.literal_eval(raw.decode("latin1"))
    except (ValueError, SyntaxError) as e:
        raise NpyFormatError(f"unparsable npy header: {e}") from None
    if not isinstance(d, dict) or set(d) != {"descr", "fortran_order", "shape"}:
        raise NpyFormatError("npy header must hold exactly descr, fortran_order and shape")
    if d["fortran_order"] is not False:
        raise NpyFormatError("fortran_order=True is rejected (SPEC.md:79)")
    if d["descr"] not in _DESCR:
        raise NpyFormatError(f"dtype {d['descr']!r} is outside {{<f4, <f8, <i4, <i8, |b1}}")
    shape = d["shape"]
    if not isinstance(shape, tuple) or any(not isinstance(s, int) or isinstance(s, bool) or s < 0 for s in shape):
        raise NpyFormatError(f"bad shape {shape!r}")
    return d["descr"], shape, 10 + hlen


def load(file, session=None):
    """Read an npy v1.0 file into a device-resident grumpy leaf."""
    from .session import asarray
    own = not hasattr(file, "read")
    f = open(file, "rb") if own else file
    try:
        descr, shape, off = read_header(f)
        dt = np.dtype(_DESCR[descr])
        n = int(np.prod(shape, dtype=np.int64)) if shape else 1
        data = f.read(n * dt.itemsize)
        if len(data) != n * dt.itemsize:
            raise NpyFormatError(f"payload holds {len(data)} bytes, shape {shape} needs {n * dt.itemsize}")
        if f.read(1):
            raise NpyFormatError("trailing bytes after the payload")
    finally:
        if own:
            f.close()
    host = np.frombuffer(data, dtype=dt).reshape(shape)
    if dt == np.bool_ and host.size and np.any(host.view(np.uint8) > 1):
        raise NpyFormatError("|b1 payload holds bytes other than 0/1")
    return asarray(host.copy(), session=session)


def plan_dot(steps) -> str:
    """DOT of a plan: one cluster per step (its nodes), edges from leaves."""
    lines = ["digraph plan {", "  compound=true;"]
    seen = set()
    for i, st in enumerate(steps):
        kind = st.kind if isinstance(st.kind, str) else str(st.kind)
        label = f"step {i}: {kind}" + (f" {st.kernel_kind}" if getattr(st, "kernel_kind", None) else "")
        lines.append(f"  subgraph cluster_{i} {{")
        lines.append(f'    label="{label}";')
        for n in getattr(st, "nodes", ()) or ():
            lines.append(f'    n{n.id} [label="{n.id}: {n.op!r} {list(n.shape)} {n.dtype.value}"];')
            seen.add(n.id)
        lines.append("  }")
    for st in steps:
        for n in getattr(st, "nodes", ()) or ():
            for p in n.preds:
                if p.id not in seen:
                    seen.add(p.id)
                    lines.append(f'  n{p.id} [shape=box,label="{p.id}: leaf {list(p.shape)} {p.dtype.value}"];')
                lines.append(f"  n{p.id} -> n{n.id};")
    lines.append("}")
    return "\n".join(lines) + "\n"


def dump_dot(target: str, out, roots: Optional[Sequence] = None, session=None) -> str:
    """Write the live DAG (target "dag") or the plan of ``roots`` / every
    pending root (target "plan") as DOT to ``out`` (a path or file)."""
    from .session import default_session
    sess = session or default_session()
    if target == "dag":
        text = sess.graph.dot()
    elif target == "plan":
        if roots is None:
            live = [n for n in sess.graph.live_nodes() if not n.is_materialized]
            used = {p.id for n in live for p in n.preds}
            nodes = [n for n in live if n.id not in used]
        else:
            nodes = [getattr(r, "node", r) for r in roots]
        text = plan_dot(sess.plan(nodes) if nodes else [])
    else:
        raise ValueError("target must be 'dag' or 'plan'")
    if hasattr(out, "write"):
        out.write(text)
    else:
        with open(os.fspath(out), "w") as f:
            f.write(text)
    return text
