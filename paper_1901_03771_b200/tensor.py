"""tensor-core: dtypes, shapes, broadcasting and materialized buffers.

Follows the reference spec module ``tensor-core``:

* ``DType`` — five element types f32, f64, i32, i64, bool8 with byte sizes
  4, 8, 4, 8, 1.
* shapes are tuples of non-negative extents; rank 0 is a scalar (SPEC.md:31-36,
  zero-size dims legal SPEC.md:72).
* ``broadcast_shapes`` — right-aligned rule.
* ``delinearize`` / ``linearize`` — row-major index maps.
* ``TensorBuffer`` — immutable contiguous row-major value.

Dtype promotion deliberately follows NumPy (NEP 50, ufunc loop resolution)
rather than SPEC.md:71's linear order: the B200 build is a drop-in for NumPy
programs, and NumPy promotes i64+f32 to f64 where the spec
says f32.  See DESIGN.md "Semantics".
"""

from __future__ import annotations

import enum
from typing import Sequence, Tuple

import numpy as np

from .errors import BadAxis, IncompatibleShapes, OutOfBounds, UnsupportedDType

Shape = Tuple[int, ...]


class DType(enum.Enum):
    """Element type tag."""

    __hash__ = object.__hash__   # members are singletons: identity hash (recording hot path)

    f32 = "f32"
    f64 = "f64"
    i32 = "i32"
    i64 = "i64"
    bool8 = "bool8"

    @property
    def np(self) -> np.dtype:
        return _TO_NP[self]

    @property
    def itemsize(self) -> int:
        return _ITEMSIZE[self]

    @property
    def ctype(self) -> str:
        """C type name used by the CUDA code generator."""
        return _CTYPE[self]

    @property
    def is_float(self) -> bool:
        return self in (DType.f32, DType.f64)

    @property
    def is_int(self) -> bool:
        return self in (DType.i32, DType.i64)

    @property
    def is_bool(self) -> bool:
        return self is DType.bool8

    def __repr__(self):
        return f"DType.{self.value}"


_TO_NP = {
    DType.f32: np.dtype(np.float32),
    DType.f64: np.dtype(np.float64),
    DType.i32: np.dtype(np.int32),
    DType.i64: np.dtype(np.int64),
    DType.bool8: np.dtype(np.bool_),
}
_FROM_NP = {v: k for k, v in _TO_NP.items()}
_ITEMSIZE = {DType.f32: 4, DType.f64: 8, DType.i32: 4, DType.i64: 8, DType.bool8: 1}
_CTYPE = {
    DType.f32: "float",
    DType.f64: "double",
    DType.i32: "int",
    DType.i64: "long long",
    DType.bool8: "bool",
}


def dtype_of(x) -> DType:
    """Map a NumPy dtype (or anything ``np.dtype`` accepts) to a ``DType``.

    Raises ``UnsupportedDType`` outside the supported set (errors.py:20).
    """
    if isinstance(x, DType):
        return x
    try:
        d = np.dtype(x)
    except TypeError as e:  # pragma: no cover - defensive
        raise UnsupportedDType(str(x)) from e
    try:
        return _FROM_NP[d.newbyteorder("=") if d.byteorder not in "=|" else d]
    except KeyError:
        raise UnsupportedDType(f"dtype {d} is outside f32/f64/i32/i64/bool8") from None


def element_count(shape: Sequence[int]) -> int:
    """Product of extents, 1 for rank 0."""
    n = 1
    for d in shape:
        n *= int(d)
    return n


def broadcast_shapes(a: Sequence[int], b: Sequence[int]) -> Shape:
    """Right-aligned broadcasting.

    >>> broadcast_shapes((1024, 1), (1024,))
    (1024, 1024)
    """
    a = tuple(a)
    b = tuple(b)
    if a == b:
        return a
    n = max(len(a), len(b))
    a2 = (1,) * (n - len(a)) + a
    b2 = (1,) * (n - len(b)) + b
    out = []
    for x, y in zip(a2, b2):
        if x == y or y == 1:
            out.append(x)
        elif x == 1:
            out.append(y)
        else:
            raise IncompatibleShapes(f"shapes {a} and {b} cannot be broadcast together")
    return tuple(out)


def broadcast_many(shapes: Sequence[Sequence[int]]) -> Shape:
    out: Shape = ()
    for s in shapes:
        out = broadcast_shapes(out, s)
    return out


def row_major_strides(shape: Sequence[int]) -> Shape:
    """Element strides of a contiguous row-major buffer."""
    st = []
    acc = 1
    for d in reversed(tuple(shape)):
        st.append(acc)
        acc *= int(d)
    return tuple(reversed(st))


def delinearize(linear: int, shape: Sequence[int]) -> Shape:
    """Row-major coordinates of a linear index.

    >>> delinearize(7, (4, 5))
    (1, 2)
    """
    n = element_count(shape)
    if linear < 0 or linear >= n:
        raise OutOfBounds(f"linear index {linear} outside [0, {n})")
    coords = []
    for d in reversed(tuple(shape)):
        coords.append(linear % d)
        linear //= d
    return tuple(reversed(coords))


def linearize(coords: Sequence[int], shape: Sequence[int]) -> int:
    """Inverse of ``delinearize``."""
    if len(coords) != len(shape):
        raise OutOfBounds(f"coords {tuple(coords)} do not match rank of {tuple(shape)}")
    lin = 0
    for c, d in zip(coords, shape):
        if c < 0 or c >= d:
            raise OutOfBounds(f"coords {tuple(coords)} outside shape {tuple(shape)}")
        lin = lin * d + c
    return lin


def normalize_axis(axis: int, ndim: int) -> int:
    if not isinstance(axis, (int, np.integer)):
        raise BadAxis(f"axis {axis!r} is not an integer")
    a = int(axis)
    if a < -ndim or a >= ndim:
        raise BadAxis(f"axis {axis} is out of bounds for rank {ndim}")
    return a + ndim if a < 0 else a


def normalize_axes(axis, ndim: int) -> Tuple[int, ...]:
    """``None`` → all axes; int or tuple → sorted unique non-negative axes."""
    if axis is None:
        return tuple(range(ndim))
    if isinstance(axis, (tuple, list)):
        out = sorted(normalize_axis(a, ndim) for a in axis)
        if len(set(out)) != len(out):
            raise BadAxis(f"repeated axis in {axis}")
        return tuple(out)
    return (normalize_axis(axis, ndim),)


class TensorBuffer:
    """Materialized n-D value: dtype, shape, contiguous row-major data.

    On the B200 path the authoritative copy is a device allocation from the
    runtime's caching pool (``device``, a ``runtime.DeviceBuffer``); ``host`` is
    an optional NumPy copy kept after the first device→host transfer.  Either
    may be absent but not both.  Immutable once constructed.
    """

    __slots__ = ("dtype", "shape", "device", "host", "__weakref__")

    def __init__(self, dtype: DType, shape: Shape, device=None, host=None):
        if device is None and host is None:
            raise ValueError("TensorBuffer needs device or host data")
        self.dtype = dtype
        self.shape = tuple(int(s) for s in shape)
        self.device = device
        self.host = host
        if host is not None:
            if host.shape != self.shape or dtype_of(host.dtype) is not dtype:
                raise ValueError("host array does not match buffer dtype/shape")
            if not host.flags.c_contiguous:
                raise ValueError("TensorBuffer host data must be C-contiguous")

    @property
    def nbytes(self) -> int:
        return element_count(self.shape) * self.dtype.itemsize

    @classmethod
    def from_numpy(cls, arr) -> "TensorBuffer":
        arr = np.asarray(arr)
        dt = dtype_of(arr.dtype)
        arr = np.asarray(arr, dtype=dt.np, order="C")   # keeps rank 0 (ascontiguousarray would not)
        return cls(dt, arr.shape, host=arr)

    def to_numpy(self) -> np.ndarray:
        """Host view of the value (to_external): one D2H copy
        the first time, then cached."""
        if self.host is None:
            self.host = self.device.to_numpy(self.dtype, self.shape)
        return self.host

    def __repr__(self):
        where = "device" if self.device is not None else "host"
        return f"TensorBuffer({self.dtype.value}, {self.shape}, {where})"
