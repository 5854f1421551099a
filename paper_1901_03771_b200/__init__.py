"""grumpy on B200 — lazy NumPy-subset arrays fused into sm_100a kernels.

Drop-in module in the sense of the paper: ``import
paper_1901_03771_b200 as grumpy`` (or the top-level ``grumpy`` alias) and use
it where a program used ``numpy``.  Operations record a DAG; printing,
``tolist``, ``np.asarray`` or storing forces the pending region, which runs as
one generated CUDA kernel per region (np.dot goes to cuBLAS).

Layout of the package (reference module in brackets, /root/reference/SPEC.md):
  tensor.py     [tensor-core]        dtypes, shapes, broadcasting, buffers
  dag.py        [expr-dag]           Node / Graph / inference
  planner.py    [fusion-planner]     Algorithm 1 + the B200 region pass
  lowering.py   [kernel-lowering]    IterSpace / IndexMap / PointProgram, lower, compile
  codegen.py    [kernel-lowering]    index maps, point programs -> CUDA C++
  executor.py   [parallel-executor]  launches through the C-ABI shim; run_map,
                                     run_map_reduce, run_map_scan, run_library
  runtime.py    C-ABI binding of libgrumpy_rt.so (include/grumpy_rt.h)
  session.py    [session]            ndarray proxy, force, fallback, stats
  distributed.py  leading-axis sharding, NCCL allreduce of partials
  streaming.py  streamed to_external: H2D / kernels / D2H overlapped in chunks
  errors.py     [errors]             same class names as lazyfuse.errors
  npyio.py      [tensor-core I/O]    npy v1.0 save/load, DOT dumps of the DAG / plan
  bench_cli.py  [bench]              `bench run|dot` CLI, BenchReport JSON
"""

from . import errors
from .errors import *  # noqa: F401,F403
from .session import (  # noqa: F401
    Session,
    SessionStats,
    array,
    asarray,
    asnumpy,
    bincount,
    default_session,
    dot,
    empty,
    force,
    full,
    full_like,
    materialize,
    ndarray,
    ones,
    ones_like,
    set_default_session,
    where,
    zeros,
    zeros_like,
)
from .session import elementwise as _elementwise
from .dag import ElemCode as _E
from .tensor import DType  # noqa: F401
from .npyio import dump_dot, load, save  # noqa: F401

# Load the native shim (and with it cuBLAS 12.9 via its rpath) before anything
# imports PyTorch, whose wheel carries an older libcublas.so.12 without the
# BF16x9 FP32 emulation the np.dot boundary uses (session.GEMM_MATH).
try:
    from . import runtime as _rt
    _rt.load_library()
except Exception:  # noqa: BLE001 — no shim yet (build() not run): fails loudly on first use
    pass

import numpy as _np

float32 = _np.float32
float64 = _np.float64
int32 = _np.int32
int64 = _np.int64
bool_ = _np.bool_
newaxis = None
pi = _np.pi
e = _np.e
inf = _np.inf
nan = _np.nan


def _u(code):
    def f(x, out=None):
        if out is not None:
            raise TypeError("grumpy ufuncs do not support out=")
        return _elementwise(code, x)
    f.__name__ = code.value
    return f


def _b(code):
    def f(x, y, out=None):
        if out is not None:
            raise TypeError("grumpy ufuncs do not support out=")
        return _elementwise(code, x, y)
    f.__name__ = code.value
    return f


exp = _u(_E.exp)
log = _u(_E.log)
sqrt = _u(_E.sqrt)
square = _u(_E.square)
sin = _u(_E.sin)
cos = _u(_E.cos)
tanh = _u(_E.tanh)
erf = _u(_E.erf)
floor = _u(_E.floor)
ceil = _u(_E.ceil)
isnan = _u(_E.isnan)
negative = _u(_E.neg)
absolute = _u(_E.abs)
abs = absolute
logical_not = _u(_E.logical_not)
add = _b(_E.add)
subtract = _b(_E.sub)
multiply = _b(_E.mul)
divide = _b(_E.div)
true_divide = divide
floor_divide = _b(_E.floordiv)
remainder = _b(_E.mod)
mod = remainder
power = _b(_E.pow)
maximum = _b(_E.maximum)
minimum = _b(_E.minimum)
less = _b(_E.cmp_lt)
greater = _b(_E.cmp_gt)
less_equal = _b(_E.cmp_le)
greater_equal = _b(_E.cmp_ge)
equal = _b(_E.cmp_eq)
not_equal = _b(_E.cmp_ne)
logical_and = _b(_E.logical_and)
logical_or = _b(_E.logical_or)
logical_xor = _b(_E.logical_xor)


def _arr(x):
    return x if isinstance(x, ndarray) else asarray(x)


def sum(a, axis=None, dtype=None, keepdims=False):  # noqa: A001
    return _arr(a).sum(axis=axis, dtype=dtype, keepdims=keepdims)


def prod(a, axis=None, dtype=None, keepdims=False):
    return _arr(a).prod(axis=axis, dtype=dtype, keepdims=keepdims)


def max(a, axis=None, keepdims=False):  # noqa: A001
    return _arr(a).max(axis=axis, keepdims=keepdims)


def min(a, axis=None, keepdims=False):  # noqa: A001
    return _arr(a).min(axis=axis, keepdims=keepdims)


amax = max
amin = min


def mean(a, axis=None, dtype=None, keepdims=False):
    return _arr(a).mean(axis=axis, dtype=dtype, keepdims=keepdims)


def std(a, axis=None, dtype=None, ddof=0, keepdims=False):
    return _arr(a).std(axis=axis, dtype=dtype, ddof=ddof, keepdims=keepdims)


def var(a, axis=None, dtype=None, ddof=0, keepdims=False):
    return _arr(a).var(axis=axis, dtype=dtype, ddof=ddof, keepdims=keepdims)


def argmax(a, axis=None, keepdims=False):
    return _arr(a).argmax(axis=axis, keepdims=keepdims)


def argmin(a, axis=None, keepdims=False):
    return _arr(a).argmin(axis=axis, keepdims=keepdims)


def cumsum(a, axis=None, dtype=None):
    return _arr(a).cumsum(axis=axis, dtype=dtype)


def cumprod(a, axis=None, dtype=None):
    return _arr(a).cumprod(axis=axis, dtype=dtype)


def transpose(a, axes=None):
    return _arr(a).transpose(*(axes or ()))


def reshape(a, shape):
    return _arr(a).reshape(shape)


def matmul(a, b):
    return dot(a, b)


def clip(a, a_min=None, a_max=None):
    return _arr(a).clip(a_min, a_max)


def expand_dims(a, axis):
    from .session import _f_expand_dims
    return _f_expand_dims(a, axis)


def broadcast_to(a, shape):
    from .session import _f_broadcast_to
    return _f_broadcast_to(a, shape)


def arange(*args, dtype=None):
    return asarray(_np.arange(*args, dtype=dtype))
