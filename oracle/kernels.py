"""numpy restatement of the 41 primitives (test oracle for minml/kernels.py:1-314).

Each ``k_<name>(call, arrays)`` returns a fresh ndarray of ``call.dtype``.
Value-domain rules: IEEE floats, wrapping integers, DomainError for integer
division by zero / negative integer powers, f64 accumulation for f32 sums
(kernels.py:139-145) and f64 contractions for f32 (kernels.py:166-239).
"""

import numpy as np

from oracle import rng
from paper_2201_12465_b200.errors import DomainError


def _cast(call, value):
    out = np.empty(tuple(call.shape), dtype=call.dtype.np)
    with np.errstate(all="ignore"):
        np.copyto(out, value, casting="unsafe")
    return out


def _operands(call, arrays):
    p = call.params
    if "scalar" in p:
        s = p["scalar"]
        return (s, arrays[0]) if p.get("scalar_side") == "left" else (arrays[0], s)
    return arrays[0], arrays[1]


def _is_int(v):
    if isinstance(v, np.ndarray):
        return v.dtype.kind in "iu"
    return type(v) is int


_UFUNC2 = {"add": np.add, "sub": np.subtract, "mul": np.multiply, "minimum": np.minimum,
           "maximum": np.maximum, "eq": np.equal, "lt": np.less, "gt": np.greater,
           "logical_and": np.logical_and, "logical_or": np.logical_or}
_UFUNC1 = {"neg": np.negative, "abs": np.abs, "exp": np.exp, "log": np.log, "sqrt": np.sqrt,
           "sin": np.sin, "cos": np.cos, "tanh": np.tanh, "logical_not": np.logical_not}


def binary(call, arrays):
    a, b = _operands(call, arrays)
    name = call.name
    with np.errstate(all="ignore"):
        if name == "div":
            if _is_int(a) and _is_int(b) and np.any(np.asarray(b) == 0):
                raise DomainError("integer division by zero")
            return _cast(call, np.true_divide(a, b))
        if name == "pow":
            try:
                return _cast(call, np.power(a, b))
            except ValueError as e:
                raise DomainError(str(e)) from None
        return _cast(call, _UFUNC2[name](a, b))


def unary(call, arrays):
    with np.errstate(all="ignore"):
        if call.name == "astype":
            return _cast(call, arrays[0])
        return _cast(call, _UFUNC1[call.name](arrays[0]))


def reduce(call, arrays):
    a = arrays[0]
    axis = call.params.get("axis")
    keep = bool(call.params.get("keepdims", False))
    with np.errstate(all="ignore"):
        if call.name == "sum":
            acc = np.float64 if a.dtype == np.float32 else a.dtype
            return _cast(call, np.sum(a, axis=axis, keepdims=keep, dtype=acc))
        if call.name == "max_reduce":
            return _cast(call, np.max(a, axis=axis, keepdims=keep))
        if call.name == "min_reduce":
            return _cast(call, np.min(a, axis=axis, keepdims=keep))
        return _cast(call, np.argmax(a, axis=axis, keepdims=keep))


def _wide(call, *arrays):
    return [x.astype(np.float64) for x in arrays] if call.dtype.name == "f32" else list(arrays)


def matmul(call, arrays):
    a, b = _wide(call, *arrays)
    with np.errstate(all="ignore"):
        return _cast(call, np.matmul(a, b))


def _patches(x, kh, kw, stride, padding):
    """[n, c, kh, kw, ho, wo] strided view of the zero-padded input."""
    n, c, h, w = x.shape
    (sh, sw), (ph, pw) = stride, padding
    xp = np.pad(x, ((0, 0), (0, 0), (ph, ph), (pw, pw)))
    ho, wo = (h + 2 * ph - kh) // sh + 1, (w + 2 * pw - kw) // sw + 1
    s = xp.strides
    return np.lib.stride_tricks.as_strided(
        xp, (n, c, kh, kw, ho, wo), (s[0], s[1], s[2], s[3], s[2] * sh, s[3] * sw), writeable=False)


def conv2d(call, arrays):
    ops = _wide(call, *arrays)
    x, w = ops[0], ops[1]
    f, c, kh, kw = w.shape
    cols = _patches(x, kh, kw, call.params["stride"], call.params["padding"])
    out = np.einsum("fcrs,ncrsyx->nfyx", w, cols, optimize=True)
    if len(ops) == 3:
        out = out + ops[2][None, :, None, None]
    return _cast(call, out)


def conv2d_grad_input(call, arrays):
    g, w = _wide(call, *arrays)
    n, f, ho, wo = g.shape
    _, c, kh, kw = w.shape
    sh, sw = call.params["stride"]
    ph, pw = call.params["padding"]
    _, _, h, wd = call.params["x_shape"]
    cols = np.einsum("fcrs,nfyx->ncrsyx", w, g, optimize=True)
    acc = np.zeros((n, c, h + 2 * ph, wd + 2 * pw), dtype=cols.dtype)
    for r in range(kh):
        for s in range(kw):
            acc[:, :, r:r + sh * ho:sh, s:s + sw * wo:sw] += cols[:, :, r, s]
    return _cast(call, acc[:, :, ph:ph + h, pw:pw + wd])


def conv2d_grad_weight(call, arrays):
    x, g = _wide(call, *arrays)
    f, c, kh, kw = call.params["w_shape"]
    cols = _patches(x, kh, kw, call.params["stride"], call.params["padding"])
    return _cast(call, np.einsum("nfyx,ncrsyx->fcrs", g, cols, optimize=True))


def reshape(call, arrays):
    return _cast(call, arrays[0].reshape(tuple(call.shape)))


def transpose(call, arrays):
    perm = call.params.get("perm") or tuple(range(arrays[0].ndim - 1, -1, -1))
    return _cast(call, np.transpose(arrays[0], perm))


def concat(call, arrays):
    with np.errstate(all="ignore"):
        return _cast(call, np.concatenate(arrays, axis=call.params["axis"]))


def slice_(call, arrays):
    p = call.params
    return _cast(call, arrays[0][tuple(slice(a, b, s) for a, b, s in zip(p["starts"], p["stops"], p["steps"]))])


def pad(call, arrays):
    p = call.params
    return _cast(call, np.pad(arrays[0], tuple(p["pad_width"]), constant_values=p.get("value", 0)))


def full(call, arrays):
    out = np.empty(tuple(call.shape), dtype=call.dtype.np)
    with np.errstate(all="ignore"):
        np.copyto(out, call.params["value"], casting="unsafe")
    return out


def arange(call, arrays):
    return _cast(call, np.arange(call.params["n"], dtype=np.int64))


def rand_uniform(call, arrays):
    p = call.params
    return _cast(call, rng.uniform(p["seed"], p["offset"], call.shape.size).reshape(tuple(call.shape)))


def rand_normal(call, arrays):
    p = call.params
    return _cast(call, rng.normal(p["seed"], p["offset"], call.shape.size).reshape(tuple(call.shape)))


def from_host(call, arrays):
    return _cast(call, call.params["array"])


def to_host(call, arrays):
    return np.array(arrays[0], copy=True)


KERNELS = {"full": full, "arange": arange, "rand_uniform": rand_uniform, "rand_normal": rand_normal,
           "from_host": from_host, "to_host": to_host, "matmul": matmul, "conv2d": conv2d,
           "conv2d_grad_input": conv2d_grad_input, "conv2d_grad_weight": conv2d_grad_weight,
           "reshape": reshape, "transpose": transpose, "concat": concat, "slice": slice_, "pad": pad}
for _n in ("add", "sub", "mul", "div", "pow", "minimum", "maximum", "eq", "lt", "gt",
           "logical_and", "logical_or"):
    KERNELS[_n] = binary
for _n in ("neg", "abs", "exp", "log", "sqrt", "sin", "cos", "tanh", "logical_not", "astype"):
    KERNELS[_n] = unary
for _n in ("sum", "max_reduce", "min_reduce", "argmax"):
    KERNELS[_n] = reduce
