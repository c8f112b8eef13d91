"""Primitive interpreter, float64 (test infrastructure only).

The four primitive categories of P:157-192 (Table 1):
  elementwise   O[x] = f(I_1[x], ..., I_n[x])
                Graph-input operands may be port-broadcast (reading A13):
                numpy right-aligned, or via attrs["port_axes"][slot].
  reduce        O[..x_{k-1}, x_{k+1}..] = (+)_{x_k} I_1[...]
  broadcast     O[..x_k..] = I_1[..x_{k-1}, x_{k+1}..]
  layout        O[x] = I_1[L(x)], L one-to-one; concat/split/pad too
  linear        matmul / conv2d; linear in every input
Shape rules follow the same definitions.
"""
from __future__ import annotations

import numpy as np
from scipy.special import erf as _erf

from .operators import conv2d, maxpool, pad as _pad

UNARY = {
    "exp": np.exp, "sqrt": np.sqrt, "erf": _erf, "relu": lambda x: np.maximum(x, 0.0),
    "sigmoid": lambda x: 1.0 / (1.0 + np.exp(-x)), "tanh": np.tanh, "neg": np.negative,
    "hardswish": lambda x: x * np.clip(x + 3.0, 0.0, 6.0) / 6.0,
    "softplus": lambda x: np.log1p(np.exp(x)), "identity": lambda x: x,
}
SCALAR = {"addc": lambda x, c: x + c, "mulc": lambda x, c: x * c, "divc": lambda x, c: x / c}
BINARY = {"add": np.add, "sub": np.subtract, "mul": np.multiply, "div": np.divide}
ELEMENTWISE = set(UNARY) | set(SCALAR) | set(BINARY)
LAYOUT = {"transpose", "reshape", "slice", "pad", "concat"}
LINEAR = {"matmul", "conv2d"}


def category(kind: str) -> str:
    if kind in ELEMENTWISE:
        return "elementwise"
    if kind in ("reduce", "broadcast", "maxpool"):
        return "reduce_broadcast"
    if kind in LAYOUT:
        return "layout"
    if kind in LINEAR:
        return "linear"
    if kind == "constant":
        return "constant"
    raise ValueError(kind)


def is_dense_linear(node, shapes_of_inputs) -> bool:
    """Reading A18: MatMul, batched MatMul, Conv with channels-per-group >= 16."""
    if node["kind"] == "matmul":
        return True
    if node["kind"] == "conv2d":
        w = shapes_of_inputs[1]
        return w[1] >= 16
    return False


def port_view(arr, out_shape, axes):
    """Port-broadcast a graph-input operand onto out_shape (reading A13)."""
    if axes is None:
        return np.broadcast_to(arr, out_shape)
    shp = [1] * len(out_shape)
    for i, a in enumerate(axes):
        shp[a] = arr.shape[i]
    return np.broadcast_to(arr.reshape(shp), out_shape)


def infer_shape(kind, attrs, in_shapes):
    if kind in UNARY or kind in SCALAR:
        return tuple(in_shapes[0])
    if kind in BINARY:
        # the full-rank operand defines the shape (port broadcasts are graph inputs)
        a, b = tuple(in_shapes[0]), tuple(in_shapes[1])
        if attrs.get("port_axes"):
            slot = int(next(iter(attrs["port_axes"])))
            return a if slot == 1 else b
        return tuple(np.broadcast_shapes(a, b))
    if kind == "reduce":
        s = list(in_shapes[0])
        del s[attrs["axis"]]
        return tuple(s)
    if kind == "broadcast":
        s = list(in_shapes[0])
        s.insert(attrs["axis"], attrs["size"])
        return tuple(s)
    if kind == "transpose":
        return tuple(in_shapes[0][p] for p in attrs["perm"])
    if kind == "reshape":
        return tuple(attrs["shape"])
    if kind == "slice":
        s = list(in_shapes[0])
        s[attrs["axis"]] = attrs["end"] - attrs["start"]
        return tuple(s)
    if kind == "pad":
        return tuple(d + lo + hi for d, (lo, hi) in zip(in_shapes[0], attrs["pads"]))
    if kind == "concat":
        s = list(in_shapes[0])
        s[attrs["axis"]] = sum(x[attrs["axis"]] for x in in_shapes)
        return tuple(s)
    if kind == "matmul":
        a, b = in_shapes
        return tuple(np.broadcast_shapes(a[:-2], b[:-2])) + (a[-2], b[-1])
    if kind == "conv2d":
        n, c, h, w = in_shapes[0]
        f, _, r, s = in_shapes[1]
        sh, sw = attrs.get("stride", (1, 1))
        ph, pw = attrs.get("pads", (0, 0))
        return (n, f, (h + 2 * ph - r) // sh + 1, (w + 2 * pw - s) // sw + 1)
    if kind == "maxpool":
        n, c, h, w = in_shapes[0]
        k, st, p = attrs["k"], attrs["stride"], attrs.get("pad", 0)
        return (n, c, (h + 2 * p - k) // st + 1, (w + 2 * p - k) // st + 1)
    if kind == "constant":
        return tuple(attrs["shape"])
    raise ValueError(kind)


def eval_primitive(kind, attrs, args, out_shape=None):
    if kind in UNARY:
        return UNARY[kind](args[0])
    if kind in SCALAR:
        return SCALAR[kind](args[0], attrs["c"])
    if kind in BINARY:
        a, b = args
        pa = attrs.get("port_axes") or {}
        if "0" in pa:
            a = port_view(a, out_shape, pa["0"])
        if "1" in pa:
            b = port_view(b, out_shape, pa["1"])
        return BINARY[kind](a, b)
    if kind == "reduce":
        op = {"sum": np.sum, "mean": np.mean, "max": np.max}[attrs["op"]]
        return op(args[0], axis=attrs["axis"])
    if kind == "broadcast":
        return np.repeat(np.expand_dims(args[0], attrs["axis"]), attrs["size"], axis=attrs["axis"])
    if kind == "transpose":
        return np.transpose(args[0], attrs["perm"])
    if kind == "reshape":
        return np.reshape(args[0], attrs["shape"])
    if kind == "slice":
        sl = [slice(None)] * args[0].ndim
        sl[attrs["axis"]] = slice(attrs["start"], attrs["end"])
        return args[0][tuple(sl)]
    if kind == "pad":
        return _pad(args[0], attrs["pads"], attrs.get("mode", "constant"), attrs.get("value", 0.0))
    if kind == "concat":
        return np.concatenate(args, axis=attrs["axis"])
    if kind == "matmul":
        return np.matmul(args[0], args[1])
    if kind == "conv2d":
        return conv2d(args[0], args[1], tuple(attrs.get("stride", (1, 1))),
                      tuple(attrs.get("pads", (0, 0))), attrs.get("groups", 1))
    if kind == "maxpool":
        return maxpool(args[0], attrs["k"], attrs["stride"], attrs.get("pad", 0))
    if kind == "constant":
        return np.full(attrs["shape"], attrs["value"], dtype=np.float64)
    raise ValueError(kind)
