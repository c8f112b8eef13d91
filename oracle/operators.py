"""Unfissioned operator interpreter, float64 (test infrastructure only).

Each operator follows its plain definition:
  Softmax      P:83-87 Eq. 1, softmax(x_i) = e^{x_i} / sum_j e^{x_j}; literal form
               without max-subtraction (reading A9).
  LayerNorm    reading A10: (x - mean) / sqrt(var + eps) * gamma + beta, biased
               variance mean((x-mean)^2) over the last axis.
  InstanceNorm reading A11: LayerNorm over H*W per (n, c), affine per channel.
  GELU         reading A12: exact erf form x * Phi(x).
  MatMul       numpy matmul semantics (batched, 2-D right operand broadcast).
  Conv         2-D cross-correlation, NCHW, zero padding, groups.
  others       their ONNX definitions (Transpose, Reshape, Slice, Pad, Concat, ...).
"""
from __future__ import annotations

import math

import numpy as np
from scipy.special import erf as _erf


def softmax(x, axis):
    e = np.exp(x)
    return e / np.sum(e, axis=axis, keepdims=True)


def layernorm(x, gamma=None, beta=None, eps=1e-5):
    mu = np.mean(x, axis=-1, keepdims=True)
    var = np.mean((x - mu) ** 2, axis=-1, keepdims=True)
    y = (x - mu) / np.sqrt(var + eps)
    if gamma is not None:
        y = y * gamma
    if beta is not None:
        y = y + beta
    return y


def instancenorm(x, gamma, beta, eps=1e-5):
    n, c, h, w = x.shape
    mu = x.mean(axis=(2, 3), keepdims=True)
    var = ((x - mu) ** 2).mean(axis=(2, 3), keepdims=True)
    y = (x - mu) / np.sqrt(var + eps)
    return y * gamma.reshape(1, c, 1, 1) + beta.reshape(1, c, 1, 1)


def gelu(x):
    return 0.5 * x * (1.0 + _erf(x / math.sqrt(2.0)))


def conv2d(x, w, stride=(1, 1), pads=(0, 0), groups=1):
    n, c, h, wd = x.shape
    f, cg, r, s = w.shape
    assert c == cg * groups and f % groups == 0
    ph, pw = pads
    sh, sw = stride
    xp = np.zeros((n, c, h + 2 * ph, wd + 2 * pw), dtype=np.float64)
    xp[:, :, ph:ph + h, pw:pw + wd] = x
    oh = (h + 2 * ph - r) // sh + 1
    ow = (wd + 2 * pw - s) // sw + 1
    out = np.zeros((n, f, oh, ow), dtype=np.float64)
    fg = f // groups
    for g in range(groups):
        xs = xp[:, g * cg:(g + 1) * cg]
        ws = w[g * fg:(g + 1) * fg]
        for i in range(r):
            for j in range(s):
                patch = xs[:, :, i:i + sh * oh:sh, j:j + sw * ow:sw]      # [n, cg, oh, ow]
                out[:, g * fg:(g + 1) * fg] += np.einsum("nchw,fc->nfhw", patch, ws[:, :, i, j])
    return out


def maxpool(x, k, stride, pad):
    n, c, h, w = x.shape
    xp = np.full((n, c, h + 2 * pad, w + 2 * pad), -np.inf)
    xp[:, :, pad:pad + h, pad:pad + w] = x
    oh = (h + 2 * pad - k) // stride + 1
    ow = (w + 2 * pad - k) // stride + 1
    out = np.full((n, c, oh, ow), -np.inf)
    for i in range(k):
        for j in range(k):
            out = np.maximum(out, xp[:, :, i:i + stride * oh:stride, j:j + stride * ow:stride])
    return out


def pad(x, pads, mode="constant", value=0.0):
    pw = [tuple(p) for p in pads]
    if mode == "constant":
        return np.pad(x, pw, mode="constant", constant_values=value)
    if mode == "reflect":
        return np.pad(x, pw, mode="reflect")
    raise ValueError(mode)


def hardswish(x):
    return x * np.clip(x + 3.0, 0.0, 6.0) / 6.0


def sigmoid(x):
    return 1.0 / (1.0 + np.exp(-x))


def softplus(x):
    return np.log1p(np.exp(x))


UNARY = {
    "Exp": np.exp, "Sqrt": np.sqrt, "Erf": _erf, "Relu": lambda x: np.maximum(x, 0.0),
    "Sigmoid": sigmoid, "Tanh": np.tanh, "Neg": np.negative, "HardSwish": hardswish,
    "Softplus": softplus, "GELU": gelu, "SiLU": lambda x: x * sigmoid(x),
    "Mish": lambda x: x * np.tanh(softplus(x)), "Identity": lambda x: x,
}
BINARY = {"Add": np.add, "Sub": np.subtract, "Mul": np.multiply, "Div": np.divide}
SCALAR = {"AddC": lambda x, c: x + c, "MulC": lambda x, c: x * c, "DivC": lambda x, c: x / c}


def eval_operator(kind: str, attrs: dict, args: list):
    """Evaluate one operator on float64 numpy arguments."""
    if kind in UNARY:
        return UNARY[kind](args[0])
    if kind in BINARY:
        return BINARY[kind](args[0], args[1])
    if kind in SCALAR:
        return SCALAR[kind](args[0], attrs["c"])
    if kind == "Softmax":
        return softmax(args[0], attrs["axis"])
    if kind == "LayerNorm":
        g = args[1] if len(args) > 1 else None
        b = args[2] if len(args) > 2 else None
        return layernorm(args[0], g, b, attrs.get("eps", 1e-5))
    if kind == "InstanceNorm":
        return instancenorm(args[0], args[1], args[2], attrs.get("eps", 1e-5))
    if kind == "MatMul":
        return np.matmul(args[0], args[1])
    if kind == "ReduceSum":
        return np.sum(args[0], axis=attrs["axis"])
    if kind == "ReduceMean":
        return np.mean(args[0], axis=attrs["axis"])
    if kind == "ReduceMax":
        return np.max(args[0], axis=attrs["axis"])
    if kind == "Transpose":
        return np.transpose(args[0], attrs["perm"])
    if kind == "Reshape":
        return np.reshape(args[0], attrs["shape"])
    if kind == "Slice":
        sl = [slice(None)] * args[0].ndim
        sl[attrs["axis"]] = slice(attrs["start"], attrs["end"])
        return args[0][tuple(sl)]
    if kind == "Concat":
        return np.concatenate(args, axis=attrs["axis"])
    if kind == "Pad":
        return pad(args[0], attrs["pads"], attrs.get("mode", "constant"), attrs.get("value", 0.0))
    if kind == "Conv":
        y = conv2d(args[0], args[1], tuple(attrs.get("stride", (1, 1))),
                   tuple(attrs.get("pads", (0, 0))), attrs.get("groups", 1))
        if len(args) > 2:
            y = y + args[2].reshape(1, -1, 1, 1)
        return y
    if kind == "MaxPool":
        return maxpool(args[0], attrs["k"], attrs["stride"], attrs.get("pad", 0))
    if kind == "Upsample2x":
        return np.repeat(np.repeat(args[0], 2, axis=2), 2, axis=3)
    if kind == "Broadcast":
        return np.repeat(np.expand_dims(args[0], attrs["axis"]), attrs["size"], axis=attrs["axis"])
    raise NotImplementedError(kind)


def kahn_order(nodes, dep_fn):
    """Kahn's algorithm, frontier resolved by smallest id."""
    import heapq
    ids = [n["id"] for n in nodes]
    deps = {i: set(dep_fn(n)) for i, n in zip(ids, nodes)}
    users = {i: [] for i in ids}
    for i, ds in deps.items():
        for d in ds:
            users[d].append(i)
    indeg = {i: len(ds) for i, ds in deps.items()}
    heap = [i for i in ids if indeg[i] == 0]
    heapq.heapify(heap)
    order = []
    while heap:
        i = heapq.heappop(heap)
        order.append(i)
        for u in users[i]:
            indeg[u] -= 1
            if indeg[u] == 0:
                heapq.heappush(heap, u)
    if len(order) != len(ids):
        raise ValueError("cycle in graph")
    return order


def eval_operator_graph(graph: dict, inputs: dict):
    """Evaluate an operator-level graph; inputs: {name: float64 array}. Returns {node_id: array}."""
    nodes = {n["id"]: n for n in graph["nodes"]}
    order = kahn_order(graph["nodes"],
                       lambda n: [r["node"] for r in n["inputs"] if "node" in r])
    env = {}
    for i in order:
        n = nodes[i]
        args = [env[r["node"]] if "node" in r else inputs[r["input"]] for r in n["inputs"]]
        env[i] = eval_operator(n["kind"], n["attrs"], args)
    return {o: env[o] for o in graph["outputs"]}
