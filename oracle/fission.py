"""Operator fission: operator graph -> primitive graph (test infrastructure only).

Rules follow P:219-222 (Fig. 5: Softmax = Exp, Reduce, Broadcast, Div) and the
canonical table of SURVEY.md §8(c), readings A9-A16:

  Softmax(x,k)     exp · reduce(sum,k) · broadcast(k) · div
  LayerNorm        reduce(mean) · bcast · sub · mul(c,c) · reduce(mean) · addc(eps) ·
                   sqrt · bcast · div [· mul(gamma^) · add(beta^)]
  InstanceNorm     reshape[N,C,HW] · (LayerNorm's first 9 over HW) · mul(gamma^) ·
                   add(beta^) · reshape[N,C,H,W]
  GELU             divc(sqrt2) · erf · addc(1) · mul(x,.) · mulc(0.5)
  SiLU / Mish      sigmoid·mul / softplus·tanh·mul
  Conv(x,W,b)      conv2d · add(b^)
  Upsample2x       bcast(3,2) · bcast(5,2) · reshape
  binary ops       computed operands of lower rank get explicit leading broadcasts;
                   graph-input operands are port-broadcast (^) (A13)

Primitive ids: operators in Kahn order with smallest id first,
then each rule's primitives in the order listed.
"""
from __future__ import annotations

import math

from .operators import kahn_order
from .primitives import infer_shape

_SIMPLE = {"Exp": "exp", "Sqrt": "sqrt", "Erf": "erf", "Relu": "relu", "Sigmoid": "sigmoid",
           "Tanh": "tanh", "Neg": "neg", "HardSwish": "hardswish", "Softplus": "softplus",
           "Identity": "identity", "AddC": "addc", "MulC": "mulc", "DivC": "divc",
           "Transpose": "transpose", "Reshape": "reshape", "Slice": "slice", "Pad": "pad",
           "Concat": "concat", "MaxPool": "maxpool", "Broadcast": "broadcast"}
_BIN = {"Add": "add", "Sub": "sub", "Mul": "mul", "Div": "div"}
_RED = {"ReduceSum": "sum", "ReduceMean": "mean", "ReduceMax": "max"}


class _PG:
    def __init__(self, graph):
        self.dtype = graph["dtype"]
        self.in_shapes = {s["name"]: tuple(s["shape"]) for s in graph["inputs"]}
        self.nodes = []
        self.op = None

    def shape(self, ref):
        return self.in_shapes[ref[1]] if ref[0] == "input" else self.nodes[ref[1]]["shape"]

    def add(self, kind, inputs, **attrs):
        shp = infer_shape(kind, attrs, [self.shape(r) for r in inputs])
        nid = len(self.nodes)
        self.nodes.append({"id": nid, "kind": kind, "attrs": attrs, "inputs": list(inputs),
                           "shape": tuple(shp), "op": self.op})
        return ("node", nid)


def _norm_axis(axis, rank):
    return axis + rank if axis < 0 else axis


def _binary(pg, kind, a, b):
    sa, sb = pg.shape(a), pg.shape(b)
    if sa == sb:
        return pg.add(kind, [a, b])
    # graph-input operand: fold the broadcast into the port (A13)
    if b[0] == "input" and len(sb) <= len(sa):
        return pg.add(kind, [a, b])
    if a[0] == "input" and len(sa) <= len(sb):
        return pg.add(kind, [a, b])
    # computed operand of lower rank: explicit leading broadcasts
    if len(sa) < len(sb):
        for i in range(len(sb) - len(sa)):
            a = pg.add("broadcast", [a], axis=0, size=sb[len(sb) - len(sa) - 1 - i])
        return pg.add(kind, [a, b])
    if len(sb) < len(sa):
        for i in range(len(sa) - len(sb)):
            b = pg.add("broadcast", [b], axis=0, size=sa[len(sa) - len(sb) - 1 - i])
        return pg.add(kind, [a, b])
    raise ValueError(f"unsupported broadcast {sa} vs {sb}")


def _ln_core(pg, x, axis, eps):
    """LayerNorm's first 9 primitives over `axis` (reading A10)."""
    n = pg.shape(x)[axis]
    m = pg.add("reduce", [x], axis=axis, op="mean")
    bm = pg.add("broadcast", [m], axis=axis, size=n)
    c = pg.add("sub", [x, bm])
    s = pg.add("mul", [c, c])
    v = pg.add("reduce", [s], axis=axis, op="mean")
    ve = pg.add("addc", [v], c=float(eps))
    sd = pg.add("sqrt", [ve])
    bsd = pg.add("broadcast", [sd], axis=axis, size=n)
    return pg.add("div", [c, bsd])


def fission(graph: dict) -> dict:
    """Return a primitive-level graph dict equivalent to the operator graph."""
    pg = _PG(graph)
    ops = {n["id"]: n for n in graph["nodes"]}
    order = kahn_order(graph["nodes"], lambda n: [r["node"] for r in n["inputs"] if "node" in r])
    out_of = {}
    for oid in order:
        op = ops[oid]
        pg.op = oid
        ins = [("node", out_of[r["node"]]) if "node" in r else ("input", r["input"])
               for r in op["inputs"]]
        k, at = op["kind"], dict(op["attrs"])
        if k in _SIMPLE:
            ref = pg.add(_SIMPLE[k], ins, **at)
        elif k in _BIN:
            ref = _binary(pg, _BIN[k], ins[0], ins[1])
        elif k in _RED:
            ax = _norm_axis(at["axis"], len(pg.shape(ins[0])))
            ref = pg.add("reduce", [ins[0]], axis=ax, op=_RED[k])
        elif k == "Softmax":
            ax = _norm_axis(at["axis"], len(pg.shape(ins[0])))
            e = pg.add("exp", [ins[0]])
            r = pg.add("reduce", [e], axis=ax, op="sum")
            b = pg.add("broadcast", [r], axis=ax, size=pg.shape(ins[0])[ax])
            ref = pg.add("div", [e, b])
        elif k == "LayerNorm":
            rank = len(pg.shape(ins[0]))
            assert _norm_axis(at.get("axis", -1), rank) == rank - 1, "LayerNorm over last axis (A10)"
            ref = _ln_core(pg, ins[0], rank - 1, at.get("eps", 1e-5))
            if len(ins) > 1:
                ref = pg.add("mul", [ref, ins[1]])
            if len(ins) > 2:
                ref = pg.add("add", [ref, ins[2]])
        elif k == "InstanceNorm":
            n, c, h, w = pg.shape(ins[0])
            r = pg.add("reshape", [ins[0]], shape=[n, c, h * w])
            y = _ln_core(pg, r, 2, at.get("eps", 1e-5))
            y = pg.add("mul", [y, ins[1]], port_axes={"1": [1]})
            y = pg.add("add", [y, ins[2]], port_axes={"1": [1]})
            ref = pg.add("reshape", [y], shape=[n, c, h, w])
        elif k == "GELU":
            a = pg.add("divc", [ins[0]], c=math.sqrt(2.0))
            e = pg.add("erf", [a])
            f = pg.add("addc", [e], c=1.0)
            g = pg.add("mul", [ins[0], f])
            ref = pg.add("mulc", [g], c=0.5)
        elif k == "SiLU":
            s = pg.add("sigmoid", [ins[0]])
            ref = pg.add("mul", [ins[0], s])
        elif k == "Mish":
            s = pg.add("softplus", [ins[0]])
            t = pg.add("tanh", [s])
            ref = pg.add("mul", [ins[0], t])
        elif k == "MatMul":
            ref = pg.add("matmul", ins)
        elif k == "Conv":
            ref = pg.add("conv2d", ins[:2], stride=list(at.get("stride", [1, 1])),
                         pads=list(at.get("pads", [0, 0])), groups=at.get("groups", 1))
            if len(ins) > 2:
                ref = pg.add("add", [ref, ins[2]], port_axes={"1": [1]})
        elif k == "Upsample2x":
            n, c, h, w = pg.shape(ins[0])
            a = pg.add("broadcast", [ins[0]], axis=3, size=2)
            b = pg.add("broadcast", [a], axis=5, size=2)
            ref = pg.add("reshape", [b], shape=[n, c, 2 * h, 2 * w])
        else:
            raise NotImplementedError(f"no fission rule for {k}")
        out_of[oid] = ref[1]
    res = {"version": 1, "level": "primitive", "dtype": graph["dtype"],
           "inputs": [dict(s) for s in graph["inputs"]],
           "nodes": pg.nodes,
           "outputs": [out_of[o] for o in graph["outputs"]],
           "op_of": _op_membership(pg, order, out_of)}
    if graph.get("rewrites"):
        # R1-R3, applied after fission when the graph asks for them
        from .rewrites import apply_r1_r3
        res = apply_r1_r3(res)
    return res


def _op_membership(pg, order, out_of):
    """Map operator id -> list of primitive ids its rule produced (for the operator-aligned
    baseline orchestration)."""
    res, start = {}, 0
    for oid in order:
        end = out_of[oid] + 1
        res[oid] = list(range(start, end))
        start = end
    return res
