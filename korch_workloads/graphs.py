"""Operator-level computation graphs of the paper's workloads (synthetic weights).

Schema (after SPEC S:131-135, plus a dtype field):

    {"version": 1, "level": "operator", "dtype": "f32"|"bf16",
     "inputs":  [{"name": str, "shape": [int...], "dtype": str,
                  "init": {"dist": "normal", "mean": m, "std": s} | {"dist": "ones"}}],
     "nodes":   [{"id": int, "kind": str, "attrs": {...},
                  "inputs": [{"node": int} | {"input": str}]}],
     "outputs": [int...]}

`dtype` at graph level is the storage dtype of every computed tensor
(SURVEY.md §8(c) A20/A25).  Operator kinds are ONNX-style; the fission rules
that lower them to primitives live separately in `oracle/fission.py` and in
the C++ library (they share no code).
"""
from __future__ import annotations

import math


class GraphBuilder:
    def __init__(self, dtype: str):
        self.g = {"version": 1, "level": "operator", "dtype": dtype,
                  "inputs": [], "nodes": [], "outputs": []}

    def input(self, name, shape, dtype=None, dist="normal", mean=0.0, std=1.0):
        init = {"dist": dist}
        if dist == "normal":
            init.update(mean=float(mean), std=float(std))
        self.g["inputs"].append({"name": name, "shape": list(shape),
                                 "dtype": dtype or self.g["dtype"], "init": init})
        return {"input": name}

    def op(self, kind, *inputs, **attrs):
        nid = len(self.g["nodes"])
        self.g["nodes"].append({"id": nid, "kind": kind, "attrs": attrs,
                                "inputs": [dict(i) for i in inputs]})
        return {"node": nid}

    def output(self, ref):
        self.g["outputs"].append(ref["node"])

    def build(self):
        return self.g


def c1_softmax_layernorm(rows: int = 4, cols: int = 128, affine: bool = True,
                         eps: float = 1e-5, dtype: str = "f32", gamma_beta_std: float = 0.1):
    """Config 1 (BASELINE.json configs[0]): x[rows,cols] -> Softmax(axis 1) -> LayerNorm.

    SURVEY.md §8(d) C1; LayerNorm reading A10 (biased variance, eps inside sqrt).
    With affine=False the LN has no gamma/beta (13-primitive variant, D3).
    """
    b = GraphBuilder(dtype)
    x = b.input("x", [rows, cols])
    ins = []
    if affine:
        ins = [b.input("ln_gamma", [cols], mean=1.0, std=gamma_beta_std),
               b.input("ln_beta", [cols], mean=0.0, std=gamma_beta_std)]
    s = b.op("Softmax", x, axis=1)
    y = b.op("LayerNorm", s, *ins, axis=-1, eps=eps)
    b.output(y)
    return b.build()


def c2_vit_attention(batch: int = 1, seq: int = 128, hidden: int = 768, heads: int = 12,
                     eps: float = 1e-5, dtype: str = "bf16"):
    """Config 2 (BASELINE.json configs[1]): ViT-B pre-LN MHSA, x + Proj(MHSA(LN(x))).

    SURVEY.md §8(c) A23 / §8(d) C2.  Attention is expressed as the separate
    ONNX-style operators of the fission table's "Attention" row: Transpose(K),
    MatMul(Q,K^T), Div(sqrt d), Softmax, MatMul(P,V).
    Weights are stored [in, out] as ONNX MatMul exports them.
    """
    d = hidden // heads
    b = GraphBuilder(dtype)
    x = b.input("x", [batch, seq, hidden])
    g = b.input("ln_gamma", [hidden], mean=1.0, std=0.1)
    be = b.input("ln_beta", [hidden], mean=0.0, std=0.1)
    wqkv = b.input("w_qkv", [hidden, 3 * hidden], std=1.0 / math.sqrt(hidden))
    bqkv = b.input("b_qkv", [3 * hidden], std=0.02)
    wo = b.input("w_o", [hidden, hidden], std=1.0 / math.sqrt(hidden))
    bo = b.input("b_o", [hidden], std=0.02)

    ln = b.op("LayerNorm", x, g, be, axis=-1, eps=eps)
    qkv = b.op("MatMul", ln, wqkv)
    qkv = b.op("Add", qkv, bqkv)
    parts = []
    for i, perm in enumerate([(0, 2, 1, 3), (0, 2, 3, 1), (0, 2, 1, 3)]):
        s = b.op("Slice", qkv, axis=2, start=i * hidden, end=(i + 1) * hidden)
        r = b.op("Reshape", s, shape=[batch, seq, heads, d])
        t = b.op("Transpose", r, perm=list(perm))
        parts.append(t)
    q, kt, v = parts
    s = b.op("MatMul", q, kt)                       # [B,H,S,S]
    s = b.op("DivC", s, c=math.sqrt(d))             # A24: divide by sqrt(d)
    p = b.op("Softmax", s, axis=3)
    o = b.op("MatMul", p, v)                        # [B,H,S,d]
    o = b.op("Transpose", o, perm=[0, 2, 1, 3])     # [B,S,H,d]
    o = b.op("Reshape", o, shape=[batch, seq, hidden])
    o = b.op("MatMul", o, wo)
    o = b.op("Add", o, bo)
    y = b.op("Add", x, o)                           # residual
    b.output(y)
    return b.build()


def chain_graph(n: int, rows: int = 8, cols: int = 64, dtype: str = "f32"):
    """A chain of n elementwise operators (Relu/Exp/MulC alternating); test helper."""
    b = GraphBuilder(dtype)
    cur = b.input("x", [rows, cols])
    kinds = [("Relu", {}), ("MulC", {"c": 0.5}), ("Exp", {})]
    for i in range(n):
        k, a = kinds[i % len(kinds)]
        cur = b.op(k, cur, **a)
    b.output(cur)
    return b.build()


CONFIGS = {
    "c1": c1_softmax_layernorm,
    "c2": c2_vit_attention,
}
