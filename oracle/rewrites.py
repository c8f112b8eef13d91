"""Primitive-graph rewrites R1-R3 (test infrastructure only).

P:224-228 (Fig. 2b): at a softmax feeding a MatMul,
  R1  the reduce primitive of Softmax is substituted by a MatMul with a constant
      tensor C_s of ones                                              (footnote P:227)
  R2  the elementwise division is swapped with the subsequent MatMul
  R3  the two MatMuls sharing an input are fused by a Pad and a Split
Readings (A28): R3 pads the other operand with 16 columns of ones (the
"ones vector ... done by padding ones", P:227 footnote; 16 keeps the merged GEMM's
N a multiple of 16 and its row stride 16-byte aligned), and the Split is two Slices
(A16); the denominator slice is reshaped to drop its unit axis before re-broadcast.

After rewriting, primitives are renumbered by Kahn's algorithm with the smallest
(pre-renumbering) id first, new primitives having ids after all existing ones in
creation order.
"""
from __future__ import annotations

from .operators import kahn_order
from .primitives import infer_shape


class _G:
    def __init__(self, pg):
        self.pg = pg
        self.nodes = {n["id"]: dict(n, inputs=list(n["inputs"])) for n in pg["nodes"]}
        self.next = max(self.nodes) + 1 if self.nodes else 0
        self.in_shapes = {s["name"]: tuple(s["shape"]) for s in pg["inputs"]}
        self.outputs = list(pg["outputs"])

    def shape(self, ref):
        return self.in_shapes[ref[1]] if ref[0] == "input" else self.nodes[ref[1]]["shape"]

    def add(self, kind, inputs, op, **attrs):
        nid = self.next
        self.next += 1
        shp = infer_shape(kind, attrs, [self.shape(r) for r in inputs])
        self.nodes[nid] = {"id": nid, "kind": kind, "attrs": attrs, "inputs": list(inputs),
                           "shape": tuple(shp), "op": op}
        return ("node", nid)

    def consumers(self, nid):
        return [v for v, n in self.nodes.items() if ("node", nid) in [tuple(r) for r in n["inputs"]]]

    def replace_uses(self, old, new_ref):
        for n in self.nodes.values():
            n["inputs"] = [new_ref if tuple(r) == ("node", old) else tuple(r) for r in n["inputs"]]
        self.outputs = [new_ref[1] if o == old else o for o in self.outputs]

    def remove_dead(self):
        changed = True
        while changed:
            changed = False
            for v in list(self.nodes):
                if v not in self.outputs and not self.consumers(v):
                    del self.nodes[v]
                    changed = True


def _sites(g: _G):
    """Softmax->MatMul sites: r = reduce_sum(e, last); b = bcast(r, last); p = div(e, b);
    o = matmul(p, V) with r, b, p single-consumer and p the matmul's first operand."""
    out = []
    for rid in sorted(g.nodes):
        r = g.nodes[rid]
        if r["kind"] != "reduce" or r["attrs"]["op"] != "sum":
            continue
        e = tuple(r["inputs"][0])
        if e[0] != "node" or r["attrs"]["axis"] != len(g.shape(e)) - 1 or len(g.shape(e)) < 2:
            continue
        cb = g.consumers(rid)
        if len(cb) != 1 or g.nodes[cb[0]]["kind"] != "broadcast":
            continue
        b = g.nodes[cb[0]]
        if b["attrs"]["axis"] != len(g.shape(e)) - 1:
            continue
        cp = g.consumers(b["id"])
        if len(cp) != 1 or g.nodes[cp[0]]["kind"] != "div":
            continue
        p = g.nodes[cp[0]]
        if [tuple(x) for x in p["inputs"]] != [e, ("node", b["id"])]:
            continue
        co = g.consumers(p["id"])
        if len(co) != 1 or g.nodes[co[0]]["kind"] != "matmul" or p["id"] in g.outputs:
            continue
        o = g.nodes[co[0]]
        if tuple(o["inputs"][0]) != ("node", p["id"]):
            continue
        out.append((rid, b["id"], p["id"], o["id"]))
    return out


def apply_r1_r3(pg: dict) -> dict:
    g = _G(pg)
    for rid, bid, pid, oid in _sites(g):
        r, b, p, o = g.nodes[rid], g.nodes[bid], g.nodes[pid], g.nodes[oid]
        e = tuple(r["inputs"][0])
        se = g.shape(e)
        n = se[-1]
        # R1: reduce_sum(e, last) -> reshape(matmul(e, C_s[n, 1]))
        cs = g.add("constant", [], r["op"], shape=[n, 1], value=1.0)
        m2 = g.add("matmul", [e, cs], r["op"])
        r1 = g.add("reshape", [m2], r["op"], shape=list(se[:-1]))
        g.replace_uses(rid, r1)
        # R2: matmul(div(e, bcast(x)), V) -> div(matmul(e, V), bcast(x))
        v = tuple(o["inputs"][1])
        nv = g.shape(v)[-1]
        m1 = g.add("matmul", [e, v], o["op"])
        bx = g.add("broadcast", [r1], p["op"], axis=len(se) - 1, size=nv)
        d = g.add("div", [m1, bx], p["op"])
        g.replace_uses(oid, d)
        # R3: matmul(e, V) and matmul(e, C_s) -> matmul(e, pad(V, ones)) + two slices
        sv = g.shape(v)
        pads = [[0, 0]] * (len(sv) - 1) + [[0, 16]]
        vh = g.add("pad", [v], o["op"], pads=pads, mode="constant", value=1.0)
        mm = g.add("matmul", [e, vh], o["op"])
        num = g.add("slice", [mm], o["op"], axis=len(se) - 1, start=0, end=nv)
        den = g.add("slice", [mm], r["op"], axis=len(se) - 1, start=nv, end=nv + 1)
        g.replace_uses(m1[1], num)
        g.replace_uses(m2[1], den)
        g.remove_dead()
    # renumber: Kahn, smallest old id first
    nodes = list(g.nodes.values())
    order = kahn_order(nodes, lambda nd: [r[1] for r in nd["inputs"] if r[0] == "node"])
    new = {old: i for i, old in enumerate(order)}
    out_nodes = []
    for old in order:
        nd = g.nodes[old]
        out_nodes.append({"id": new[old], "kind": nd["kind"], "attrs": nd["attrs"],
                          "inputs": [("node", new[r[1]]) if r[0] == "node" else tuple(r) for r in nd["inputs"]],
                          "shape": tuple(nd["shape"]), "op": nd.get("op")})
    res = dict(pg)
    res["nodes"] = out_nodes
    res["outputs"] = [new[o] for o in g.outputs]
    res.pop("op_of", None)
    return res
