"""Execution states, convex subgraphs and candidate kernels (test infrastructure only).

Definitions:
  convex subgraph   no p1, p2 in P', q not in P' with p1 ~> q ~> p2
  execution state   for every edge (p1,p2): p2 in P' => p1 in P'
  Theorem 1         convex <=> difference of two execution states
Candidate kernels follow readings A3/A4: a candidate is a convex
set P' with a unique sink o (o has no successor inside P'); o is its single
output ("each candidate kernel ... produces one output tensor").
Pruning: more than max_prims primitives, or >= 2 dense linear
primitives (reading A18), is rejected before profiling.

This module deliberately does NOT run Alg. 1's DFS: states are enumerated by
their definition (include/exclude in topological order), convexity by
reachability.  The library's Alg. 1 output is compared against these.
"""
from __future__ import annotations

from itertools import combinations

from .operators import kahn_order
from .primitives import is_dense_linear


class PGraph:
    """Node-only view of a primitive graph: preds/succs over primitive ids."""

    def __init__(self, pg: dict):
        self.pg = pg
        self.n = len(pg["nodes"])
        self.preds = [sorted({r[1] for r in nd["inputs"] if r[0] == "node"}) for nd in pg["nodes"]]
        self.succs = [[] for _ in range(self.n)]
        for v, ps in enumerate(self.preds):
            for u in ps:
                self.succs[u].append(v)
        self.outputs = set(pg["outputs"])
        self.topo = kahn_order([{"id": i} for i in range(self.n)], lambda nd: self.preds[nd["id"]])
        self.topo_index = {v: i for i, v in enumerate(self.topo)}
        self._reach = None

    @classmethod
    def from_edges(cls, n, edges, outputs=None):
        nodes = [{"id": i, "kind": "relu", "attrs": {}, "inputs": [], "shape": (1,)} for i in range(n)]
        for u, v in edges:
            nodes[v]["inputs"].append(("node", u))
        if outputs is None:
            outputs = [i for i in range(n) if not any(u == i for u, _ in edges)]
        return cls({"nodes": nodes, "outputs": outputs, "inputs": []})

    def reach(self):
        """reach[u] = set of nodes v with a non-empty path u ~> v."""
        if self._reach is None:
            r = [set() for _ in range(self.n)]
            for u in reversed(self.topo):
                for v in self.succs[u]:
                    r[u].add(v)
                    r[u] |= r[v]
            self._reach = r
        return self._reach


def is_execution_state(g: PGraph, s) -> bool:
    return all(p in s for v in s for p in g.preds[v])


def is_convex(g: PGraph, s) -> bool:
    """Definition, checked directly by reachability."""
    s = set(s)
    reach = g.reach()
    outside = [q for q in range(g.n) if q not in s]
    for q in outside:
        if any(q in reach[p1] for p1 in s) and any(p2 in reach[q] for p2 in s):
            return False
    return True


def execution_states(g: PGraph, cap: int = 1_000_000):
    """All predecessor-closed subsets, INCLUDING the empty state (reading A1).

    Enumerated by deciding include/exclude for nodes in topological order: a node may be
    included only if all its predecessors are included.
    """
    topo = g.topo
    out = []

    def rec(i, cur):
        if len(out) > cap:
            raise RuntimeError("state explosion")
        if i == len(topo):
            out.append(frozenset(cur))
            return
        v = topo[i]
        rec(i + 1, cur)                       # exclude v
        if all(p in cur for p in g.preds[v]):  # include v
            cur.add(v)
            rec(i + 1, cur)
            cur.remove(v)

    rec(0, set())
    return out


def convex_sets_from_states(states):
    """Theorem 1: { D2 \\ D1 : D1 subset D2 }, non-empty, deduplicated."""
    res = set()
    for d1 in states:
        for d2 in states:
            if d1 < d2:
                res.add(d2 - d1)
    return res


def convex_sets_brute_force(g: PGraph):
    """All non-empty subsets checked against the convexity definition (small graphs)."""
    res = set()
    for k in range(1, g.n + 1):
        for c in combinations(range(g.n), k):
            if is_convex(g, c):
                res.add(frozenset(c))
    return res


def sinks(g: PGraph, s):
    return [v for v in s if not any(w in s for w in g.succs[v])]


def candidates(g: PGraph, convex_sets, max_prims=16, prune_linear=True, attention_pairs=False):
    """Unique-sink candidates (A4) after the P:626 pruning, in canonical order.

    Canonical order: sort by (output id, popcount, member-id tuple).
    attention_pairs (NEXT item N2): keep a candidate with exactly two dense
    linears L1, L2 when L1 feeds L2's first operand (the A side) and not its second.
    Returns a list of (members: tuple sorted, output: int).
    """
    pg = g.pg
    dense = set()
    if prune_linear and "inputs" in pg:
        shapes = {s["name"]: tuple(s["shape"]) for s in pg["inputs"]}
        for nd in pg["nodes"]:
            if nd["kind"] in ("matmul", "conv2d"):
                ins = [shapes[r[1]] if r[0] == "input" else pg["nodes"][r[1]]["shape"]
                       for r in nd["inputs"]]
                if is_dense_linear(nd, ins):
                    dense.add(nd["id"])
    reach = g.reach() if attention_pairs else None

    def attention_ok(pair):
        a, b = sorted(pair, key=lambda v: g.topo_index[v])
        ins = pg["nodes"][b]["inputs"]
        if pg["nodes"][a]["kind"] != "matmul" or pg["nodes"][b]["kind"] != "matmul":
            return False
        feeds = lambda r: r[0] == "node" and (r[1] == a or r[1] in reach[a])
        return feeds(ins[0]) and not feeds(ins[1])

    out = []
    for s in convex_sets:
        sk = sinks(g, s)
        if len(sk) != 1:
            continue
        if len(s) > max_prims:
            continue
        if prune_linear:
            d = dense & s
            if len(d) > 2 or (len(d) == 2 and not (attention_pairs and attention_ok(d))):
                continue
        out.append((tuple(sorted(s)), sk[0]))
    out.sort(key=lambda c: (c[1], len(c[0]), c[0]))
    return out


def partition(g: PGraph, max_nodes: int = 64):
    """Reading A17 (P:121 leaves the rule unspecified): cut at articulation tensors.

    A cut may follow position i of the topological order (Kahn, smallest id first) when
    at most k primitives of the prefix topo[0..i] are consumed after it (they are
    materialised).  k starts at 1 (single articulation tensors) and grows (up to 8) until
    no part exceeds 2 * max_nodes.  Parts are grown greedily: when a part would exceed
    max_nodes it is closed at the latest cut inside it.  Returns lists of primitive ids."""
    for k in range(1, 9):
        parts = _partition_k(g, max_nodes, k)
        if max(len(p) for p in parts) <= 2 * max_nodes:
            break
    return parts


def _partition_k(g: PGraph, max_nodes: int, max_cross: int):
    topo = g.topo
    n = len(topo)
    pos = {v: i for i, v in enumerate(topo)}
    last_use = [max((pos[w] for w in g.succs[v]), default=-1) for v in topo]
    # cuts never split an operator's fission fragment (keeps operator-aligned kernels)
    span = {}
    for v in topo:
        op = g.pg["nodes"][v].get("op")
        op = ("p", v) if op is None or op < 0 else op
        lo, hi = span.get(op, (n, -1))
        span[op] = (min(lo, pos[v]), max(hi, pos[v]))
    inside = [0] * (n + 1)
    for lo, hi in span.values():
        if hi > lo:
            inside[lo] += 1
            inside[hi] -= 1
    cut_after = []
    active = 0
    open_ops = 0
    ends = [0] * (n + 1)
    for i, v in enumerate(topo):
        if last_use[i] > i:
            active += 1
            ends[last_use[i]] += 1
        active -= ends[i]
        open_ops += inside[i]
        cut_after.append(1 <= active <= max_cross and i < n - 1 and open_ops == 0)
    parts, start, last_cut = [], 0, None
    for i in range(n):
        if i - start + 1 > max_nodes and last_cut is not None and last_cut >= start:
            parts.append(topo[start:last_cut + 1])
            start = last_cut + 1
            last_cut = None
            for j in range(start, i):       # cuts between the new start and i
                if cut_after[j]:
                    last_cut = j
        if cut_after[i]:
            last_cut = i
    parts.append(topo[start:])
    return [sorted(p) for p in parts]


def candidates_partitioned(g: PGraph, parts, max_prims=16, prune_linear=True):
    """Candidates of every part (convex unique-sink sets inside one part), canonical order.

    A set inside one part is convex in G iff it is convex in the part: a path leaving a
    part through its cut tensor never returns to it."""
    out = []
    n_states = 0
    for part in parts:
        ps = set(part)
        idx = {v: i for i, v in enumerate(part)}
        ext_specs = {}
        sub_nodes = []
        for v in part:
            nd = dict(g.pg["nodes"][v])
            ins = []
            for r in nd["inputs"]:
                if r[0] == "node" and r[1] not in ps:   # produced by an earlier part
                    name = f"__p{r[1]}"
                    ext_specs[name] = {"name": name, "shape": list(g.pg["nodes"][r[1]]["shape"])}
                    ins.append(("input", name))
                elif r[0] == "node":
                    ins.append(("node", idx[r[1]]))
                else:
                    ins.append(r)
            sub_nodes.append(dict(nd, id=idx[v], inputs=ins))
        local = {"nodes": sub_nodes, "outputs": [],
                 "inputs": list(g.pg.get("inputs", [])) + list(ext_specs.values())}
        sg = PGraph(local)
        st = execution_states(sg)
        n_states += len(st)
        back = {i: v for v, i in idx.items()}
        for members, o in candidates(sg, convex_sets_from_states(st), max_prims, prune_linear):
            out.append((tuple(sorted(back[m] for m in members)), back[o]))
    out.sort(key=lambda c: (c[1], len(c[0]), c[0]))
    return out, n_states


def candidate_inputs(g: PGraph, members):
    """Primitive inputs of a candidate: nodes outside P' feeding P' (the I matrix row)."""
    m = set(members)
    return sorted({p for v in m for p in g.preds[v] if p not in m})
