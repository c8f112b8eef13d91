"""Multi-output candidate kernels and their orchestration (test infrastructure only).

SURVEY.md §8(f) N1.  Alg. 1 profiles every pair (P', O) with O a *possible output set*
of P' (every u in O has an edge (u, v) with v outside P'); the paper's
implementation keeps one output per kernel and names lifting that
restriction as future work.  Reading A32 fixes what a
multi-output candidate is and when a selection of them can run:

  candidate    (P', o, E): P' convex with the unique sink o (reading A4), E a non-empty
               set of *secondary* outputs, E subset of X(P') \\ {o}, |E| <= max_outputs - 1,
               where X(P') = {u in P' : u has a successor outside P', or u in T} (P:358-360
               plus reading A3), and every e in E has the shape of o (the kernel's
               iteration domain covers e element for element).  Materialised: {o} + E.
  Eq. 3        sum_i O_ij u_i >= 1 for p_j in T, O_ij = 1 iff p_j in {o_i} + E_i.
  Eq. 4'       kernels run in the topological order of their sinks (reading A6), so
               "computed by prior kernels" reads: for every selected k and
               every input p_j of K_k, some selected i with p_j in O_i and
               topo(o_i) < topo(o_k).  For single-output kernels this IS Eq. 4 (a
               producer of an input of K_k has its sink p_j before o_k); with secondary
               outputs it rules out the mutual-production cycles that Eq. 4 alone allows
               (SPEC S:507-515), so no cycle cuts are needed.

Candidates are triples (members, o, extras) with extras a sorted tuple (() for the
single-output ones); 2-tuples are read as extras = ().

Solvers (exact, independent of the library and of any LP solver):
  exhaustive_mo       all 2^M subsets (small M)
  producer_search_mo  branch-and-bound over producer assignments: the unmet
                      requirements of a partial selection are (tensor, deadline) pairs --
                      graph outputs, and every input of a selected kernel with that
                      kernel's sink as deadline; branch on the latest unmet tensor over
                      every producer whose sink precedes the deadline; bound = cost +
                      sum over unmet tensors of min_p c_p / |O_p| (a kernel meets at most
                      |O_p| of them).  Complete: from an optimal selection S, assigning
                      each requirement to its earliest producer in S reaches a feasible
                      subset of S.
"""
from __future__ import annotations

import math
from itertools import combinations

from .enumeration import candidate_inputs


def outputs_of(c):
    """Materialised tensors of a candidate: the sink first, then its secondary outputs."""
    return (c[1],) + (tuple(c[2]) if len(c) > 2 else ())


def possible_outputs(g, members):
    """X(P') (P:358-360 with reading A3): members with a consumer outside P' or in T."""
    m = set(members)
    return sorted(u for u in m if u in g.outputs or any(v not in m for v in g.succs[u]))


def multi_output_candidates(g, cands, max_outputs=2, same_shape=True):
    """Single-output candidates (members, o) -> the list extended with every
    (members, o, E) of reading A32, in canonical order (o, |P'|, members, E)."""
    out = [(tuple(m), o, ()) for m, o, *_ in cands]
    if max_outputs > 1:
        shapes = [tuple(nd["shape"]) for nd in g.pg["nodes"]]
        for m, o, *_ in cands:
            xs = [u for u in possible_outputs(g, m) if u != o and (not same_shape or shapes[u] == shapes[o])]
            for k in range(1, min(max_outputs - 1, len(xs)) + 1):
                for e in combinations(xs, k):
                    out.append((tuple(m), o, tuple(e)))
    out.sort(key=lambda c: (c[1], len(c[0]), c[0], c[2]))
    return out


def feasible_mo(cands, sel, outputs, cand_inputs, topo_index):
    """Eq. 3 and Eq. 4' (reading A32) for a selection."""
    sel = list(sel)
    produced = set()
    for i in sel:
        produced.update(outputs_of(cands[i]))
    if not set(outputs) <= produced:
        return False
    for k in sel:
        tk = topo_index[cands[k][1]]
        for j in cand_inputs[k]:
            if not any(j in outputs_of(cands[i]) and topo_index[cands[i][1]] < tk for i in sel):
                return False
    return True


def exhaustive_mo(cands, costs, outputs, cand_inputs, topo_index):
    """Minimum over all 2^M subsets. Returns (cost, [selections achieving it])."""
    m = len(cands)
    best, arg = math.inf, []
    for mask in range(1 << m):
        sel = [i for i in range(m) if mask >> i & 1]
        c = sum(costs[i] for i in sel)
        if c > best:
            continue
        if feasible_mo(cands, sel, outputs, cand_inputs, topo_index):
            if c < best:
                best, arg = c, [sel]
            else:
                arg.append(sel)
    return best, arg


def producer_search_mo(cands, costs, outputs, cand_inputs, topo_index):
    """Exact minimum by branch-and-bound over producer assignments (module docstring).

    Returns (cost, selection sorted); ties: fewest kernels, then the lexicographically
    smallest sorted index tuple (reading A8)."""
    producers = {}
    for i, c in enumerate(cands):
        for t in outputs_of(c):
            producers.setdefault(t, []).append(i)
    if any(t not in producers for t in outputs):
        return math.inf, None
    share = {t: min(costs[i] / len(outputs_of(cands[i])) for i in ps) for t, ps in producers.items()}
    sink = [topo_index[c[1]] for c in cands]
    never = math.inf
    best = [math.inf, None]
    seen = set()

    def key(cost, sel):
        return (cost, len(sel), tuple(sorted(sel)))

    def unmet(sel):
        """Requirements (tensor, deadline) not met by `sel`: graph outputs (deadline
        never) and every input of a selected kernel (deadline = that kernel's sink)."""
        req = [(t, never) for t in outputs] + [(j, sink[k]) for k in sel for j in cand_inputs[k]]
        return [(t, d) for t, d in req
                if not any(t in outputs_of(cands[i]) and sink[i] < d for i in sel)]

    def rec(sel, cost):
        fs = frozenset(sel)
        if fs in seen:
            return
        seen.add(fs)
        pend = unmet(sel)
        if cost + sum(share[t] for t in {t for t, _ in pend}) > best[0]:
            return
        if not pend:
            k = key(cost, sel)
            if best[1] is None or k < key(best[0], best[1]):
                best[0], best[1] = cost, list(sel)
            return
        # branch on the unmet requirement latest in topological order (every producer of
        # it that would meet it: a kernel outputting t whose sink precedes the deadline)
        t, d = max(pend, key=lambda r: (topo_index[r[0]], -r[1]))
        for i in producers.get(t, []):
            if sink[i] < d and i not in fs:
                sel.append(i)
                rec(sel, cost + costs[i])
                sel.pop()

    rec([], 0)
    return best[0], (sorted(best[1]) if best[1] is not None else None)


def kernel_order_mo(cands, sel, topo_index):
    """Sequential order: topological index of the sink (reading A6), ties by index."""
    return sorted(sel, key=lambda i: (topo_index[cands[i][1]], i))


def cand_inputs_of(g, cands):
    return [candidate_inputs(g, c[0]) for c in cands]


def eval_orchestration_mo(pg: dict, cands, sel, inputs: dict, topo_index, storage=None):
    """Execute a multi-output orchestration kernel by kernel: kernels in the
    order of their sinks (reading A6); each computes its members in float64 from the
    materialised tensors and materialises {o} + E rounded to the storage dtype (A25); the
    first kernel to materialise a tensor binds it (A7)."""
    from .evaluate import round_to_storage
    from .primitives import eval_primitive
    storage = storage or pg["dtype"]
    nodes = pg["nodes"]
    mat = {}
    for k in kernel_order_mo(cands, sel, topo_index):
        c = cands[k]
        mset = set(c[0])
        local = {}
        for v in sorted(c[0], key=lambda v: topo_index[v]):
            args = []
            for r in nodes[v]["inputs"]:
                if r[0] == "input":
                    args.append(inputs[r[1]])
                elif r[1] in mset:
                    args.append(local[r[1]])
                else:
                    if r[1] not in mat:
                        raise ValueError(f"kernel {k} input p{r[1]} not materialised by a prior kernel")
                    args.append(mat[r[1]])
            local[v] = eval_primitive(nodes[v]["kind"], nodes[v]["attrs"], args, nodes[v]["shape"])
        for t in outputs_of(c):
            if t not in mat:
                mat[t] = round_to_storage(local[t], storage)
    return {o: mat[o] for o in pg["outputs"]}
