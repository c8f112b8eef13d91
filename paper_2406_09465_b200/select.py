"""Kernel orchestration optimizer: the BLP of P:377-413, solved host-side.

This is caller-side code, not the hot path: the library exports
candidates and costs, this module picks u, and korch_set_orchestration accepts it.

  minimise   sum_i c_i u_i                                  (Eq. 2)
  s.t.       sum_i O_ij u_i >= 1          for p_j in T       (Eq. 3)
             sum_i O_ij u_i >= I_kj u_k   for all j, k       (Eq. 4)
with O_ij = 1 iff p_j is a materialised output of K_i (reading A2; the sink, plus the
secondary outputs of a multi-output candidate, N1 / reading A32) and I_kj = 1 iff p_j
is an input of K_k.  With secondary outputs Eq. 4 becomes Eq. 4' (reading A32): the
producers counted for an input of K_k are those whose sink precedes K_k's sink (kernels
run in sink order, A6), which for single-output candidates is Eq. 4 unchanged.  Solved with HiGHS (scipy.optimize.milp) in place of
PuLP/CBC (not installed).  Costs are integer nanoseconds; the objective
c_i*(M+1) + 1 breaks ties toward fewer kernels (reading A8).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np
from scipy.optimize import Bounds, LinearConstraint, milp
from scipy.sparse import coo_matrix

INF = (1 << 63) - 1

_SEL_LIB = None


def _select_lib():
    """libkorch_select.so (include/korch_select.h), built in-tree by build.py."""
    global _SEL_LIB
    if _SEL_LIB is None:
        path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libkorch_select.so")
        lib = C.CDLL(path)
        P32, P64 = C.POINTER(C.c_int32), C.POINTER(C.c_int64)
        lib.korch_select_exact.argtypes = [C.c_int32, C.c_int32, P32, P32, P32, P64, C.c_int32, P32, C.c_int64,
                                           C.c_double, P64, P32, P64]
        lib.korch_select_exact.restype = C.c_int32
        _SEL_LIB = lib
    return _SEL_LIB


def solve_exact(cands, costs, outputs, live=None, time_limit=60.0, max_states=20_000_000):
    """Exact optimum by the native A* search over producer assignments
    (libkorch_select.so).  Returns (objective_ns, selection) or None when a limit was
    reached before optimality was proven."""
    live = [i for i, c in enumerate(costs) if c < INF] if live is None else list(live)
    # tensor numbering: a topological order of the "input -> output" relation of the
    # live candidates (inputs always precede the output in the primitive DAG)
    tensors = sorted({cands[i]["output"] for i in live} | {j for i in live for j in cands[i]["inputs"]} |
                     set(outputs))
    succ = {t: [] for t in tensors}
    indeg = {t: 0 for t in tensors}
    edges = set()
    for i in live:
        for j in cands[i]["inputs"]:
            if (j, cands[i]["output"]) not in edges:
                edges.add((j, cands[i]["output"]))
                succ[j].append(cands[i]["output"])
                indeg[cands[i]["output"]] += 1
    import heapq
    ready = [t for t in tensors if indeg[t] == 0]
    heapq.heapify(ready)
    order = []
    while ready:
        t = heapq.heappop(ready)
        order.append(t)
        for w in succ[t]:
            indeg[w] -= 1
            if indeg[w] == 0:
                heapq.heappush(ready, w)
    if len(order) != len(tensors) or len(tensors) > 512:
        return None
    loc = {t: k for k, t in enumerate(order)}
    m = len(live)
    out = (C.c_int32 * max(1, m))(*[loc[cands[i]["output"]] for i in live])
    off, ins = [0], []
    for i in live:
        ins.extend(loc[j] for j in cands[i]["inputs"])
        off.append(len(ins))
    off_a = (C.c_int32 * (m + 1))(*off)
    in_a = (C.c_int32 * max(1, len(ins)))(*ins)
    cost_a = (C.c_int64 * max(1, m))(*[int(costs[i]) for i in live])
    req = sorted({loc[t] for t in outputs})
    req_a = (C.c_int32 * max(1, len(req)))(*req)
    best, nexp = C.c_int64(), C.c_int64()
    sel = (C.c_int32 * max(1, m))()
    st = _select_lib().korch_select_exact(len(order), m, out, off_a, in_a, cost_a, len(req), req_a, max_states,
                                          float(time_limit), C.byref(best), sel, C.byref(nexp))
    global LAST_EXPANDED
    LAST_EXPANDED += nexp.value
    if st == -6:
        raise ValueError("infeasible: some required tensor has no generable producer chain")
    if st != 0:
        return None
    chosen = sorted(live[k] for k in range(m) if sel[k])
    return int(best.value), chosen


LAST_EXPANDED = 0  # A* states expanded by the last solve (all parts)
LAST_SOLVER = ""   # "exact" (native A*) or "highs" for the last solve


def outputs_of(c):
    """Materialised tensors of a candidate: the sink, then its secondary outputs (N1)."""
    return [c["output"]] + list(c.get("extra_outputs", ()))


def prune_dominated(cands, costs, live):
    """Exact reduction of the BLP before the MILP.

    * Dominance: candidate i is dominated by j if both produce the same tensor, j reads a
      subset of i's inputs (Eq. 4 then asks for no more materialised tensors) and
      c_j <= c_i (ties: the lower index stays).  Swapping i for j in any feasible
      selection keeps it feasible and neither raises the cost nor the kernel count, so an
      optimum (with A8's tie-break) survives.
    * Dead candidates: one that reads a tensor nobody (left) can produce can never be
      selected under Eq. 4; removed to a fixpoint.
    Returns the surviving candidate indices (sorted)."""
    by_out = {}
    for i in live:
        by_out.setdefault(cands[i]["output"], []).append(i)
    keep = []
    for o, group in by_out.items():
        # same sink (so the same place in the schedule, Eq. 4'); j dominates i when it
        # materialises a superset of i's outputs from a subset of its inputs at no more cost
        group.sort(key=lambda i: (costs[i], len(cands[i]["inputs"]), -len(outputs_of(cands[i])), i))
        kept = []
        for i in group:
            ins = frozenset(cands[i]["inputs"])
            outs = frozenset(outputs_of(cands[i]))
            if any(costs[j] <= costs[i] and ins_j <= ins and outs <= outs_j for j, ins_j, outs_j in kept):
                continue
            kept.append((i, ins, outs))
        keep.extend(i for i, _, _ in kept)
    alive = set(keep)
    topo = _sink_rank(cands, live)
    changed = True
    while changed:
        changed = False
        # earliest sink rank at which each tensor is materialised by a live candidate
        first = {}
        for i in alive:
            for t in outputs_of(cands[i]):
                first[t] = min(first.get(t, 1 << 60), topo[cands[i]["output"]])
        for i in list(alive):
            if any(first.get(j, 1 << 60) >= topo[cands[i]["output"]] for j in cands[i]["inputs"]):
                alive.discard(i)
                changed = True
    return sorted(alive)


def _sink_rank(cands, live):
    """Schedule position of every live candidate's sink (reading A6): the library's
    topological index ("sink_topo", set by KorchGraph.enumerate).  Without it (host tests
    with hand-made single-output candidates) any topological rank of the sinks gives the
    same Eq. 4; secondary outputs need the library's order, so it is then required."""
    if all("sink_topo" in cands[i] for i in live):
        return {cands[i]["output"]: cands[i]["sink_topo"] for i in live}
    if any(cands[i].get("extra_outputs") for i in live):
        raise ValueError("multi-output candidates need their sink's topological index ('sink_topo')")
    import heapq
    nodes, succ, indeg = set(), {}, {}
    for i in live:
        o = cands[i]["output"]
        nodes.add(o)
        for j in cands[i]["inputs"]:
            nodes.add(j)
            if o not in succ.setdefault(j, set()):
                succ[j].add(o)
                indeg[o] = indeg.get(o, 0) + 1
    ready = [t for t in nodes if indeg.get(t, 0) == 0]
    heapq.heapify(ready)
    rank = {}
    while ready:
        t = heapq.heappop(ready)
        rank[t] = len(rank)
        for w in succ.get(t, ()):
            indeg[w] -= 1
            if indeg[w] == 0:
                heapq.heappush(ready, w)
    return rank


def solve_blp(cands, costs, outputs, time_limit=600.0, exact=True, exact_time_limit=120.0):
    """cands: list of dicts with 'output' and 'inputs'; costs: int ns (INF = rejected).

    Exact reductions first (prune_dominated), then the native exact A* search
    (solve_exact); HiGHS on the MILP only if the search hits its limits.
    Returns (objective_ns, sorted list of selected candidate indices)."""
    global LAST_OPTIMAL, LAST_GAP, LAST_SOLVER
    live = prune_dominated(cands, costs, [i for i, c in enumerate(costs) if c < INF])
    for t in outputs:
        if not any(t in outputs_of(cands[i]) for i in live):
            raise ValueError(f"infeasible: output p{t} has no generable producer")
    multi = any(cands[i].get("extra_outputs") for i in live)
    # the native A* search resolves one producer per tensor (single-output candidates);
    # with secondary outputs the MILP with Eq. 4' is solved instead (to optimality)
    if exact and not multi:
        r = solve_exact(cands, costs, outputs, live, time_limit=min(time_limit, exact_time_limit))
        if r is not None:
            LAST_SOLVER = "exact" if LAST_SOLVER in ("", "exact") else "mixed"
            return r
    LAST_SOLVER = "highs" if LAST_SOLVER in ("", "highs") else "mixed"
    idx = {i: k for k, i in enumerate(live)}
    m = len(live)
    producers = {}
    for i in live:
        for t in outputs_of(cands[i]):
            producers.setdefault(t, []).append(idx[i])
    rank = _sink_rank(cands, live)
    pos = {i: rank[cands[i]["output"]] for i in live}
    rows, cols, vals, lb = [], [], [], []
    r = 0
    for t in outputs:                                          # Eq. 3
        ps = producers.get(t, [])
        if not ps:
            raise ValueError(f"infeasible: output p{t} has no generable producer")
        for k in ps:
            rows.append(r); cols.append(k); vals.append(1.0)
        lb.append(1.0)
        r += 1
    for i in live:                                             # Eq. 4 (Eq. 4')
        k = idx[i]
        for j in cands[i]["inputs"]:
            ps = [p for p in producers.get(j, []) if pos[live[p]] < pos[i]]
            for p in ps:
                rows.append(r); cols.append(p); vals.append(1.0)
            rows.append(r); cols.append(k); vals.append(-1.0)
            lb.append(0.0)
            r += 1
    a = coo_matrix((vals, (rows, cols)), shape=(r, m)).tocsr()
    # A8 tie-break toward fewer kernels: an optimal selection has at most one producer per
    # tensor (A7), so it has at most (#distinct outputs) kernels and a weight of that + 1
    # per ns keeps any 1 ns difference in sum(c) above every kernel-count difference
    w = float(len({t for i in live for t in outputs_of(cands[i])}) + 1)
    c = np.array([float(costs[i]) * w + 1.0 for i in live])
    res = milp(c, integrality=np.ones(m), bounds=Bounds(0, 1),
               constraints=LinearConstraint(a, np.array(lb), np.inf),
               options={"time_limit": time_limit, "mip_rel_gap": 0.0})
    if res.x is None:
        raise RuntimeError(f"HiGHS failed: {res.message}")
    LAST_OPTIMAL = LAST_OPTIMAL and res.status == 0  # 0 = optimal; 1 = time limit (best found)
    gap = getattr(res, "mip_gap", 0.0)
    LAST_GAP = max(LAST_GAP, float(gap) if gap is not None and res.status != 0 else 0.0)
    sel = sorted(live[k] for k in range(m) if res.x[k] > 0.5)
    return int(sum(costs[i] for i in sel)), sel


LAST_OPTIMAL = True  # False if some part of the last solve stopped at its time limit
LAST_GAP = 0.0       # largest relative MIP gap left by a time-limited part


def solve_partitioned(cands, costs, outputs, time_limit=600.0):
    """Per-part decomposition of the BLP (parts from partitioning, reading A17).

    Parts interact only through cut tensors (a part's primitives consumed by a later
    part), so the global optimum is the sum of per-part optima with
    T_part = (graph outputs in the part) + (its primitives consumed by later parts)."""
    global LAST_OPTIMAL, LAST_GAP, LAST_EXPANDED, LAST_SOLVER
    LAST_OPTIMAL, LAST_GAP, LAST_EXPANDED, LAST_SOLVER = True, 0.0, 0, ""
    parts = sorted({c.get("part", 0) for c in cands})
    if len(parts) <= 1:
        return solve_blp(cands, costs, outputs, time_limit)
    part_of = {}
    for c in cands:
        for m in c["members"]:
            part_of[m] = c.get("part", 0)
    needed_by_later = set()
    for c in cands:
        for j in c["inputs"]:
            if part_of.get(j, c["part"]) != c["part"]:
                needed_by_later.add(j)
    total, sel = 0, []
    for p in parts:
        idx = [i for i, c in enumerate(cands) if c.get("part", 0) == p]
        sub = [cands[i] for i in idx]
        members = {m for c in sub for m in c["members"]}
        t_p = sorted(({o for o in outputs if o in members} | needed_by_later) & members)
        # inputs produced by earlier parts are available (their T made them so)
        sub_local = [dict(c, inputs=[j for j in c["inputs"] if j in members]) for c in sub]
        obj, s = solve_blp(sub_local, [costs[i] for i in idx], t_p, time_limit)
        total += obj
        sel.extend(idx[k] for k in s)
    return total, sorted(sel)


def operator_aligned(cands, prim_graph):
    """The 'one kernel per unfused operator' orchestration: for every
    operator, the candidate whose members are exactly that operator's fission fragment."""
    by_op = {}
    for n in prim_graph["nodes"]:
        by_op.setdefault(n["op"], []).append(n["id"])
    key = {tuple(c["members"]): i for i, c in enumerate(cands) if not c.get("extra_outputs")}
    sel = []
    for op, members in sorted(by_op.items()):
        i = key.get(tuple(sorted(members)))
        if i is None:
            raise ValueError(f"operator {op}'s fragment {members} is not a candidate")
        sel.append(i)
    return sorted(sel)


def singletons(cands, n_prims):
    """One kernel per primitive (the fully unfused orchestration)."""
    key = {tuple(c["members"]): i for i, c in enumerate(cands) if not c.get("extra_outputs")}
    return sorted(key[(p,)] for p in range(n_prims))


def greedy_fusion(cands, costs, prim_graph, outputs):
    """Fission followed by greedy fusion, without the BLP: the ablation of P:505-518 (the
    paper feeds the fissioned primitive graph to TensorRT and lets it pick the kernels) and
    the 'always fuse what can be fused' policy of P:611-616 (TVM fuses the whole
    memory-bound subgraph).  Start from one kernel per primitive; walk the primitives in
    topological order and merge a primitive's kernel into its consumer's when the consumer
    kernel is that kernel's only consumer and the union is a generable candidate (same
    templates, cost < inf).  Primitives are visited consumers first (reverse topological
    order) so producers join the kernel their consumers already formed (TVM's
    producer-into-consumer fusion).  Every kernel materialises its sink; the result is a
    partition (no redundant computation).  Returns the selection (sorted candidate indices)."""
    gen = {}
    for i, c in enumerate(cands):
        if costs[i] < INF and not c.get("extra_outputs"):
            gen[frozenset(c["members"])] = i
    nodes = prim_graph["nodes"]
    succ = {n["id"]: set() for n in nodes}
    for n in nodes:
        for r in n["inputs"]:
            if "node" in r:
                succ[r["node"]].add(n["id"])
    group = {n["id"]: frozenset([n["id"]]) for n in nodes}   # primitive -> its kernel's members
    topo = prim_graph_topo(prim_graph)
    for v in sorted(succ, key=lambda x: -topo[x]):
        g = group[v]
        sinks = [u for u in g if not (succ[u] & g)]
        if len(sinks) != 1 or sinks[0] != v or v in outputs:
            continue
        consumers = {frozenset(group[w]) for w in succ[v]}
        if len(consumers) != 1:
            continue
        (cg,) = consumers
        merged = g | cg
        if merged in gen:
            for u in merged:
                group[u] = merged
    kernels = set(group.values())
    if any(g not in gen for g in kernels):
        raise ValueError("greedy fusion left a kernel with no generable candidate")
    return sorted(gen[g] for g in kernels)


_TOPO_CACHE = {}


def prim_graph_topo(prim_graph):
    key = id(prim_graph)
    if key not in _TOPO_CACHE:
        import heapq
        nodes = prim_graph["nodes"]
        preds = {n["id"]: {r["node"] for r in n["inputs"] if "node" in r} for n in nodes}
        succ = {v: [] for v in preds}
        for v, ps in preds.items():
            for u in ps:
                succ[u].append(v)
        indeg = {v: len(p) for v, p in preds.items()}
        ready = [v for v, d in indeg.items() if not d]
        heapq.heapify(ready)
        pos = {}
        while ready:
            v = heapq.heappop(ready)
            pos[v] = len(pos)
            for w in succ[v]:
                indeg[w] -= 1
                if not indeg[w]:
                    heapq.heappush(ready, w)
        _TOPO_CACHE[key] = pos
    return _TOPO_CACHE[key]
