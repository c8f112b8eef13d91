"""Kernel orchestration optimizer: the BLP of P:377-413, solved host-side.

This is caller-side code, not the hot path: the library exports
candidates and costs, this module picks u, and korch_set_orchestration accepts it.

  minimise   sum_i c_i u_i                                  (Eq. 2)
  s.t.       sum_i O_ij u_i >= 1          for p_j in T       (Eq. 3)
             sum_i O_ij u_i >= I_kj u_k   for all j, k       (Eq. 4)
with O_ij = 1 iff p_j is the materialised output of K_i (reading A2) and I_kj = 1
iff p_j is an input of K_k.  Solved with HiGHS (scipy.optimize.milp) in place of
PuLP/CBC (not installed).  Costs are integer nanoseconds; the objective
c_i*(M+1) + 1 breaks ties toward fewer kernels (reading A8).
"""
from __future__ import annotations

import numpy as np
from scipy.optimize import Bounds, LinearConstraint, milp
from scipy.sparse import coo_matrix

INF = (1 << 63) - 1


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
        group.sort(key=lambda i: (costs[i], len(cands[i]["inputs"]), i))
        kept = []
        for i in group:
            ins = frozenset(cands[i]["inputs"])
            if any(costs[j] <= costs[i] and ins_j <= ins for j, ins_j in kept):
                continue
            kept.append((i, ins))
        keep.extend(i for i, _ in kept)
    alive = set(keep)
    changed = True
    while changed:
        changed = False
        produced = {cands[i]["output"] for i in alive}
        for i in list(alive):
            if any(j not in produced for j in cands[i]["inputs"]):
                alive.discard(i)
                changed = True
    return sorted(alive)


def solve_blp(cands, costs, outputs, time_limit=600.0):
    """cands: list of dicts with 'output' and 'inputs'; costs: int ns (INF = rejected).

    Returns (objective_ns, sorted list of selected candidate indices)."""
    live = prune_dominated(cands, costs, [i for i, c in enumerate(costs) if c < INF])
    idx = {i: k for k, i in enumerate(live)}
    m = len(live)
    producers = {}
    for i in live:
        producers.setdefault(cands[i]["output"], []).append(idx[i])
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
    for i in live:                                             # Eq. 4
        k = idx[i]
        for j in cands[i]["inputs"]:
            ps = producers.get(j, [])
            for p in ps:
                rows.append(r); cols.append(p); vals.append(1.0)
            rows.append(r); cols.append(k); vals.append(-1.0)
            lb.append(0.0)
            r += 1
    a = coo_matrix((vals, (rows, cols)), shape=(r, m)).tocsr()
    # A8 tie-break toward fewer kernels: an optimal selection has at most one producer per
    # tensor (A7), so it has at most (#distinct outputs) kernels and a weight of that + 1
    # per ns keeps any 1 ns difference in sum(c) above every kernel-count difference
    w = float(len({cands[i]["output"] for i in live}) + 1)
    c = np.array([float(costs[i]) * w + 1.0 for i in live])
    res = milp(c, integrality=np.ones(m), bounds=Bounds(0, 1),
               constraints=LinearConstraint(a, np.array(lb), np.inf),
               options={"time_limit": time_limit, "mip_rel_gap": 0.0})
    if res.x is None:
        raise RuntimeError(f"HiGHS failed: {res.message}")
    global LAST_OPTIMAL, LAST_GAP
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
    global LAST_OPTIMAL, LAST_GAP
    LAST_OPTIMAL, LAST_GAP = True, 0.0
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
    key = {tuple(c["members"]): i for i, c in enumerate(cands)}
    sel = []
    for op, members in sorted(by_op.items()):
        i = key.get(tuple(sorted(members)))
        if i is None:
            raise ValueError(f"operator {op}'s fragment {members} is not a candidate")
        sel.append(i)
    return sorted(sel)


def singletons(cands, n_prims):
    """One kernel per primitive (the fully unfused orchestration)."""
    key = {tuple(c["members"]): i for i, c in enumerate(cands)}
    return sorted(key[(p,)] for p in range(n_prims))
