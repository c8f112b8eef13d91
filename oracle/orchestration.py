"""Kernel orchestration problem, exact solutions (test infrastructure only).

P:377-413.  Selection u in {0,1}^M minimising Cost(u) = sum c_i u_i (Eq. 2)
subject to
  Eq. 3  sum_i O_ij u_i >= 1            for every output primitive p_j in T
  Eq. 4  sum_i O_ij u_i >= I_kj u_k      for every p_j in P, kernel k
with I_kj = 1 iff p_j is an input of K_k and O_ij = 1 iff p_j is the
(materialised, single) output of K_i — reading A2 (P:386 prints "input" for O
as well; "how many times p_j is executed" and Eq. 3 fix O as output).

Two exact solvers, independent of the library and of any LP solver:
  exhaustive       all 2^M subsets (M <= ~20)
  producer search  choose exactly one producing candidate for every tensor that
                   must be materialised (T plus the inputs of chosen kernels),
                   depth-first with the bound "cost so far + cheapest producer of
                   every pending tensor" (distinct tensors need distinct kernels
                   because each kernel has one output).  Complete for positive
                   costs: a second producer of a tensor can be dropped.
"""
from __future__ import annotations

import math


def feasible(cands, sel, outputs, cand_inputs):
    """Eq. 3 and Eq. 4 for a selection (iterable of candidate indices)."""
    sel = list(sel)
    produced = {cands[i][1] for i in sel}
    if not set(outputs) <= produced:
        return False
    for k in sel:
        for j in cand_inputs[k]:
            if j not in produced:
                return False
    return True


def exhaustive(cands, costs, outputs, cand_inputs):
    """Minimum over all 2^M subsets. Returns (cost, [selections achieving it])."""
    m = len(cands)
    best, arg = math.inf, []
    for mask in range(1 << m):
        sel = [i for i in range(m) if mask >> i & 1]
        c = sum(costs[i] for i in sel)
        if c > best:
            continue
        if feasible(cands, sel, outputs, cand_inputs):
            if c < best:
                best, arg = c, [sel]
            else:
                arg.append(sel)
    return best, arg


def producer_search(cands, costs, outputs, cand_inputs, topo_index):
    """Exact minimum by branch-and-bound over producer assignments.

    Returns (cost, selection sorted).  Among equal-cost optima it keeps the one with
    the fewest kernels, then the lexicographically smallest sorted index tuple
    (tie-break reading A8).
    """
    producers = {}
    for i, (_, o) in enumerate(cands):
        producers.setdefault(o, []).append(i)
    for o in producers:
        producers[o].sort(key=lambda i: (costs[i], i))
    minc = {o: costs[ps[0]] for o, ps in producers.items()}
    if any(t not in producers for t in outputs):
        return math.inf, None

    best = [math.inf, None]

    def key(cost, sel):
        return (cost, len(sel), tuple(sorted(sel)))

    def rec(pending, assigned, sel, cost):
        bound = cost + sum(minc.get(t, math.inf) for t in pending)
        if bound > best[0]:
            return
        if not pending:
            k = key(cost, sel)
            if best[1] is None or k < key(best[0], best[1]):
                best[0], best[1] = cost, list(sel)
            return
        # resolve the pending tensor latest in topological order first
        t = max(pending, key=lambda x: topo_index[x])
        rest = pending - {t}
        for i in producers.get(t, []):
            new = {j for j in cand_inputs[i] if j not in assigned and j not in rest}
            sel.append(i)
            assigned.add(t)
            rec(rest | new, assigned, sel, cost + costs[i])
            assigned.discard(t)
            sel.pop()

    rec(frozenset(outputs), set(), [], 0)
    return best[0], (sorted(best[1]) if best[1] is not None else None)


def count_producer_assignments(cands, outputs, cand_inputs, topo_index):
    """Number of distinct producer assignments (SURVEY.md Appendix A column)."""
    producers = {}
    for i, (_, o) in enumerate(cands):
        producers.setdefault(o, []).append(i)
    memo = {}

    def rec(pending, assigned):
        if not pending:
            return 1
        key = (pending, assigned)
        if key in memo:
            return memo[key]
        t = max(pending, key=lambda x: topo_index[x])
        rest = pending - {t}
        tot = 0
        for i in producers.get(t, []):
            new = frozenset(j for j in cand_inputs[i] if j not in assigned and j not in rest)
            tot += rec(rest | new, assigned | {t})
        memo[key] = tot
        return tot

    return rec(frozenset(outputs), frozenset())


def kernel_order(cands, sel, topo_index):
    """Sequential order: by topological index of the output (reading A6),
    ties by candidate index; duplicate producers keep the earliest (A7)."""
    return sorted(sel, key=lambda i: (topo_index[cands[i][1]], i))
