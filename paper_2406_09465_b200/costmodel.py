"""Lightweight cost model that discards candidates before profiling.

The paper names this as its future work for tuning time ("building a
lightweight cost model to quickly discard inefficient candidates"); its tuning time is
dominated by candidate profiling.  Here:

  predict   t_hat_i = exp(w_k . phi_i) per template class k (pw / rr / gemm), phi_i =
            [1, log B_i, log(1 + F_i), log |P'_i|, #reduce, #window op, #layout op,
            #MatMul/Conv, log(1 + output elements)], fitted by least squares on log measured
            costs of OTHER graphs (tuning databases, tunedb.py) -- nothing of the graph
            being tuned is profiled to build its model.
  prune     reduced-cost fixing at the predicted costs: solve the LP relaxation of
            Eq. 2-4 (Eq. 4' with secondary outputs; value LP) and the BLP itself (value
            UB) with t_hat; a candidate whose LP reduced cost exceeds UB - LP cannot be in
            any selection cheaper than UB, so it is kept only if
            rc_i <= (UB - LP) + slack * t_hat_i (slack absorbs prediction error: it could
            still enter an optimum if its prediction were off by that much); the
            operator-aligned candidates are always kept (the optimum found never exceeds
            one kernel per operator, reading A5).  Only the kept candidates are profiled;
            the BLP is then solved exactly on them.  With exact predictions and slack 0
            every optimal selection survives.
  measure   recall = (exact optimum over all candidates, measured costs) / (exact optimum
            over the kept ones, same measured costs) <= 1, and the fraction profiled.

Host-side, caller-side code (like select.py): it decides what korch_profile is asked to
time; every cost it is evaluated against is an on-device measurement.
"""
from __future__ import annotations

import math

import numpy as np
from scipy.optimize import linprog
from scipy.sparse import coo_matrix

from .select import INF, _sink_rank, outputs_of, solve_blp

CLASSES = ("pw", "rr", "gemm")
LAYOUT = {"transpose", "reshape", "slice", "concat", "pad", "broadcast"}
WINDOW = {"conv2d", "maxpool"}


def features(c, kinds, shapes):
    """phi_i for candidate dict `c` (KorchGraph.enumerate) given primitive kinds / shapes."""
    mk = [kinds[m] for m in c["members"]]
    out_el = 1
    for d in shapes[c["output"]]:
        out_el *= d
    return np.array([1.0, math.log(max(1, c["bytes"])), math.log1p(c["flops"]), math.log(len(mk)),
                     sum(k == "reduce" for k in mk), sum(k in WINDOW for k in mk), sum(k in LAYOUT for k in mk),
                     sum(k in ("matmul", "conv2d") for k in mk), math.log1p(out_el)])


def graph_features(kg, cands=None):
    cands = kg.cands if cands is None else cands
    kinds = {n["id"]: n["kind"] for n in kg.prim["nodes"]}
    shapes = {n["id"]: n["shape"] for n in kg.prim["nodes"]}
    return [features(c, kinds, shapes) for c in cands]


class CostModel:
    """Per-class log-linear regression with a small ridge term."""

    def __init__(self, ridge=1e-3):
        self.ridge = ridge
        self.w = {}

    def fit(self, samples):
        """samples: iterable of (klass, phi, measured ns)."""
        by = {}
        for k, phi, ns in samples:
            if k in CLASSES and 0 < ns < INF:
                by.setdefault(k, []).append((phi, math.log(ns)))
        for k, rows in by.items():
            X = np.array([r[0] for r in rows])
            y = np.array([r[1] for r in rows])
            A = X.T @ X + self.ridge * len(rows) * np.eye(X.shape[1])
            self.w[k] = np.linalg.solve(A, X.T @ y)
        return self

    def predict(self, klass, phi):
        if klass not in self.w:
            return INF
        return float(math.exp(float(self.w[klass] @ phi)))


def lp_reduced_costs(cands, pred, outputs, live):
    """Reduced costs of the LP relaxation of Eq. 2 / 3 / 4' (select.solve_blp's rows) at
    the predicted costs; returns {candidate: reduced cost} for `live`."""
    idx = {i: k for k, i in enumerate(live)}
    m = len(live)
    producers = {}
    for i in live:
        for t in outputs_of(cands[i]):
            producers.setdefault(t, []).append(idx[i])
    rank = _sink_rank(cands, live)
    pos = {i: rank[cands[i]["output"]] for i in live}
    rows, cols, vals, rhs = [], [], [], []
    r = 0
    for t in outputs:                                   # -sum_i O_it u_i <= -1
        for k in producers.get(t, []):
            rows.append(r); cols.append(k); vals.append(-1.0)
        rhs.append(-1.0)
        r += 1
    for i in live:                                      # u_k - sum_p u_p <= 0
        for j in cands[i]["inputs"]:
            for p in producers.get(j, []):
                if pos[live[p]] < pos[i]:
                    rows.append(r); cols.append(p); vals.append(-1.0)
            rows.append(r); cols.append(idx[i]); vals.append(1.0)
            rhs.append(0.0)
            r += 1
    a = coo_matrix((vals, (rows, cols)), shape=(r, m)).tocsr()
    c = np.array([pred[i] for i in live])
    res = linprog(c, A_ub=a, b_ub=np.array(rhs), bounds=(0, 1), method="highs")
    if res.status != 0:
        raise RuntimeError(f"LP relaxation failed: {res.message}")
    rc = np.asarray(res.lower.marginals)                # >= 0 for variables at their lower bound
    return {i: float(rc[idx[i]]) for i in live}, float(res.fun)


def prune(cands, pred, outputs, keep_always=(), slack=0.5):
    """Candidates to profile: LP reduced cost <= slack * predicted cost, plus keep_always.
    Partitioned graphs are handled per part as select.solve_partitioned does."""
    live_all = [i for i, p in enumerate(pred) if p < INF]
    parts = sorted({c.get("part", 0) for c in cands})
    part_of = {m: c.get("part", 0) for c in cands for m in c["members"]}
    needed_by_later = {j for c in cands for j in c["inputs"] if part_of.get(j, c.get("part", 0)) != c.get("part", 0)}
    keep = set(keep_always)
    for p in parts:
        live = [i for i in live_all if cands[i].get("part", 0) == p]
        if not live:
            continue
        members = {m for i in live for m in cands[i]["members"]}
        t_p = sorted(({o for o in outputs if o in members} | needed_by_later) & members)
        sub = {i: dict(cands[i], inputs=[j for j in cands[i]["inputs"] if j in members]) for i in live}
        sub_c = [sub.get(i, cands[i]) for i in range(len(cands))]
        rc, lp = lp_reduced_costs(sub_c, pred, t_p, live)
        # UB: the predicted cost of the BLP optimum at the (integer-rounded) predictions
        _, ssel = solve_blp([sub_c[i] for i in live], [int(round(pred[i])) for i in live], t_p)
        ub = sum(pred[live[k]] for k in ssel)
        gap = max(0.0, ub - lp)
        keep.update(i for i in live if rc[i] <= gap + slack * pred[i] + 1e-6 * (1 + ub))
    return sorted(keep)
