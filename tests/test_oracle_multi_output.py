"""Pins for oracle/multi_output.py (reading A32).

What fixes the answers, independently of the code under test:
  * hand-counted cost examples (tests/golden/multi_output_examples.json), including the
    mutual-production cycle that Eq. 4 alone admits;
  * the candidate definition re-derived by brute force: every subset, convexity by the
    definition, unique sink, every secondary output checked against the
    possible-output-set definition P:358-360 edge by edge;
  * three independent exact solvers: 2^M exhaustive, producer-assignment B&B and the
    Eq. 2-3-4' BLP solved by HiGHS;
  * with max_outputs = 1 everything reduces to the single-output oracle (Eq. 4' = Eq. 4);
  * executing any feasible multi-output orchestration equals plain graph evaluation.
"""
import json
import os
from itertools import combinations

import numpy as np
import pytest
from scipy.optimize import Bounds, LinearConstraint, milp
from scipy.sparse import lil_matrix

from korch_workloads import c1_softmax_layernorm, make_inputs
from oracle.enumeration import PGraph, candidate_inputs, candidates, convex_sets_from_states, execution_states, is_convex
from oracle.evaluate import eval_primitive_graph
from oracle.fission import fission
from oracle.multi_output import (eval_orchestration_mo, exhaustive_mo, feasible_mo, multi_output_candidates,
                                 outputs_of, producer_search_mo)
from oracle.orchestration import feasible, producer_search

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "multi_output_examples.json")))


def highs_mo(cands, costs, outputs, cin, topo):
    """Eq. 2 / Eq. 3 / Eq. 4' as a BLP (HiGHS): O_ij = 1 for every materialised output."""
    m = len(cands)
    rows, lb = [], []
    for t in outputs:
        rows.append({i: 1.0 for i, c in enumerate(cands) if t in outputs_of(c)})
        lb.append(1.0)
    for k in range(m):
        for j in cin[k]:
            r = {i: 1.0 for i, c in enumerate(cands) if j in outputs_of(c) and topo[c[1]] < topo[cands[k][1]]}
            r[k] = r.get(k, 0.0) - 1.0
            rows.append(r)
            lb.append(0.0)
    a = lil_matrix((len(rows), m))
    for ri, r in enumerate(rows):
        for i, v in r.items():
            a[ri, i] = v
    res = milp(np.asarray(costs, float), integrality=np.ones(m), bounds=Bounds(0, 1),
               constraints=LinearConstraint(a.tocsr(), lb, np.inf))
    if res.status != 0:
        return float("inf"), None
    return round(res.fun), [i for i in range(m) if res.x[i] > 0.5]


@pytest.mark.parametrize("case", GOLD["cases"], ids=lambda c: c["name"])
def test_golden_multi_output_examples(case):
    g = PGraph.from_edges(case["n"], [tuple(e) for e in case["edges"]], case["outputs"])
    cands = [(tuple(m), o, tuple(e)) for m, o, e in case["cands"]]
    cin = [candidate_inputs(g, c[0]) for c in cands]
    b1, args = exhaustive_mo(cands, case["costs"], case["outputs"], cin, g.topo_index)
    assert b1 == case["opt"]
    assert sorted(case["sel"]) in [sorted(a) for a in args]
    b2, s2 = producer_search_mo(cands, case["costs"], case["outputs"], cin, g.topo_index)
    assert b2 == case["opt"] and feasible_mo(cands, s2, case["outputs"], cin, g.topo_index)
    b3, _ = highs_mo(cands, case["costs"], case["outputs"], cin, g.topo_index)
    assert b3 == case["opt"]
    single = [i for i, c in enumerate(cands) if not c[2]]
    bs, _ = producer_search([cands[i][:2] for i in single], [case["costs"][i] for i in single],
                            case["outputs"], [cin[i] for i in single], g.topo_index)
    assert bs == case["single_output_opt"]
    if "cyclic_sel" in case:
        sel = case["cyclic_sel"]
        produced = {t for i in sel for t in outputs_of(cands[i])}
        # Eq. 3 and Eq. 4 (set form) hold ...
        assert set(case["outputs"]) <= produced and all(j in produced for i in sel for j in cin[i])
        # ... but the kernels need each other's secondary outputs: no order runs them
        assert not feasible_mo(cands, sel, case["outputs"], cin, g.topo_index)


def _brute_multi(g, max_outputs, max_prims=99):
    """Definition-level enumeration: subsets -> convex -> unique sink ->
    secondary outputs from the possible output set, same shape as the sink."""
    out = []
    for k in range(1, g.n + 1):
        for s in combinations(range(g.n), k):
            if len(s) > max_prims or not is_convex(g, s):
                continue
            ss = set(s)
            sk = [v for v in s if not any((v, w) in g.edges_set for w in ss)]
            if len(sk) != 1:
                continue
            o = sk[0]
            poss = [u for u in s if u != o and (u in g.outputs or any(v not in ss for (x, v) in g.edges_set if x == u))]
            out.append((tuple(s), o, ()))
            for r in range(1, max_outputs):
                for e in combinations(poss, r):
                    out.append((tuple(s), o, tuple(e)))
    return sorted(out, key=lambda c: (c[1], len(c[0]), c[0], c[2]))


def _dags(rng, count, nmax=5, p=0.45):
    for _ in range(count):
        n = int(rng.integers(2, nmax + 1))
        edges = [(i, j) for i in range(n) for j in range(i + 1, n) if rng.random() < p]
        g = PGraph.from_edges(n, edges)
        g.edges_set = set(edges)
        yield g


@pytest.mark.parametrize("max_outputs", [1, 2, 3])
def test_candidates_match_definition(max_outputs):
    rng = np.random.default_rng(5)
    for g in _dags(rng, 60):
        single = candidates(g, convex_sets_from_states(execution_states(g)), max_prims=99)
        assert multi_output_candidates(g, single, max_outputs) == _brute_multi(g, max_outputs)


def test_max_outputs_one_is_the_single_output_problem():
    rng = np.random.default_rng(7)
    for g in _dags(rng, 40):
        single = candidates(g, convex_sets_from_states(execution_states(g)), max_prims=99)
        mo = multi_output_candidates(g, single, 1)
        assert [c[:2] for c in mo] == single
        costs = [int(rng.integers(1, 20)) for _ in single]
        cin = [candidate_inputs(g, m) for m, _ in single]
        outs = sorted(g.outputs)
        b1, s1 = producer_search(single, costs, outs, cin, g.topo_index)
        b2, s2 = producer_search_mo(mo, costs, outs, cin, g.topo_index)
        assert b1 == b2 and feasible(single, s2, outs, cin)


def test_three_exact_solvers_agree_random_dags():
    rng = np.random.default_rng(13)
    done = wins = 0
    for g in _dags(rng, 4000, nmax=6, p=0.5):
        single = candidates(g, convex_sets_from_states(execution_states(g)), max_prims=99)
        cands = multi_output_candidates(g, single, 2)
        if len(cands) > 15 or len(cands) == len(single):
            continue
        costs = [int(rng.integers(1, 20)) for _ in cands]
        cin = [candidate_inputs(g, c[0]) for c in cands]
        outs = sorted(g.outputs)
        b1, args = exhaustive_mo(cands, costs, outs, cin, g.topo_index)
        b2, s2 = producer_search_mo(cands, costs, outs, cin, g.topo_index)
        b3, s3 = highs_mo(cands, costs, outs, cin, g.topo_index)
        assert b1 == b2 == b3
        assert sorted(s2) in [sorted(a) for a in args]
        assert feasible_mo(cands, s3, outs, cin, g.topo_index)
        sidx = [i for i, c in enumerate(cands) if not c[2]]
        bs, _ = exhaustive_mo([cands[i] for i in sidx], [costs[i] for i in sidx], outs, [cin[i] for i in sidx],
                              g.topo_index)
        assert b1 <= bs                       # a superset of candidates never costs more
        wins += b1 < bs
        done += 1
        if done >= 80:
            break
    assert done >= 80 and wins > 0


def test_execution_equals_plain_graph_evaluation_c1():
    """Every feasible multi-output orchestration computes the graph (math unchanged):
    optimal selections under many random cost tables, fp64 storage."""
    g0 = c1_softmax_layernorm()
    pg = fission(g0)
    g = PGraph(pg)
    single = candidates(g, convex_sets_from_states(execution_states(g)))
    cands = multi_output_candidates(g, single, 2)
    assert len(cands) > len(single)
    cin = [candidate_inputs(g, c[0]) for c in cands]
    ins = {k: v[0] for k, v in make_inputs(g0, seed=0).items()}
    want = eval_primitive_graph(pg, ins)
    rng = np.random.default_rng(3)
    used_multi = 0
    for trial in range(12):
        costs = [int(rng.integers(1, 50)) for _ in cands]
        # favour secondary outputs so the optimum uses them
        costs = [max(1, c // 3) if cands[i][2] else c for i, c in enumerate(costs)]
        b, sel = producer_search_mo(cands, costs, pg["outputs"], cin, g.topo_index)
        assert feasible_mo(cands, sel, pg["outputs"], cin, g.topo_index)
        used_multi += any(cands[i][2] for i in sel)
        got = eval_orchestration_mo(pg, cands, sel, ins, g.topo_index, "f64")
        for o in pg["outputs"]:
            np.testing.assert_allclose(got[o], want[o], rtol=1e-12, atol=1e-12)
    assert used_multi > 0
