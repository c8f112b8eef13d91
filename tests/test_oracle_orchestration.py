"""Pins for oracle/orchestration.py and oracle/evaluate.py.

Two exact oracle methods (2^M exhaustive, producer-assignment branch-and-bound) are
checked against each other, against the SPEC/SURVEY cost examples, and against a third
independent method: the Eq. 2-4 BLP solved by HiGHS (scipy.optimize.milp)."""
import json
import os

import numpy as np
import pytest
from scipy.optimize import Bounds, LinearConstraint, milp
from scipy.sparse import lil_matrix

from korch_workloads import c1_softmax_layernorm, c2_vit_attention, make_inputs
from oracle.enumeration import PGraph, candidate_inputs, candidates, convex_sets_from_states, execution_states
from oracle.evaluate import eval_orchestration, eval_primitive_graph
from oracle.fission import fission
from oracle.orchestration import count_producer_assignments, exhaustive, feasible, producer_search

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "orchestration_examples.json")))


def highs_blp(cands, costs, outputs, cand_inputs, n_prims):
    """Eq. 2-4 with O = materialised output (reading A2), solved by HiGHS."""
    m = len(cands)
    rows, lb = [], []
    for t in outputs:                                            # Eq. 3
        rows.append({i: 1.0 for i, (_, o) in enumerate(cands) if o == t})
        lb.append(1.0)
    for k in range(m):                                           # Eq. 4
        for j in cand_inputs[k]:
            r = {i: 1.0 for i, (_, o) in enumerate(cands) if o == j}
            r[k] = r.get(k, 0.0) - 1.0
            rows.append(r)
            lb.append(0.0)
    a = lil_matrix((len(rows), m))
    for ri, r in enumerate(rows):
        for i, v in r.items():
            a[ri, i] = v
    res = milp(np.asarray(costs, float), integrality=np.ones(m),
               bounds=Bounds(0, 1), constraints=LinearConstraint(a.tocsr(), lb, np.inf))
    assert res.status == 0, res.message
    sel = [i for i in range(m) if res.x[i] > 0.5]
    return round(res.fun), sel


def _setup(n, edges, outputs):
    g = PGraph.from_edges(n, edges, outputs)
    return g


@pytest.mark.parametrize("case", GOLD["cases"], ids=lambda c: c["name"])
def test_golden_cost_examples(case):
    g = _setup(case["n"], [tuple(e) for e in case["edges"]], case["outputs"])
    cands = [(tuple(m), o) for m, o in case["cands"]]
    cin = [candidate_inputs(g, m) for m, _ in cands]
    best, args = exhaustive(cands, case["costs"], case["outputs"], cin)
    assert best == case["opt"]
    assert sorted(case["sel"]) in [sorted(a) for a in args]
    c2, sel2 = producer_search(cands, case["costs"], case["outputs"], cin, g.topo_index)
    assert c2 == case["opt"] and feasible(cands, sel2, case["outputs"], cin)
    c3, sel3 = highs_blp(cands, case["costs"], case["outputs"], cin, g.n)
    assert c3 == case["opt"]


def test_spec_members_reading_is_unsound():
    """Reading A2 / D4: with O = 'members', {a,b}+{b,c} would cost 2 but never materialises a
    tensor the {b,c} kernel needs; under the output reading that selection is infeasible."""
    case = [c for c in GOLD["cases"] if c["name"] == "d4_output_reading"][0]
    g = _setup(3, [(0, 1), (1, 2)], [2])
    cands = [(tuple(m), o) for m, o in case["cands"]]
    cin = [candidate_inputs(g, m) for m, _ in cands]
    assert not feasible(cands, [3, 4], [2], cin)


def _random_dag(rng, n, p):
    return [(i, j) for i in range(n) for j in range(i + 1, n) if rng.random() < p]


def test_three_methods_agree_random_dags():
    rng = np.random.default_rng(11)
    done = 0
    while done < 120:
        n = int(rng.integers(2, 7))
        edges = _random_dag(rng, n, 0.45)
        g = PGraph.from_edges(n, edges)
        cands = candidates(g, convex_sets_from_states(execution_states(g)), max_prims=99)
        if len(cands) > 16:
            continue
        costs = [int(rng.integers(1, 20)) for _ in cands]
        outs = sorted(g.outputs)
        cin = [candidate_inputs(g, m) for m, _ in cands]
        b1, _ = exhaustive(cands, costs, outs, cin)
        b2, s2 = producer_search(cands, costs, outs, cin, g.topo_index)
        b3, s3 = highs_blp(cands, costs, outs, cin, n)
        assert b1 == b2 == b3
        assert feasible(cands, s2, outs, cin) and feasible(cands, s3, outs, cin)
        done += 1


def _c1_setup():
    pg = fission(c1_softmax_layernorm())
    g = PGraph(pg)
    cands = candidates(g, convex_sets_from_states(execution_states(g)))
    cin = [candidate_inputs(g, m) for m, _ in cands]
    return pg, g, cands, cin


def test_c1_producer_assignment_count():
    """C1 with affine folded has 402,440 producer assignments."""
    pg, g, cands, cin = _c1_setup()
    assert count_producer_assignments(cands, pg["outputs"], cin, g.topo_index) == 402440


def test_c1_exact_search_matches_highs():
    pg, g, cands, cin = _c1_setup()
    rng = np.random.default_rng(5)
    for _ in range(3):
        # costs shaped like launches: ~2us + size-dependent term, integer ns
        costs = [int(2000 + 120 * len(m) + rng.integers(0, 500)) for m, _ in cands]
        b2, s2 = producer_search(cands, costs, pg["outputs"], cin, g.topo_index)
        b3, s3 = highs_blp(cands, costs, pg["outputs"], cin, g.n)
        assert b2 == b3
        assert feasible(cands, s2, pg["outputs"], cin)


def _feasible_random_selection(rng, g, cands, cin, outputs):
    producers = {}
    for i, (_, o) in enumerate(cands):
        producers.setdefault(o, []).append(i)
    need, sel, have = list(outputs), [], set()
    while need:
        t = need.pop()
        if t in have:
            continue
        i = int(rng.choice(producers[t]))
        sel.append(i)
        have.add(t)
        need.extend(j for j in cin[i] if j not in have)
    return sel


@pytest.mark.parametrize("builder", [c1_softmax_layernorm, lambda: c2_vit_attention(seq=16, hidden=64, heads=4)])
def test_orchestration_eval_equals_graph_eval(builder):
    """Any feasible orchestration computes the same function (fp64, no rounding): the
    orchestration changes only where results are materialised."""
    gr = builder()
    pg = fission(gr)
    g = PGraph(pg)
    cands = candidates(g, convex_sets_from_states(execution_states(g)))
    cin = [candidate_inputs(g, m) for m, _ in cands]
    ins = {k: v[0] for k, v in make_inputs(gr, seed=2).items()}
    ref = eval_primitive_graph(pg, ins)
    rng = np.random.default_rng(0)
    for _ in range(20):
        sel = _feasible_random_selection(rng, g, cands, cin, pg["outputs"])
        assert feasible(cands, sel, pg["outputs"], cin)
        got = eval_orchestration(pg, cands, sel, ins, g.topo_index, storage="f64")
        for o in pg["outputs"]:
            np.testing.assert_allclose(got[o], ref[o], rtol=1e-11, atol=1e-11)


def test_orchestration_eval_bf16_rounding_points():
    """With bf16 storage only kernel outputs are rounded (reading A25): a whole-graph kernel
    differs from fp64 by at most one bf16 rounding of the output."""
    gr = c1_softmax_layernorm(dtype="bf16")
    pg = fission(gr)
    g = PGraph(pg)
    cands = candidates(g, convex_sets_from_states(execution_states(g)))
    whole = [i for i, (m, o) in enumerate(cands) if len(m) == g.n]
    assert len(whole) == 1
    ins = {k: v[0] for k, v in make_inputs(gr, seed=0).items()}
    ref = eval_primitive_graph(pg, ins)[pg["outputs"][0]]
    got = eval_orchestration(pg, cands, whole, ins, g.topo_index)[pg["outputs"][0]]
    np.testing.assert_allclose(got, ref, rtol=2 ** -8, atol=0)
