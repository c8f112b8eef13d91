"""Pins for oracle/enumeration.py: definitions, Theorem 1 by brute force, paper counts."""
import itertools
import json
import os

import numpy as np
import pytest

from korch_workloads import c1_softmax_layernorm, c2_vit_attention
from oracle.enumeration import (PGraph, candidates, convex_sets_brute_force, convex_sets_from_states,
                                execution_states, is_convex, is_execution_state, sinks)
from oracle.fission import fission

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "enumeration_counts.json")))


def _all_dags(n):
    pairs = [(i, j) for i in range(n) for j in range(i + 1, n)]
    for mask in range(1 << len(pairs)):
        yield [pairs[k] for k in range(len(pairs)) if mask >> k & 1]


def _random_dag(rng, n, p):
    perm = rng.permutation(n)
    return [(int(perm[i]), int(perm[j])) for i in range(n) for j in range(i + 1, n) if rng.random() < p]


def test_states_match_definition_brute_force():
    for n in range(1, 6):
        for edges in _all_dags(n):
            g = PGraph.from_edges(n, edges)
            got = set(execution_states(g))
            ref = {frozenset(c) for k in range(n + 1) for c in itertools.combinations(range(n), k)
                   if is_execution_state(g, set(c))}
            assert got == ref


def test_theorem1_all_small_dags():
    """Theorem 1: convex <=> difference of two execution states, every DAG on <= 5 nodes."""
    for n in range(1, 6):
        for edges in _all_dags(n):
            g = PGraph.from_edges(n, edges)
            assert convex_sets_from_states(execution_states(g)) == convex_sets_brute_force(g)


def test_theorem1_random_dags():
    rng = np.random.default_rng(7)
    for _ in range(60):
        n = int(rng.integers(6, 11))
        g = PGraph.from_edges(n, _random_dag(rng, n, float(rng.uniform(0.15, 0.5))))
        assert convex_sets_from_states(execution_states(g)) == convex_sets_brute_force(g)


def test_paper_convexity_statement():
    """on a chain p1->p3->p5 with p1->p2->p5 style paths, {p1,p2,p5} is not convex when
    p5 depends on p3 which depends on p1; a set with no outside intermediate is convex."""
    # nodes 1..5 -> ids 0..4 ; p1->p3, p3->p5, p1->p2, p2->p5, p1->p4
    g = PGraph.from_edges(5, [(0, 2), (2, 4), (0, 1), (1, 4), (0, 3)])
    assert not is_convex(g, {0, 1, 4})
    assert is_convex(g, {0, 1, 2, 4})
    assert is_convex(g, {0, 3})


def test_chain_and_isolated_counts():
    for n in range(1, 9):
        chain = PGraph.from_edges(n, [(i, i + 1) for i in range(n - 1)])
        st = execution_states(chain)
        assert len(st) == n + 1
        assert len(candidates(chain, convex_sets_from_states(st), max_prims=99)) == n * (n + 1) // 2
        iso = PGraph.from_edges(n, [])
        assert len(execution_states(iso)) == 2 ** n                  # exponential in width


@pytest.mark.parametrize("case", GOLD["small"], ids=lambda c: c["name"])
def test_small_golden_counts(case):
    g = PGraph.from_edges(case["n"], [tuple(e) for e in case["edges"]])
    st = execution_states(g)
    cs = convex_sets_from_states(st)
    assert len(st) == case["states"]
    assert len(cs) == case["convex"]
    assert len(candidates(g, cs, max_prims=99)) == case["unique_sink"]


def test_config_golden_counts():
    builders = {"c1": lambda: c1_softmax_layernorm(), "c1_noaffine": lambda: c1_softmax_layernorm(affine=False),
                "c2": lambda: c2_vit_attention()}
    for case in GOLD["configs"]:
        pg = fission(builders[case["name"]]())
        g = PGraph(pg)
        st = execution_states(g)
        cs = convex_sets_from_states(st)
        assert g.n == case["prims"] and len(st) == case["states"] and len(cs) == case["convex"]
        assert len(candidates(g, cs, max_prims=10 ** 9, prune_linear=False)) == case["unique_sink"]
        if "pruned16" in case:
            assert len(candidates(g, cs, 16)) == case["pruned16"]
            assert len(candidates(g, cs, 12)) == case["pruned12"]


def test_partition_pins():
    """Reading A17: cuts only at articulation tensors; SPEC S:102 chain example."""
    from oracle.enumeration import partition
    chain = PGraph.from_edges(6, [(i, i + 1) for i in range(5)])
    assert partition(chain, 3) == [[0, 1, 2], [3, 4, 5]]
    diamond = PGraph.from_edges(4, [(0, 1), (0, 2), (1, 3), (2, 3)])
    assert partition(diamond, 2) == [[0], [1, 2, 3]]                       # only `a` is a cut tensor
    two = PGraph.from_edges(8, [(0, 1), (0, 2), (1, 3), (2, 3), (3, 4), (4, 5), (4, 6), (5, 7), (6, 7)])
    parts = partition(two, 4)
    assert sorted(v for p in parts for v in p) == list(range(8))
    for p in parts[:-1]:                                                   # one tensor crosses each cut
        later = {v for q in parts[parts.index(p) + 1:] for v in q}
        crossing = {u for u in p if any(w in later for w in two.succs[u])}
        assert len(crossing) == 1
    assert partition(two, 100) == [list(range(8))]


def test_partitioned_candidates_are_global_candidates():
    """Every within-part candidate is a convex unique-sink set of the whole graph."""
    from oracle.enumeration import candidates_partitioned, partition
    pg = fission(c2_vit_attention(seq=16, hidden=64, heads=4))
    g = PGraph(pg)
    glob = set(candidates(g, convex_sets_from_states(execution_states(g))))
    for pm in (6, 10, 16):
        parts = partition(g, pm)
        cands, _ = candidates_partitioned(g, parts)
        assert set(cands) <= glob
        for members, o in cands:
            assert is_convex(g, set(members))
            assert len({next(i for i, p in enumerate(parts) if m in p) for m in members}) == 1


def test_unique_sink_members_reach_output():
    """Reading A4: every member of a unique-sink candidate reaches its output."""
    pg = fission(c2_vit_attention(seq=16, hidden=64, heads=4))
    g = PGraph(pg)
    reach = g.reach()
    for members, o in candidates(g, convex_sets_from_states(execution_states(g))):
        assert sinks(g, set(members)) == [o]
        assert all(v == o or o in reach[v] for v in members)
