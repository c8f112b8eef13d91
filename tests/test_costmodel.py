"""N3: the cost-model pruning step.  Pins: with exact predictions the pruned
candidate set still contains an optimal orchestration (LP reduced-cost argument); the
kept set always admits a feasible selection (operator-aligned kernels kept); the model
fits a log-linear truth exactly."""
import math

import numpy as np
import pytest

from korch_workloads import c1_softmax_layernorm, c2_vit_attention
from paper_2406_09465_b200 import Context, KorchGraph, solve_blp
from paper_2406_09465_b200.costmodel import CostModel, graph_features, prune
from paper_2406_09465_b200.select import INF


@pytest.fixture(scope="module")
def ctx():
    return Context(-1)


def _sub_optimum(kg, cands, costs, keep):
    sub = [c if i in keep else INF for i, c in enumerate(costs)]
    return kg.select(sub)[0]


@pytest.mark.parametrize("graph", [c1_softmax_layernorm, lambda: c2_vit_attention(seq=32, hidden=128, heads=2)])
def test_exact_predictions_keep_an_optimum(ctx, graph):
    kg = KorchGraph(ctx, graph())
    cands = kg.enumerate()
    rng = np.random.default_rng(0)
    for _ in range(3):
        costs = [int(rng.integers(500, 20000)) if c["klass"] != "rejected" else INF for c in cands]
        full, _ = kg.select(costs)
        keep = prune(cands, [float(c) for c in costs], kg.outputs, kg.operator_aligned(), slack=0.0)
        assert len(keep) < sum(c < INF for c in costs)
        assert _sub_optimum(kg, cands, costs, set(keep)) == full


def test_noisy_predictions_feasible_and_bounded(ctx):
    kg = KorchGraph(ctx, c1_softmax_layernorm())
    cands = kg.enumerate()
    rng = np.random.default_rng(1)
    costs = [int(rng.integers(500, 20000)) if c["klass"] != "rejected" else INF for c in cands]
    base = sum(costs[i] for i in kg.operator_aligned())
    for slack in (0.0, 0.5):
        pred = [c * math.exp(rng.normal(0, 0.5)) if c < INF else INF for c in costs]
        keep = set(prune(cands, pred, kg.outputs, kg.operator_aligned(), slack=slack))
        obj = _sub_optimum(kg, cands, costs, keep)
        assert kg.select(costs)[0] <= obj <= base


def test_model_recovers_log_linear_truth(ctx):
    kg = KorchGraph(ctx, c2_vit_attention(seq=32, hidden=128, heads=2))
    cands = kg.enumerate()
    phi = graph_features(kg)
    w = np.array([1.0, 0.3, 0.05, 0.2, 0.1, 0.0, 0.05, 0.3, 0.1])
    samples = [(c["klass"], p, math.exp(float(w @ p))) for c, p in zip(cands, phi) if c["klass"] != "rejected"]
    m = CostModel(ridge=1e-10).fit(samples)
    for k, p, ns in samples[:50]:
        assert abs(m.predict(k, p) / ns - 1) < 1e-4
