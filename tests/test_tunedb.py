"""Tuning database bookkeeping (paper_2406_09465_b200/tunedb.py), host only: records are
keyed by kernel name, a candidate takes its fastest recorded variant, candidates with an
unrecorded variant are reported for live profiling, and records from another code
generator / graph / device are refused."""
import numpy as np
import pytest

from korch_workloads import c1_softmax_layernorm, c2_vit_attention
from paper_2406_09465_b200 import INF, Context, KorchGraph, tunedb
from paper_2406_09465_b200._lib import LIB


@pytest.fixture(scope="module")
def ctx():
    return Context(-1)


def _fake_db(kg, graph, opts, rng, drop=()):
    kernels = {}
    for i, c in enumerate(kg.cands):
        if c["klass"] == "rejected" or i in drop:
            continue
        for n in kg.variant_names(i):
            kernels.setdefault(n, int(rng.integers(1000, 9000)))
    return {"version": LIB.korch_version().decode(), "device": tunedb.device_name(),
            "graph_key": tunedb.graph_key(graph, opts), "kernels": kernels}


def test_apply_takes_fastest_variant_and_reports_missing(ctx):
    g = c2_vit_attention(seq=32, hidden=128, heads=2)
    kg = KorchGraph(ctx, g)
    opts = {"attention_pairs": True}
    kg.enumerate(**opts)
    gen = kg.generable()
    multi = [i for i in gen if kg.variant_info(i)[0] > 1]
    assert multi
    drop = {gen[0]}
    db = _fake_db(kg, g, opts, np.random.default_rng(0), drop)
    ok, why = tunedb.usable(db, g, opts)
    assert ok, why
    costs, missing = tunedb.apply(kg, db)
    # a kernel shared by several candidates keeps one record; dropped candidates are
    # missing unless every variant of theirs is shared with a recorded candidate
    assert set(missing) <= drop
    for i in multi[:20]:
        if i in missing:
            continue
        ns = [db["kernels"][n] for n in kg.variant_names(i)]
        assert costs[i] == min(ns)
        assert kg.variant_info(i)[1] == ns.index(min(ns))
    rej = [i for i, c in enumerate(kg.cands) if c["klass"] == "rejected"]
    assert all(costs[i] == INF for i in rej)


def test_failed_variants_and_refusals(ctx):
    g = c1_softmax_layernorm()
    kg = KorchGraph(ctx, g)
    kg.enumerate()
    db = _fake_db(kg, g, {}, np.random.default_rng(1))
    i = kg.generable()[0]
    for n in kg.variant_names(i):
        db["kernels"][n] = None                  # every variant failed -> cost inf
    costs, missing = tunedb.apply(kg, db)
    assert costs[i] == INF and not missing
    assert not tunedb.usable(db, g, {"max_prims": 8})[0]                    # other enumeration
    assert not tunedb.usable(db, c1_softmax_layernorm(rows=8), {})[0]       # other graph
    assert not tunedb.usable(dict(db, version="korch-b200 0.1 codegen 00-11"), g, {})[0]
    assert not tunedb.usable(dict(db, device="NVIDIA H100"), g, {})[0]
    # a generator change that leaves the prelude alone keeps the records usable (kernel
    # names cover the rest)
    v = db["version"]
    assert tunedb.usable(dict(db, version=v.rsplit("-", 1)[0] + "-ffffffffffffffff"), g, {})[0]
    assert tunedb.prelude_salt(v) == v.rsplit("codegen ", 1)[1].split("-")[0]
