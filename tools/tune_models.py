#!/usr/bin/env python
"""Tune the paper's whole models on the GPU and record the tuning database
(paper_2406_09465_b200/tunedb.py): enumerate (partitioned, reading A17), compile every
generable candidate (NVRTC sm_100a), profile every candidate and launch variant on the
device, solve Eq. 2-4 exactly, and write one JSON per (model, batch) with every
candidate's measured cost, its fastest variant, the selection and the operator-aligned
baseline.  bench.py reads these records instead of re-profiling ~3k-10k candidates per
model inside the benchmark run.

    python tools/tune_models.py [--out DIR] [--batch B] model [model ...]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2406_09465_b200 as K  # noqa: E402
import paper_2406_09465_b200.select as S  # noqa: E402
from paper_2406_09465_b200 import tunedb  # noqa: E402
from bench import model_enum_opts, model_graph  # noqa: E402


def fit_cost_model(exclude, db_dir):
    """N3: the cost model fitted on the OTHER models' recorded bs-1 databases."""
    from paper_2406_09465_b200.costmodel import CostModel, graph_features
    ctx = K.Context(-1)
    samples = []
    for fn in sorted(os.listdir(db_dir)):
        if not fn.endswith("_b1.json") or fn.startswith(exclude + "_"):
            continue
        db = tunedb.load(os.path.join(db_dir, fn))
        if not db or db.get("model") in (None, exclude):
            continue
        kg = K.KorchGraph(ctx, model_graph(db["model"]))
        cands = kg.enumerate(**db["enum_opts"])
        feats = graph_features(kg, cands)
        rec = db["kernels"]
        for i, c in enumerate(cands):
            if c["klass"] == "rejected":
                continue
            ns = [rec.get(n) for n in kg.variant_names(i)]
            ns = [v for v in ns if v is not None]
            if ns:
                samples.append((c["klass"], feats[i], min(ns)))
    return CostModel().fit(samples), len(samples)


def tune(name, batch, out_dir, max_outputs=1, prune_slack=None, db_dir=None):
    import torch
    t0 = time.perf_counter()
    graph = model_graph(name, batch)
    ctx = K.Context(torch.cuda.current_device())
    kg = K.KorchGraph(ctx, graph)
    opts = model_enum_opts(kg)
    if max_outputs > 1:
        opts["max_outputs"] = max_outputs     # N1 multi-output candidates (reading A32)
    cands = kg.enumerate(**opts)
    t_enum = time.perf_counter() - t0
    pruned = None
    todo = None
    if prune_slack is not None:
        # N3: predict every candidate's cost with a model fitted on the other
        # models, keep only the candidates reduced-cost fixing cannot exclude, and compile
        # and profile just those
        from paper_2406_09465_b200.costmodel import graph_features, prune
        t1 = time.perf_counter()
        model, n_train = fit_cost_model(name, db_dir)
        feats = graph_features(kg, cands)
        pred = [model.predict(c["klass"], f) if c["klass"] != "rejected" else S.INF for c, f in zip(cands, feats)]
        todo = prune(cands, pred, kg.outputs, kg.operator_aligned(), slack=prune_slack)
        pruned = {"slack": prune_slack, "kept": len(todo), "generable": len(kg.generable()), "train_samples": n_train,
                  "predict_prune_s": time.perf_counter() - t1}
    t1 = time.perf_counter()
    kg.compile(todo)
    t_comp = time.perf_counter() - t1
    t1 = time.perf_counter()
    if todo is None:
        costs = kg.profile()
    else:
        costs = [S.INF] * len(cands)
        for i, c in zip(todo, kg.profile(todo)):
            costs[i] = c
    t_prof = time.perf_counter() - t1
    t1 = time.perf_counter()
    obj, sel = kg.select(costs)
    t_sel = time.perf_counter() - t1
    if pruned is not None:   # only the kept candidates were timed: record the search result only
        out = {"model": name, "batch": batch, "pruned": pruned, "objective_ns": obj, "selection": sel,
               "n_candidates": len(cands), "tuning_s": {"enumerate": t_enum, "compile": t_comp, "profile": t_prof,
                                                         "select": t_sel}}
        path = os.path.join(out_dir, f"{name}_b{batch}_pruned{prune_slack}.json")
        with open(path, "w") as f:
            json.dump(out, f, indent=1)
        print(f"[tune-pruned] {name} b{batch}: kept {pruned['kept']} / {pruned['generable']}, compile {t_comp:.0f}s, "
              f"profile {t_prof:.0f}s, objective {obj} ns -> {path}", flush=True)
        del kg
        ctx.close()
        return
    base = kg.operator_aligned()
    greedy = S.greedy_fusion(kg.cands, costs, kg.prim, kg.outputs)     # P:505-518 ablation (A35)
    db = tunedb.record(kg, costs, graph, opts, extra={
        "model": name, "batch": batch, "n_candidates": len(cands), "n_generable": len(kg.generable()),
        "selection": sel, "objective_ns": obj, "blp_optimal": S.LAST_OPTIMAL, "solver": S.LAST_SOLVER,
        "operator_aligned": base, "operator_aligned_ns": sum(costs[i] for i in base),
        "greedy_fusion": greedy, "greedy_fusion_ns": sum(costs[i] for i in greedy),
        "compile_failures": len(kg.compile_failures),
        "tuning_s": {"enumerate": t_enum, "compile": t_comp, "profile": t_prof, "select": t_sel}})
    path = os.path.join(out_dir, f"{name}_b{batch}" + (f"_mo{max_outputs}" if max_outputs > 1 else "") + ".json")
    tunedb.save(path, db)
    print(f"[tune] {name} b{batch}: {len(cands)} candidates, compile {t_comp:.0f}s, profile {t_prof:.0f}s, "
          f"select {t_sel:.2f}s ({S.LAST_SOLVER}, optimal={S.LAST_OPTIMAL}), objective {obj} ns "
          f"vs operator-aligned {db['operator_aligned_ns']} ns -> {path}", flush=True)
    del kg
    ctx.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("models", nargs="+")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "tuning_db"))
    ap.add_argument("--batch", default="1", help="comma list of local batch sizes")
    ap.add_argument("--max-outputs", type=int, default=1, help="> 1: also multi-output candidates (N1)")
    ap.add_argument("--prune-slack", type=float, default=None,
                    help="N3: compile / profile only the candidates the cost model keeps (fitted on the other models)")
    ap.add_argument("--db-dir", default=os.path.join(ROOT, "profiles", "tuning_db"))
    a = ap.parse_args()
    for b in [int(x) for x in a.batch.split(",")]:
        for m in a.models:
            tune(m, b, a.out, a.max_outputs, a.prune_slack, a.db_dir)


if __name__ == "__main__":
    main()
