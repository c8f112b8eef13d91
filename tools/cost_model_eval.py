#!/usr/bin/env python
"""N3 evaluation: how much profiling the cost model saves and what it costs in
orchestration quality, measured against the full on-device profile recorded in the
tuning databases (profiles/tuning_db, written on a B200 by tools/tune_models.py).

For every model M with a database: fit the cost model on the OTHER models' measured
costs (leave-one-model-out), predict M's candidate costs, prune by reduced-cost fixing
(costmodel.prune), then solve the BLP exactly on the kept candidates with M's MEASURED
costs and compare with the optimum over all candidates:

    recall   = optimum(all) / optimum(kept)      (1.0 = nothing lost)
    profiled = kept / generable                   (fraction of candidates to time)

Also reports the model's accuracy (median |log error|, Spearman rank correlation) and
the fission + greedy-fusion ablation (select.greedy_fusion) next to the
operator-aligned plan and the BLP optimum, all on measured costs.  Runs on the host (no
GPU): candidates are enumerated by the library on a host-only context and costs come
from the databases.

    python tools/cost_model_eval.py [--slack 0.5] [--out profiles/r02_cost_model.json]
"""
import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2406_09465_b200 as K  # noqa: E402
from paper_2406_09465_b200 import tunedb  # noqa: E402
from paper_2406_09465_b200.costmodel import CostModel, graph_features, prune  # noqa: E402
from paper_2406_09465_b200.select import INF, greedy_fusion  # noqa: E402
from bench import model_enum_opts, model_graph  # noqa: E402


def load_model(ctx, name, db_dir, batch=1):
    db = tunedb.load(os.path.join(db_dir, f"{name}_b{batch}.json"))
    if db is None:
        return None
    graph = model_graph(name, batch)
    kg = K.KorchGraph(ctx, graph)
    opts = db.get("enum_opts") or model_enum_opts(kg)
    cands = kg.enumerate(**opts)
    rec = db["kernels"]
    costs = []
    for i, c in enumerate(cands):
        if c["klass"] == "rejected":
            costs.append(INF)
            continue
        ns = [rec.get(n) for n in kg.variant_names(i)]
        ns = [INF if v is None else v for v in ns]
        costs.append(min(ns) if ns else INF)
    return kg, cands, costs, db


def spearman(a, b):
    ra = np.argsort(np.argsort(a))
    rb = np.argsort(np.argsort(b))
    return float(np.corrcoef(ra, rb)[0, 1])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--db", default=os.path.join(ROOT, "profiles", "tuning_db"))
    ap.add_argument("--slack", type=float, nargs="+", default=[0.0, 0.25, 0.5, 1.0])
    ap.add_argument("--models", default="candy,efficientvit,yolox,segformer")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_cost_model.json"))
    a = ap.parse_args()
    ctx = K.Context(-1)
    data = {}
    for m in a.models.split(","):
        r = load_model(ctx, m, a.db)
        if r is not None:
            data[m] = r
    feats = {m: graph_features(kg, cands) for m, (kg, cands, costs, db) in data.items()}
    out = {"slack": a.slack, "models": {}, "method": __doc__.strip().splitlines()[0]}
    for m, (kg, cands, costs, db) in data.items():
        t0 = time.perf_counter()
        train = [(cands2[i]["klass"], feats[m2][i], costs2[i]) for m2, (kg2, cands2, costs2, _) in data.items()
                 if m2 != m for i in range(len(cands2)) if costs2[i] < INF]
        model = CostModel().fit(train)
        gen = [i for i, c in enumerate(costs) if c < INF]
        pred = [model.predict(cands[i]["klass"], feats[m][i]) if costs[i] < INF else INF for i in range(len(cands))]
        logerr = [abs(math.log(pred[i] / costs[i])) for i in gen]
        full, _ = kg.select(costs)
        base = kg.operator_aligned()
        greedy = greedy_fusion(cands, costs, kg.prim, kg.outputs)
        res = {"candidates": len(cands), "generable": len(gen), "train_samples": len(train),
               "model_median_abs_log_err": float(np.median(logerr)), "model_spearman": spearman(
                   [pred[i] for i in gen], [costs[i] for i in gen]),
               "optimum_all_ns": full, "operator_aligned_ns": sum(costs[i] for i in base),
               "greedy_fusion_ns": sum(costs[i] for i in greedy), "greedy_fusion_kernels": len(greedy),
               "operator_aligned_kernels": len(base), "pruning": []}
        for s in a.slack:
            keep = set(prune(cands, pred, kg.outputs, base, slack=s))
            sub = [c if i in keep else INF for i, c in enumerate(costs)]
            obj, _ = kg.select(sub)
            res["pruning"].append({"slack": s, "kept": len(keep), "profiled_frac": len(keep) / len(gen),
                                   "optimum_kept_ns": obj, "recall": full / obj,
                                   "profile_s_saved_est": None})
        rec_t = (db.get("tuning_s") or {}).get("profile")
        if rec_t:
            for p in res["pruning"]:
                p["profile_s_saved_est"] = rec_t * (1 - p["profiled_frac"])
        res["eval_s"] = time.perf_counter() - t0
        out["models"][m] = res
        print(m, json.dumps({k: v for k, v in res.items() if k != "pruning"}), flush=True)
        for p in res["pruning"]:
            print("   ", p, flush=True)
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
