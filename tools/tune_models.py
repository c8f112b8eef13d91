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
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2406_09465_b200 as K  # noqa: E402
import paper_2406_09465_b200.select as S  # noqa: E402
from paper_2406_09465_b200 import tunedb  # noqa: E402
from bench import model_enum_opts, model_graph  # noqa: E402


def tune(name, batch, out_dir, max_outputs=1):
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
    t1 = time.perf_counter()
    kg.compile()
    t_comp = time.perf_counter() - t1
    t1 = time.perf_counter()
    costs = kg.profile()
    t_prof = time.perf_counter() - t1
    t1 = time.perf_counter()
    obj, sel = kg.select(costs)
    t_sel = time.perf_counter() - t1
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
    a = ap.parse_args()
    for b in [int(x) for x in a.batch.split(",")]:
        for m in a.models:
            tune(m, b, a.out, a.max_outputs)


if __name__ == "__main__":
    main()
