#!/usr/bin/env python
"""Replay a paper model's bs-1 orchestration (the exact optimum over the costs of its
committed tuning database) for profilers: plain stream launches (KORCH_EXEC_DIRECT=1), a
few steps, and the names of its most expensive kernels written to a file (for ncu -k).

    python tools/replay_model.py yolox --steps 2 --top 4 --names gpurun_out/yolox_top.txt
    KORCH_EXEC_DIRECT=1 ncu --set full -k regex:'name1|name2' python tools/replay_model.py yolox
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("model")
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--top", type=int, default=4)
    ap.add_argument("--names", default=None, help="write the top kernels' names (one per line) here")
    ap.add_argument("--plan-out", default=None, help="write the plan (candidates, variants, costs) as JSON")
    args = ap.parse_args()
    os.environ.setdefault("KORCH_EXEC_DIRECT", "1")
    import torch

    import paper_2406_09465_b200 as K
    from bench import TUNING_DB, model_enum_opts, model_graph
    from korch_workloads import make_inputs
    from paper_2406_09465_b200 import tunedb

    graph = model_graph(args.model)
    ctx = K.Context(0)
    kg = K.KorchGraph(ctx, graph)
    opts = model_enum_opts(kg)
    cands = kg.enumerate(**opts)
    db = tunedb.load(os.path.join(TUNING_DB, f"{args.model}_b1.json"))
    ok, why = tunedb.usable(db, graph, opts)
    if not ok:
        raise SystemExit(f"no usable tuning database: {why}")
    costs, missing = tunedb.apply(kg, db)
    if missing:
        for i, c in zip(missing, kg.profile(missing)):
            costs[i] = c
    obj, sel = kg.select(costs)
    kg.set_orchestration(sel)
    order = kg.plan()
    top = sorted(order, key=lambda i: -costs[i])[: args.top]
    if args.names:
        with open(args.names, "w") as f:
            for i in top:
                f.write(kg.kernel_name(i) + "\n")
    if args.plan_out:
        kinds = {n["id"]: n["kind"] for n in kg.prim["nodes"]}
        json.dump({"model": args.model, "objective_ns": obj,
                   "kernels": [{"cand": i, "ns": costs[i], "name": kg.kernel_name(i), "variant": kg.variant_info(i)[2],
                                "bytes": cands[i]["bytes"], "flops": cands[i]["flops"],
                                "kinds": [kinds[m] for m in cands[i]["members"]]} for i in order]},
                  open(args.plan_out, "w"), indent=1)
    ins = make_inputs(graph, seed=0)
    dev = K.torch_inputs(graph, {k: v[1] for k, v in ins.items()})
    outs, ws = kg.torch_outputs(), kg.torch_workspace()
    for _ in range(args.steps):
        kg.execute(dev, outs, ws, torch.cuda.current_stream())
    torch.cuda.synchronize()
    print(f"replayed {args.model}: {len(order)} kernels, objective {obj} ns, top {[kg.kernel_name(i) for i in top]}")


if __name__ == "__main__":
    main()
