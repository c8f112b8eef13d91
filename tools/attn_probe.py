#!/usr/bin/env python
"""Fused two-GEMM attention candidates (N2) of C2: their profiled costs next to the split
plan's kernels, and a saved selection that forces the largest attention candidate into
the plan so that tools/replay.py can put it under ncu:

    python tools/attn_probe.py --batch 1 --save gpurun_out/sel_attn.json
    KORCH_EXEC_DIRECT=1 ncu -k regex:korch_attn -c 1 --set full ... python tools/replay.py gpurun_out/sel_attn.json
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
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--save", default=None)
    args = ap.parse_args()
    import paper_2406_09465_b200 as K
    from bench import config_graph
    graph, _ = config_graph("c2", args.batch)
    ctx = K.Context(0)
    kg = K.KorchGraph(ctx, graph)
    cands = kg.enumerate(attention_pairs=True)
    costs = kg.profile()
    obj, sel = kg.select(costs)
    print(f"BLP plan {sel}: {obj} ns")
    for i in sel:
        print(f"  [{i}] {costs[i]} ns {cands[i]['klass']} {len(cands[i]['members'])}p  {kg.variant_info(i)[2]}")
    att = [c for c in cands if c["klass"] == "gemm" and "attention" in kg.variant_info(c["index"])[2]]
    for c in sorted(att, key=lambda c: costs[c["index"]]):
        print(f"attn [{c['index']}] {costs[c['index']]} ns members {c['members']} -> p{c['output']}  "
              f"{kg.variant_info(c['index'])[2]}")
    if att and args.save:
        big = max(att, key=lambda c: (len(c["members"]), -costs[c["index"]]))
        forced = list(costs)
        forced[big["index"]] = 1
        _, fsel = kg.select(forced)
        print(f"forced plan {fsel}: {sum(costs[i] for i in fsel)} ns (measured costs)")
        json.dump({"config": "c2", "batch": args.batch, "selection": fsel, "attention_pairs": True,
                   "variants": {str(i): kg.variant_info(i)[1] for i in fsel}}, open(args.save, "w"))
    ctx.close()


if __name__ == "__main__":
    main()
