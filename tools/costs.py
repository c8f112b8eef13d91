#!/usr/bin/env python
"""Inspect a saved selection (bench.py --save-selection): the chosen plan and, per output
primitive, the cheapest candidates with their member sets, variant tags and costs."""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    sel = json.load(open(sys.argv[1]))
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    import paper_2406_09465_b200 as K
    from bench import config_graph
    graph, _ = config_graph(sel["config"], sel.get("batch", 1))
    kg = K.KorchGraph(K.Context(-1), graph)
    cands = kg.enumerate(attention_pairs=sel.get("attention_pairs", False))
    costs = sel["all_costs_ns"]
    var = sel["all_variants"]
    kinds = {n["id"]: n["kind"] for n in kg.prim["nodes"]}
    print("plan:", sel["selection"], "sum", sum(costs[i] for i in sel["selection"]))
    for i in sel["selection"]:
        c = cands[i]
        if var[i] >= 0:
            kg.set_variant(i, var[i])
        print(f"  [{i}] {costs[i]:6d} ns  {c['klass']:4s} out p{c['output']} members {c['members']}  {kg.variant_info(i)[2]}")
    by_out = {}
    for c in cands:
        if costs[c["index"]] < (1 << 62):
            by_out.setdefault(c["output"], []).append(c["index"])
    for o in sorted(by_out):
        best = sorted(by_out[o], key=lambda i: costs[i])[:top]
        print(f"p{o} ({kinds[o]}):", ", ".join(f"[{i}] {costs[i]}ns {len(cands[i]['members'])}p" for i in best))


if __name__ == "__main__":
    main()
