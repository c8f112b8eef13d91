#!/usr/bin/env python
"""Tune one config at a given batch (enumerate, profile, BLP) on cuda:0 and save the plan
in bench.py's --save-selection format, for tools/replay.py under ncu.

    python tools/save_selection.py c2 64 gpurun_out/sel_c2_b64.json
"""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    name, batch, dst = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    import paper_2406_09465_b200 as K
    from bench import config_graph
    graph, _ = config_graph(name, batch)
    kg = K.KorchGraph(K.Context(0), graph)
    cands = kg.enumerate(attention_pairs=True)
    costs = kg.profile()
    _, sel = kg.select(costs)
    kg.set_orchestration(sel)
    order = kg.plan()
    json.dump({"config": name, "batch": batch, "selection": sel, "attention_pairs": True,
               "variants": {str(i): kg.variant_info(i)[1] for i in order},
               "tags": {str(i): kg.variant_info(i)[2] for i in order},
               "kernels": {str(i): kg.kernel_name(i) for i in order},
               "costs_ns": {str(i): costs[i] for i in order}}, open(dst, "w"), indent=1)
    for i in order:
        print(i, costs[i], kg.variant_info(i)[2], cands[i]["flops"])


if __name__ == "__main__":
    main()
