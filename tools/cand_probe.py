#!/usr/bin/env python
"""Per-launch-variant costs of chosen candidates of a benchmark config (where does a
candidate's time go?), and a launch-only mode for ncu.

    python tools/cand_probe.py c2 79 90                 # every variant's warm cost
    python tools/cand_probe.py c2 90 --variant 4 --launches 3   # just launch it (under ncu)
"""
from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("cands", type=int, nargs="+")
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--variant", type=int, default=None)
    ap.add_argument("--launches", type=int, default=3)
    a = ap.parse_args()
    import paper_2406_09465_b200 as K
    from bench import config_graph
    graph, _ = config_graph(a.config, a.batch)
    ctx = K.Context(0)
    kg = K.KorchGraph(ctx, graph)
    cands = kg.enumerate(attention_pairs=True)
    kg.compile(a.cands)
    for i in a.cands:
        if a.variant is not None:
            kg.set_variant(i, a.variant)
            for _ in range(a.launches):
                kg.profile([i], warmup=1, launches=1, trials=1, tune=False)
            print("launched", i, kg.variant_info(i)[2])
            continue
        kg.profile([i])
        warm = kg.variant_costs(i)
        best = kg.variant_info(i)[1]
        tags = []
        for v in range(len(warm)):
            kg.set_variant(i, v)
            tags.append(kg.variant_info(i)[2])
        kg.set_variant(i, best)
        cold = kg.profile([i], flush_l2=True, trials=5, tune=False)[0]
        print(f"cand {i}: {len(cands[i]['members'])} members, bytes {cands[i]['bytes']}, chosen v{best}, "
              f"cold {cold} ns")
        for v, (ns, tag) in enumerate(zip(warm, tags)):
            print(f"  v{v}: {ns} ns  {tag}")


if __name__ == "__main__":
    main()
