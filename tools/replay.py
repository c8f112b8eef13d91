#!/usr/bin/env python
"""Replay a saved orchestration for profilers (ncu): no tuning launches, plain stream
launches (KORCH_EXEC_DIRECT=1), a few steps.

    python bench.py ... --save-selection gpurun_out/sel_c2.json
    KORCH_EXEC_DIRECT=1 ncu ... python tools/replay.py gpurun_out/sel_c2.json --steps 3
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
    ap.add_argument("selection")
    ap.add_argument("--steps", type=int, default=3)
    args = ap.parse_args()
    os.environ.setdefault("KORCH_EXEC_DIRECT", "1")
    import torch

    import paper_2406_09465_b200 as K
    from bench import config_graph
    from korch_workloads import make_inputs

    sel = json.load(open(args.selection))
    graph, _ = config_graph(sel["config"], sel.get("batch", 1))
    ctx = K.Context(0)
    kg = K.KorchGraph(ctx, graph)
    kg.enumerate(attention_pairs=sel.get("attention_pairs", False))
    kg.set_orchestration(sel["selection"], variants=sel.get("variants"))
    ins = make_inputs(graph, seed=0)
    dev = K.torch_inputs(graph, {k: v[1] for k, v in ins.items()})
    outs, ws = kg.torch_outputs(), kg.torch_workspace()
    for _ in range(args.steps):
        kg.execute(dev, outs, ws, torch.cuda.current_stream())
    torch.cuda.synchronize()
    print("replayed", sel["config"], "kernels:", kg.plan())


if __name__ == "__main__":
    main()
