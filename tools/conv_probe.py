#!/usr/bin/env python
"""Per-variant costs of a model's single-convolution candidates (all launch variants,
warm graph replay) -- quick look at template choices without a full tuning run.

    python tools/conv_probe.py candy --min-members 1 --max-members 2 --limit 6
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("model")
    ap.add_argument("--max-members", type=int, default=2)
    ap.add_argument("--limit", type=int, default=8)
    ap.add_argument("--prefix", default="korch_dconv")
    ap.add_argument("--cands", default="", help="comma list of candidate indices (instead of the first --limit)")
    a = ap.parse_args()
    import paper_2406_09465_b200 as K
    from bench import model_enum_opts, model_graph
    ctx = K.Context(0)
    kg = K.KorchGraph(ctx, model_graph(a.model))
    cs = kg.enumerate(**model_enum_opts(kg))
    kinds = {n["id"]: n["kind"] for n in kg.prim["nodes"]}
    ids = [c["index"] for c in cs if c["klass"] != "rejected" and len(c["members"]) <= a.max_members
           and any(n.startswith(a.prefix) for n in kg.variant_names(c["index"]))][: a.limit]
    if a.cands:
        ids = [int(x) for x in a.cands.split(",")]
    kg.profile(ids)
    for i in ids:
        src = kg.source(i)
        tags = [l.split("variant: ")[1] for l in src.splitlines() if l.startswith("// variant:")]
        print([kinds[m] for m in cs[i]["members"]], flush=True)
        for v, t in enumerate(tags):
            print(f"   {kg.variant_costs(i)[v]:>9} ns  {t[:110]}", flush=True)


if __name__ == "__main__":
    main()
