#!/usr/bin/env python
"""Markdown tables from a bench.py JSON line (for DESIGN.md's measured section).

    python tools/bench_table.py profiles/r02_bench.json
"""
from __future__ import annotations

import json
import sys


def main():
    d = json.load(open(sys.argv[1]))
    print(f"C2 bs 1: {d['value'] * 1e3:.1f} us cold-L2 ({d.get('warm_l2_ms_per_step', 0) * 1e3:.1f} us warm), "
          f"e2e {d['e2e']['value'] * 1e3:.1f} us, {d['kernels_per_step']} kernels, roofline frac "
          f"{d['roofline']['frac']:.3f}, one kernel per operator {d['selection']['operator_aligned_ms'] * 1e3:.1f} us, "
          f"clocks {d['clocks']}")
    print()
    print("| model | latency ms (p10-p90) | kernels | one kernel per operator ms | speedup | fission + greedy ms | "
          "multi-output (N1) ms | e2e ms | oracle rel L2 / max | optimal |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    for m, v in (d.get("models") or {}).items():
        if "error" in v:
            print(f"| {m} | error: {v['error'][:80]} |")
            continue
        dist = v["latency_ms_dist"]
        gf = v.get("greedy_fusion", {})
        mo = v.get("multi_output", {})
        print(f"| {m} | {v['latency_ms']:.3f} ({dist['p10']:.3f}-{dist['p90']:.3f}) | {v['kernels']} | "
              f"{v['operator_aligned_ms']:.3f} ({v['operator_aligned_kernels']}) | {v['speedup_vs_operator_aligned']:.2f}x | "
              f"{gf.get('latency_ms', float('nan')):.3f} ({gf.get('kernels')}) | "
              f"{mo.get('latency_ms', float('nan')):.3f} | {v['e2e_ms']:.3f} | "
              f"{v.get('oracle_rel_l2', float('nan')):.1e} / {v.get('oracle_rel_err', float('nan')):.1e} | {v['blp_optimal']} |")
    print()
    print("| model | dominant kernel | class | achieved | frac | variant |")
    print("|---|---|---|---|---|---|")
    for m, v in (d.get("models") or {}).items():
        if "dominant" in v:
            r = v["dominant"]
            print(f"| {m} | {r['name']} | {r['class']} | {r['achieved']:.1f} {r['unit']} | {r['frac']:.3f} | {r['variant'][:70]} |")
    bt = d.get("model_batch_throughput") or {}
    if bt:
        print()
        print("| model | global batch | GPUs | local batch | ms | images/s | kernels |")
        print("|---|---|---|---|---|---|---|")
        for m, v in bt.items():
            if "error" in v:
                print(f"| {m} | error: {v['error'][:80]} |")
                continue
            print(f"| {m} | {v['global_batch']} | {v['n_gpus']} | {v['local_batch']} | {v['ms']:.3f} | "
                  f"{v['throughput']['value']:.0f} | {v['kernels']} |")


if __name__ == "__main__":
    main()
