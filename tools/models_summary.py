#!/usr/bin/env python
"""Collect the per-model result lines of a `bench.py --models ...` log (the
"[models] {...}" lines written as each model finishes) into one JSON file.

    python tools/models_summary.py gpurun_out/models.log profiles/r01_models.json
"""
from __future__ import annotations

import json
import sys


def main():
    src, dst = sys.argv[1], sys.argv[2]
    res = {}
    for line in open(src):
        if line.startswith("[models] {"):
            res.update(json.loads(line[len("[models] "):]))
    out = {"source": "bench.py --models (bs 1, paper input sizes; one B200)", "models": res}
    json.dump(out, open(dst, "w"), indent=1)
    for name, v in res.items():
        print(f"{name:14s} {v['latency_ms']:.3f} ms ({v['kernels']} kernels)  one-kernel-per-operator "
              f"{v['operator_aligned_ms']:.3f} ms ({v['operator_aligned_kernels']})  x{v['speedup_vs_operator_aligned']:.2f}"
              f"  oracle rel err {v.get('oracle_rel_err', float('nan')):.1e}  blp optimal {v.get('blp_optimal')}")


if __name__ == "__main__":
    main()
