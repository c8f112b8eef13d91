#!/usr/bin/env python
"""Summarise ncu captures into committed profiles/ files.

    python tools/ncu_summary.py full  gpurun_out/prof.ncu-rep   profiles/r01_c2_ncu_full.json
    python tools/ncu_summary.py launches gpurun_out/launches.csv profiles/r01_c2_launches.json

`full` reads `ncu -i <rep> --page raw --csv` and keeps, per kernel (averaged over its
captured launches), the duration, DRAM bytes read/written, tensor-pipe and DRAM
throughput percentages, registers and warps; `launches` reads a
gpu__time_duration.sum launch list and reports each kernel's share of the step.
"""
from __future__ import annotations

import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
         "ns": 1, "us": 1e3, "usecond": 1e3, "msecond": 1e6, "nsecond": 1, "ms": 1e6}

METRICS = {
    "duration_ns": "gpu__time_duration.sum",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "tensor_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "regs": "launch__registers_per_thread",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "smem_dyn": "launch__shared_mem_per_block_dynamic",
}


def _num(v, unit):
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return None
    return x * SCALE.get(unit, 1)


def full(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    acc = defaultdict(lambda: defaultdict(list))
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        for key, m in METRICS.items():
            if m in hdr:
                i = hdr.index(m)
                v = _num(r[i], units[i])
                if v is not None:
                    acc[name][key].append(v)
    kernels = {}
    for name, d in acc.items():
        k = {key: sum(v) / len(v) for key, v in d.items()}
        k["dram_bytes"] = k.get("dram_read", 0) + k.get("dram_write", 0)
        k["launches_captured"] = len(next(iter(d.values())))
        kernels[name] = k
    json.dump({"source": rep, "kind": "ncu --set full --clock-control none", "kernels": kernels},
              open(out, "w"), indent=1)
    return kernels


def launches(path, out):
    text = open(path).read()
    start = text.index('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    per = defaultdict(list)
    order = []
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        n = r["Kernel Name"]
        if n not in per:
            order.append(n)
        per[n].append(_num(r["Metric Value"], r["Metric Unit"]))
    tot = sum(sum(v) / len(v) for v in per.values())
    res = {"source": path, "kind": "ncu --metrics gpu__time_duration.sum --clock-control none (cold, serialised)",
           "step_ns_sum": tot,
           "kernels": [{"name": n, "launches": len(per[n]), "avg_ns": sum(per[n]) / len(per[n]),
                        "share": (sum(per[n]) / len(per[n])) / tot} for n in order]}
    json.dump(res, open(out, "w"), indent=1)
    return res


if __name__ == "__main__":
    mode, src, dst = sys.argv[1:4]
    r = full(src, dst) if mode == "full" else launches(src, dst)
    print(json.dumps(r, indent=1)[:3000])
