#!/usr/bin/env python
"""Per-variant timings of GEMM candidates across shapes (where does a small-M GEMM's time
go?).  Prints, for the MatMul-alone candidate and the fully fused candidate of
MatMul(x, W) + bias + residual, every launch variant's profiled ns (warm, graph replay)."""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def graph(m, k, n, epilogue=True):
    from korch_workloads.graphs import GraphBuilder
    b = GraphBuilder("bf16")
    x = b.input("x", [1, m, k])
    w = b.input("w", [k, n], std=k ** -0.5)
    y = b.op("MatMul", x, w)
    if epilogue:
        bias = b.input("bias", [n], std=0.1)
        r = b.input("r", [1, m, n])
        y = b.op("Add", y, bias)
        y = b.op("Add", y, r)
    b.output(y)
    return b.build()


def main():
    import paper_2406_09465_b200 as K
    from korch_workloads.graphs import GraphBuilder
    ctx = K.Context(0)
    # launch floor: a trivial elementwise kernel
    b = GraphBuilder("bf16")
    b.output(b.op("Relu", b.input("x", [1, 8])))
    kg = K.KorchGraph(ctx, b.build())
    kg.enumerate()
    print("floor (relu[1,8]) ns:", kg.profile()[0])
    shapes = [(128, 64, 768), (128, 256, 768), (128, 768, 768), (128, 768, 2304), (128, 3072, 768),
              (512, 768, 768), (2048, 768, 2304)]
    for (m, k, n) in shapes:
        kg = K.KorchGraph(ctx, graph(m, k, n))
        cands = kg.enumerate()
        costs = kg.profile()
        for c in cands:
            if c["klass"] != "gemm":
                continue
            nv, best, _ = kg.variant_info(c["index"])
            vc = kg.variant_costs(c["index"])
            tags = []
            for v in range(nv):
                kg.set_variant(c["index"], v)
                t = kg.variant_info(c["index"])[2]
                tags.append(t.split(" M=")[0].replace("gemm BM=128 ", "").replace(" BK=64", "")
                            .replace(" A=K-major B=N-major", "") + (" cl" if "epi=cl" in t else ""))
            kg.set_variant(c["index"], best)
            row = "  ".join(f"{t}:{ns}" for t, ns in sorted(zip(tags, vc), key=lambda z: z[1]))
            print(f"M={m} K={k} N={n} members={c['members']} best={costs[c['index']]} ns | {row}")


if __name__ == "__main__":
    main()
