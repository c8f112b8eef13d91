#!/usr/bin/env python
"""Achieved HBM GB/s of single-kernel layout / reduction candidates at sizes far above L2:
transposes (TR class), column reductions (CR class) and the row reductions (RR) beside
them, every launch variant, cold L2.  Answers "do the layout-sensitive row-template
lowerings need shared-memory staging?" with measurements."""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def cases():
    from korch_workloads.graphs import GraphBuilder

    def one(name, dtype, shape, kind, **attrs):
        b = GraphBuilder(dtype)
        x = b.input("x", shape)
        b.output(b.op(kind, x, **attrs))
        return name, b.build()
    yield one("transpose 2D [8192,8192] bf16", "bf16", [8192, 8192], "Transpose", perm=[1, 0])
    yield one("transpose 2D [8192,8192] f32", "f32", [8192, 8192], "Transpose", perm=[1, 0])
    yield one("NCHW->N(HW)C [1,64,256x256] bf16", "bf16", [1, 64, 65536], "Transpose", perm=[0, 2, 1])
    yield one("N(HW)C->NCHW [1,65536,64] bf16", "bf16", [1, 65536, 64], "Transpose", perm=[0, 2, 1])
    yield one("[16,2048,2048]->[16,2048,2048]^T bf16", "bf16", [16, 2048, 2048], "Transpose", perm=[0, 2, 1])
    yield one("row reduce [65536,1024] f32", "f32", [65536, 1024], "ReduceSum", axis=1)
    yield one("column reduce [1024,65536] f32 axis 0", "f32", [1024, 65536], "ReduceSum", axis=0)
    yield one("column reduce [64,1024,1024] bf16 axis 1", "bf16", [64, 1024, 1024], "ReduceMean", axis=1)
    yield one("copy-like relu [8192,8192] bf16", "bf16", [8192, 8192], "Relu")


def main():
    import paper_2406_09465_b200 as K
    ctx = K.Context(0)
    for name, g in cases():
        kg = K.KorchGraph(ctx, g)
        cands = kg.enumerate()
        for c in cands:
            i = c["index"]
            if c["klass"] == "rejected":
                print(f"{name}: [{i}] rejected: {kg.variant_info(i)}")
                continue
            ns = kg.profile([i], flush_l2=True, trials=5, warmup=1, launches=3)[0]
            nv, best, tag = kg.variant_info(i)
            vc = kg.variant_costs(i)
            print(f"{name}: [{i}] {c['klass']} members={c['members']} bytes={c['bytes']} "
                  f"cold {ns} ns -> {c['bytes'] / ns:.0f} GB/s | best variant '{tag}' | warm per variant {vc}")
    ctx.close()


if __name__ == "__main__":
    main()
