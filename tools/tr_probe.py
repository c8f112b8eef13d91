#!/usr/bin/env python
"""Launch the vector-tile transpose of [8192, 8192] bf16 a few times (for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import paper_2406_09465_b200 as K
    from korch_workloads.graphs import GraphBuilder
    b = GraphBuilder("bf16")
    b.output(b.op("Transpose", b.input("x", [8192, 8192]), perm=[1, 0]))
    ctx = K.Context(0)
    kg = K.KorchGraph(ctx, b.build())
    kg.enumerate()
    nv = kg.variant_info(0)[0]
    for v in range(nv):
        kg.set_variant(0, v)
        if "VJ=8" in kg.variant_info(0)[2] and "TA=64" in kg.variant_info(0)[2]:
            break
    print("variant", kg.variant_info(0)[2], kg.profile([0], flush_l2=True, trials=3, tune=False))


if __name__ == "__main__":
    main()
