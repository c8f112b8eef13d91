"""Host-side checks of the round-2 code generators (no GPU: the library generates CUDA
source for sm_100a on the CPU).  They pin the launch-variant structure the GPU parity
tests then execute: KB6-D descriptor offsets, clamped guarded loads, the barrier-free
split-K reduction, the vector transpose tiles, and the bench's flop count for window
candidates."""
import re

import pytest

from korch_workloads.graphs import GraphBuilder


@pytest.fixture(scope="module")
def ctx():
    from paper_2406_09465_b200 import Context
    return Context(-1)


def _conv_graph(c, f, r, h, w, pad):
    b = GraphBuilder("bf16")
    x = b.input("x", [1, c, h, w])
    y = b.op("Conv", x, b.input("w", [f, c, r, r], std=0.05), b.input("bias", [f], std=0.1),
             stride=[1, 1], pads=[pad, pad], groups=1)
    b.output(y)
    return b.build()


def _variant_sources(kg, i):
    src = kg.source(i)
    parts = re.split(r"^// variant: ", src, flags=re.M)[1:]
    return {p.split("\n", 1)[0]: p for p in parts}


def test_kb6d_descriptor_offsets(ctx):
    """KB6-D: the A operand of tap (r, s) starts at ((g*R + r)*IW + s)*16 in the staged
    window, LBO = R*IW*16 (channel groups), SBO = 128 (8-pixel row groups), no swizzle;
    N = F rounded up to 16; R*S*C/16 MMAs per tile."""
    from paper_2406_09465_b200 import KorchGraph
    c, f, r = 32, 3, 9
    kg = KorchGraph(ctx, _conv_graph(c, f, r, 20, 200, 4))
    cands = kg.enumerate()
    conv = [x["index"] for x in cands if x["klass"] != "rejected"
            and any(n.startswith("korch_tconv") for n in kg.variant_names(x["index"]))]
    assert conv
    srcs = _variant_sources(kg, conv[0])
    tag, body = next((t, s) for t, s in srcs.items() if t.startswith("tc-direct-conv"))
    iw = 128 + r - 1
    assert f"N=16 CP={c}" in tag and f"{r * r * c // 16} MMAs per tile" in tag
    assert f"{r * iw * 16}, 128, 0)" in body            # A: LBO, SBO, layout 0 (no swizzle)
    assert "umma_desc(spatch + (unsigned)(((2 * kc * %d + r) * %d + s) * 16)" % (r, iw) in body
    assert f"{16 * 16}, 128, 0)" in body                # B: LBO = N * 16


def test_guarded_loads_read_clamped_addresses(ctx):
    """A guarded element load never forms an out-of-tensor address (the clamp of
    `g ? ld1(p + (g ? addr : 0)) : 0`), so a speculated predicated-off load stays inside."""
    from paper_2406_09465_b200 import KorchGraph
    b = GraphBuilder("bf16")
    x = b.input("x", [1, 16, 16, 16])
    y = b.op("Conv", b.op("Relu", x), b.input("w", [16, 1, 3, 3], std=0.3), b.input("bias", [16], std=0.1),
             stride=[1, 1], pads=[1, 1], groups=16)
    b.output(y)
    kg = KorchGraph(ctx, b.build())
    cands = kg.enumerate()
    seen = 0
    for c in cands:
        if c["klass"] == "rejected":
            continue
        for line in kg.source(c["index"]).splitlines():
            m = re.search(r"\(\((\(unsigned\).*?)\)\) \? \(ld1\(p\d+ \+ \(", line)
            if m:
                assert f"(({m.group(1)})) ? (" in line.split("ld1(", 1)[1], line
                seen += 1
    assert seen > 0


def test_split_k_reduction_is_barrier_free(ctx):
    """Cluster split-K variants reduce through st.async into a receive mbarrier armed before
    the dependency wait (relaxed cluster barrier), with no cluster barrier after the main
    loop."""
    from paper_2406_09465_b200 import KorchGraph
    b = GraphBuilder("bf16")
    x = b.input("x", [1, 128, 768])
    b.output(b.op("Add", b.op("MatMul", x, b.input("w", [768, 2304], std=0.03)), b.input("bias", [2304], std=0.1)))
    kg = KorchGraph(ctx, b.build())
    cands = kg.enumerate()
    mm = [c["index"] for c in cands if c["klass"] == "gemm"]
    srcs = {}
    for i in mm:
        srcs.update(_variant_sources(kg, i))
    red = {t: s for t, s in srcs.items() if "red=st.async" in t}
    assert red
    for t, s in red.items():
        k = s.index("pdl_wait();")
        assert "barrier.cluster.arrive.relaxed" in s[:k] and "mbar_expect_tx(rbar" in s[:k], t
        assert "st.async.shared::cluster.mbarrier::complete_tx::bytes" in s[k:], t
        assert "cluster_sync();" not in s[k:], t


def test_vector_transpose_tiles(ctx):
    """Tile transposes offer 8-j vector variants whose staging reads 16 bytes per thread."""
    from paper_2406_09465_b200 import KorchGraph
    b = GraphBuilder("bf16")
    b.output(b.op("Transpose", b.input("x", [256, 512]), perm=[1, 0]))
    kg = KorchGraph(ctx, b.build())
    kg.enumerate()
    tags = list(_variant_sources(kg, 0))
    assert any("VJ=8" in t and "stage=16B" in t for t in tags), tags


def test_bench_linear_flops_for_window_candidates(ctx):
    """bench.linear_flops: 2 * output elements * C/groups * R * S for a convolution."""
    from bench import linear_flops
    from paper_2406_09465_b200 import KorchGraph
    c, f, r, h, w = 32, 3, 9, 20, 200
    kg = KorchGraph(ctx, _conv_graph(c, f, r, h, w, 4))
    cands = kg.enumerate()
    conv_ids = [n["id"] for n in kg.prim["nodes"] if n["kind"] == "conv2d"]
    cand = next(x for x in cands if conv_ids[0] in x["members"])
    assert linear_flops(kg, cand["members"]) == 2.0 * (f * h * w) * c * r * r
