"""GPU parity: the CUDA path (through the C ABI) against the oracle, element by element,
on the same seeded inputs.  Tolerances (BASELINE.json north star, reading A21):
per output tensor ||gpu - oracle||_inf <= rtol * ||oracle||_inf, rtol = 1e-4 (fp32
storage) / 2e-2 (bf16 storage); layout-only graphs bit-exact."""
import numpy as np
import pytest

from korch_workloads import c1_softmax_layernorm, c2_vit_attention, make_inputs
from korch_workloads.graphs import GraphBuilder
from oracle.enumeration import PGraph, candidates, convex_sets_from_states, execution_states
from oracle.evaluate import eval_orchestration, eval_primitive_graph
from oracle.fission import fission

torch = pytest.importorskip("torch")

RTOL = {"f32": 1e-4, "bf16": 2e-2}


@pytest.fixture(scope="module")
def ctx():
    from paper_2406_09465_b200 import Context
    return Context(0)


class Case:
    """One graph loaded both ways: the library (device) and the oracle (host, fp64)."""

    def __init__(self, ctx, graph, seed=0, max_prims=16):
        from paper_2406_09465_b200 import KorchGraph, torch_inputs
        self.graph = graph
        self.kg = KorchGraph(ctx, graph)
        self.cands = self.kg.enumerate(max_prims=max_prims)
        self.pg = fission(graph)
        self.G = PGraph(self.pg)
        self.ref = candidates(self.G, convex_sets_from_states(execution_states(self.G)), max_prims=max_prims)
        assert [(tuple(c["members"]), c["output"]) for c in self.cands] == [(tuple(m), o) for m, o in self.ref]
        ins = make_inputs(graph, seed=seed)
        self.values = {k: v[0] for k, v in ins.items()}
        self.dev_in = torch_inputs(graph, {k: v[1] for k, v in ins.items()})
        self.storage = graph["dtype"]

    def completion(self, must):
        """A feasible selection containing `must`, completed with generable producers."""
        gen = {c["index"] for c in self.cands if c["klass"] != "rejected"}
        prod = {}
        for c in self.cands:
            if c["index"] in gen:
                prod.setdefault(c["output"], []).append(c["index"])
        for o in prod:  # prefer the smallest producer
            prod[o].sort(key=lambda i: (len(self.cands[i]["members"]), i))
        sel, have = list(must), {self.cands[i]["output"] for i in must}
        need = [j for i in must for j in self.cands[i]["inputs"]] + list(self.kg.outputs)
        while need:
            t = need.pop()
            if t in have:
                continue
            i = prod[t][0]
            sel.append(i)
            have.add(t)
            need.extend(self.cands[i]["inputs"])
        return sorted(set(sel))

    def run(self, sel):
        self.kg.set_orchestration(sel)
        outs = self.kg.torch_outputs()
        ws = self.kg.torch_workspace()
        self.kg.execute(self.dev_in, outs, ws, torch.cuda.current_stream())
        torch.cuda.synchronize()
        return [o.float().cpu().numpy().astype(np.float64) for o in outs]

    def oracle(self, sel):
        return eval_orchestration(self.pg, self.ref, sel, self.values, self.G.topo_index, self.storage)

    def check(self, sel, rtol=None, exact=False):
        got = self.run(sel)
        ref = self.oracle(sel)
        rtol = RTOL[self.storage] if rtol is None else rtol
        for k, o in enumerate(self.kg.outputs):
            r = ref[o]
            assert got[k].shape == r.shape
            if exact:
                np.testing.assert_array_equal(got[k], r)
            else:
                err = np.max(np.abs(got[k] - r))
                scale = np.max(np.abs(r))
                assert err <= rtol * scale, f"sel={sel}: err {err:.3e} > {rtol} * {scale:.3e}"
        return got, ref


@pytest.mark.gpu
def test_c1_every_candidate(ctx):
    """Every C1 candidate kernel (all 120) runs inside a feasible orchestration and matches."""
    c = Case(ctx, c1_softmax_layernorm())
    gen = [x["index"] for x in c.cands if x["klass"] != "rejected"]
    assert len(gen) == len(c.cands) == 120
    for i in gen:
        c.check(c.completion([i]))


@pytest.mark.gpu
@pytest.mark.parametrize("rows,cols", [(4, 128), (1000, 128), (37, 100), (3, 2048), (5, 4096), (64, 96)])
def test_c1_shapes_whole_and_singletons(ctx, rows, cols):
    """Several tiles, ragged tails (masked rows), block-reduce rows (> 32 threads)."""
    c = Case(ctx, c1_softmax_layernorm(rows=rows, cols=cols))
    whole = [x["index"] for x in c.cands if len(x["members"]) == c.kg.n_prims]
    c.check(whole)
    c.check(c.kg.singletons())
    c.check(c.kg.operator_aligned())


@pytest.mark.gpu
def test_c1_invariants_on_gpu(ctx):
    """Softmax rows sum to 1 (fp32 <= 1e-5) and LayerNorm (eps=0, no affine) has mean 0 / var 1."""
    g = c1_softmax_layernorm(rows=64, cols=128, affine=False, eps=0.0)
    c = Case(ctx, g)
    whole = [x["index"] for x in c.cands if len(x["members"]) == c.kg.n_prims][0]
    y = c.run([whole])[0]
    np.testing.assert_allclose(y.mean(1), 0, atol=1e-5)
    np.testing.assert_allclose(y.var(1), 1, atol=1e-4)
    g2 = GraphBuilder("f32")
    x = g2.input("x", [64, 128])
    g2.output(g2.op("Softmax", x, axis=1))
    c2 = Case(ctx, g2.build())
    s = c2.run(c2.kg.singletons())[0]
    np.testing.assert_allclose(s.sum(1), 1, atol=1e-5)


@pytest.mark.gpu
def test_full_pipeline_c1(ctx):
    """enumerate -> profile -> BLP -> execute; the chosen orchestration matches the oracle
    and its cost is no worse than the operator-aligned baseline's."""
    c = Case(ctx, c1_softmax_layernorm())
    costs = c.kg.profile()
    assert all(0 < x < (1 << 62) for x in costs)
    obj, sel = c.kg.select(costs)
    base = c.kg.operator_aligned()
    assert obj <= sum(costs[i] for i in base)
    c.check(sel)


def _layout_graph(dtype):
    b = GraphBuilder(dtype)
    x = b.input("x", [4, 6, 8, 16])
    y = b.op("Transpose", x, perm=[0, 2, 1, 3])
    y = b.op("Reshape", y, shape=[32, 96])
    y = b.op("Slice", y, axis=1, start=16, end=80)
    y = b.op("Pad", y, pads=[[1, 0], [0, 2]], mode="constant", value=0.0)
    y = b.op("Transpose", y, perm=[1, 0])
    b.output(y)
    return b.build()


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_layout_only_bit_exact(ctx, dtype):
    c = Case(ctx, _layout_graph(dtype))
    for i in [x["index"] for x in c.cands if x["klass"] != "rejected"]:
        c.check(c.completion([i]), exact=True)


def _every_variant(c, idx, exact):
    for i in idx:
        nv, _, _ = c.kg.variant_info(i)
        for v in range(nv):
            c.kg.set_variant(i, v)
            c.check(c.completion([i]), exact=exact)


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_layout_every_variant_bit_exact(ctx, dtype):
    """Every launch variant, including the shared-memory staged tiles (TR), of every
    candidate of the layout graph: bit-exact."""
    c = Case(ctx, _layout_graph(dtype))
    tiles = 0
    for x in c.cands:
        if x["klass"] == "rejected":
            continue
        nv = c.kg.variant_info(x["index"])[0]
        for v in range(nv):
            c.kg.set_variant(x["index"], v)
            tiles += "tile" in c.kg.variant_info(x["index"])[2]
    assert tiles > 0
    _every_variant(c, [x["index"] for x in c.cands if x["klass"] != "rejected"], exact=True)


def _transpose_chain(dtype, n, a, b):
    """Ragged transposes (tile edges in both axes) feeding elementwise work, and an
    NCHW <-> tokens round trip with a reflect pad (guarded staged loads)."""
    gb = GraphBuilder(dtype)
    x = gb.input("x", [n, a, b])
    r = gb.input("r", [n, b, a])
    bias = gb.input("bias", [a], std=0.1)
    y = gb.op("Transpose", x, perm=[0, 2, 1])               # [n, b, a]
    y = gb.op("Add", y, r)
    y = gb.op("Add", y, bias)
    y = gb.op("GELU", y)
    z = gb.op("Reshape", y, shape=[n, b, a, 1])
    z = gb.op("Transpose", z, perm=[0, 2, 1, 3])            # [n, a, b, 1]
    z = gb.op("Pad", z, pads=[[0, 0], [0, 0], [1, 1], [0, 0]], mode="reflect")
    z = gb.op("Relu", z)
    gb.output(z)
    return gb.build()


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("n,a,b", [(1, 64, 96), (2, 45, 70), (3, 130, 33)])
def test_transpose_tiles_every_variant(ctx, dtype, n, a, b):
    c = Case(ctx, _transpose_chain(dtype, n, a, b))
    idx = [x["index"] for x in c.cands if x["klass"] in ("pw", "rr")]
    assert any("tile" in _tags(c, i) for i in idx)
    _every_variant(c, idx, exact=False)


def _column_graph(kind, dtype, shape, axis):
    gb = GraphBuilder(dtype)
    x = gb.input("x", shape)
    if kind == "Softmax":
        y = gb.op("Softmax", gb.op("MulC", x, c=0.5), axis=axis)     # reduce + broadcast back
    else:
        y = gb.op("Relu", gb.op(kind, gb.op("Neg", x), axis=axis))
    gb.output(y)
    return gb.build()


@pytest.mark.gpu
@pytest.mark.parametrize("kind,dtype,shape,axis", [("ReduceSum", "f32", [200, 96], 0),
                                                   ("ReduceMean", "bf16", [3, 70, 50], 1),
                                                   ("ReduceMax", "f32", [130, 2, 33], 0),
                                                   ("Softmax", "f32", [64, 100], 0),
                                                   ("Softmax", "bf16", [2, 96, 40], 1)])
def test_column_reductions_every_variant(ctx, kind, dtype, shape, axis):
    """Reductions along a non-innermost axis: every variant, including the column mapping
    (CR: lanes over consecutive rows, shared-memory row combine, ragged row blocks)."""
    c = Case(ctx, _column_graph(kind, dtype, shape, axis))
    idx = [x["index"] for x in c.cands if x["klass"] == "rr"]
    assert any("col" in _tags(c, i) for i in idx)
    _every_variant(c, idx, exact=False)


def _contraction_graph(dtype, batch, tokens, d):
    """EfficientViT's K^T V at a large token:d ratio: K = tokens, N = d + 1."""
    gb = GraphBuilder(dtype)
    k = gb.input("k", [batch, tokens, d])
    v = gb.input("v", [batch, tokens, d + 1])
    kt = gb.op("Transpose", gb.op("Relu", k), perm=[0, 2, 1])
    y = gb.op("MatMul", kt, v)
    gb.output(gb.op("MulC", y, c=1.0 / tokens))
    return gb.build()


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_large_k_contraction_as_row_reduction(ctx, dtype):
    c = Case(ctx, _contraction_graph(dtype, 2, 8192, 16))
    gen = [x["index"] for x in c.cands if x["klass"] != "rejected"]
    assert any(len(x["members"]) >= 3 and x["klass"] == "rr" for x in c.cands)
    _every_variant(c, gen, exact=False)


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_long_elementwise_rows_chunked(ctx, dtype):
    """Rows longer than the register tile (L = 20480) are cut into chunks."""
    gb = GraphBuilder(dtype)
    x = gb.input("x", [2, 3, 20480])
    gb.output(gb.op("GELU", gb.op("Add", x, gb.input("b", [20480], std=0.1))))
    c = Case(ctx, gb.build())
    gen = [x["index"] for x in c.cands if x["klass"] != "rejected"]
    assert len(gen) == len(c.cands)
    _every_variant(c, gen, exact=False)


def _ln_linear_graph(m, k, n, batch=1):
    b = GraphBuilder("bf16")
    x = b.input("x", [batch, m, k])
    g = b.input("g", [k], mean=1.0, std=0.1)
    be = b.input("be", [k], std=0.1)
    w = b.input("w", [k, n], std=k ** -0.5)
    bias = b.input("bias", [n], std=0.1)
    y = b.op("LayerNorm", x, g, be, axis=-1, eps=1e-5)
    y = b.op("MatMul", y, w)
    y = b.op("Add", y, bias)
    b.output(b.op("GELU", y))
    return b.build()


@pytest.mark.gpu
@pytest.mark.parametrize("m,k,n,batch", [(128, 768, 256, 1), (200, 256, 48, 1), (70, 64, 200, 2), (200, 256, 128, 1)])
def test_prologue_gemm_every_variant(ctx, m, k, n, batch):
    """KB5-P: LayerNorm computed in the GEMM's A prologue (resident swizzled A tile),
    ragged M and N, batched, every launch variant -- including KB5-PC, the cluster-shared
    prologue (one RP-row slice per CTA, TMA store to the scratch, multicast back), on a
    full and a ragged (M = 200) tile row."""
    c = Case(ctx, _ln_linear_graph(m, k, n, batch))
    idx = [x["index"] for x in c.cands if "prologue" in _tags(c, x["index"])]
    assert any(len(c.cands[i]["members"]) >= 12 for i in idx)
    if n in (256, 128):
        assert any("cluster-prologue CN=8" in _tags(c, i) for i in idx)
    _every_variant(c, idx, exact=False)


def _tags(c, i):
    nv, ch, _ = c.kg.variant_info(i)
    t = []
    for v in range(nv):
        c.kg.set_variant(i, v)
        t.append(c.kg.variant_info(i)[2])
    if ch >= 0:
        c.kg.set_variant(i, ch)
    return " ".join(t)


@pytest.mark.gpu
def test_misc_memory_bound_ops(ctx):
    b = GraphBuilder("f32")
    x = b.input("x", [2, 8, 10, 12])
    g = b.input("g", [8], mean=1.0, std=0.1)
    be = b.input("be", [8], std=0.1)
    y = b.op("InstanceNorm", x, g, be, eps=1e-5)
    y = b.op("Relu", y)
    y = b.op("Pad", y, pads=[[0, 0], [0, 0], [1, 1], [1, 1]], mode="reflect")
    y = b.op("GELU", y)
    y = b.op("Upsample2x", y)
    b.output(y)
    c = Case(ctx, b.build())
    gen = [x["index"] for x in c.cands if x["klass"] != "rejected"]
    assert len(gen) > 0
    for i in gen[:: max(1, len(gen) // 40)]:
        c.check(c.completion([i]))
    c.check(c.kg.operator_aligned())


@pytest.mark.gpu
@pytest.mark.parametrize("shape", [(1, 32, 20, 24, 32, 3, 1, 32), (1, 3, 16, 40, 16, 3, 1, 1), (2, 12, 9, 33, 8, 5, 2, 1),
                                   (1, 16, 8, 64, 16, 7, 3, 16)])
def test_simt_conv_row_vector_reads(ctx, shape):
    """SIMT convolutions (depthwise / few channels per group) with stride 1 along W read a
    thread's 8-output window row with one unaligned 16-byte load (interior) or guarded
    element loads (edges, ragged row tail): every generable candidate against the oracle."""
    n, c_, h, w, f, k, p, groups = shape
    b = GraphBuilder("bf16")
    x = b.input("x", [n, c_, h, w])
    wt = b.input("w", [f, c_ // groups, k, k], std=0.3)
    bias = b.input("bias", [f], std=0.1)
    y = b.op("Conv", x, wt, bias, stride=[1, 1], pads=[p, p], groups=groups)
    b.output(b.op("SiLU", y))
    c = Case(ctx, b.build())
    gen = [x["index"] for x in c.cands if x["klass"] != "rejected"]
    assert gen
    for i in gen:
        nv, _, _ = c.kg.variant_info(i)
        for v in range(nv):
            c.kg.set_variant(i, v)
            c.check(c.completion([i]))


def _cnn_graph(dtype="bf16"):
    b = GraphBuilder(dtype)
    x = b.input("x", [1, 16, 20, 24])
    w = b.input("w", [32, 16, 3, 3], std=0.08)
    bias = b.input("bias", [32], std=0.1)
    y = b.op("Conv", x, w, bias, stride=[1, 1], pads=[1, 1], groups=1)
    y = b.op("SiLU", y)
    y = b.op("MaxPool", y, k=3, stride=2, pad=1)                      # [1,32,10,12]
    dw = b.input("dw", [32, 1, 3, 3], std=0.3)
    z = b.op("Conv", y, dw, stride=[2, 2], pads=[1, 1], groups=32)    # depthwise, stride 2
    z = b.op("HardSwish", z)
    pw = b.input("pw", [24, 32, 1, 1], std=0.2)
    z = b.op("Conv", z, pw, stride=[1, 1], pads=[0, 0], groups=1)     # pointwise
    z = b.op("Upsample2x", z)                                          # [1,24,10,12]
    y2 = b.op("Slice", y, axis=1, start=0, end=8)
    c = b.op("Concat", z, y2, axis=1)                                  # [1,32,10,12]
    g = b.input("g", [32], mean=1.0, std=0.1)
    be = b.input("be", [32], std=0.1)
    c = b.op("InstanceNorm", c, g, be, eps=1e-5)
    c = b.op("Relu", c)
    c = b.op("Pad", c, pads=[[0, 0], [0, 0], [1, 1], [1, 1]], mode="reflect")
    w3 = b.input("w3", [3, 32, 3, 3], std=0.05)
    c = b.op("Conv", c, w3, stride=[1, 1], pads=[0, 0], groups=1)
    b.output(c)
    return b.build()


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_cnn_primitives(ctx, dtype):
    """Dense / depthwise / strided / pointwise convolutions (+bias), max-pool, concat,
    slice, upsample, InstanceNorm, reflect pad, SiLU, HardSwish: every generable
    candidate inside a feasible orchestration, then the BLP plan."""
    c = Case(ctx, _cnn_graph(dtype))
    gen = [x["index"] for x in c.cands if x["klass"] != "rejected"]
    assert len(gen) > 50
    for i in gen:
        c.check(c.completion([i]))
    costs = c.kg.profile()
    obj, sel = c.kg.select(costs)
    c.check(sel)


def _conv_graph(n, c, h, w, f, k, s, p):
    b = GraphBuilder("bf16")
    x = b.input("x", [n, c, h, w])
    wt = b.input("w", [f, c, k, k], std=(c * k * k) ** -0.5)
    bias = b.input("b", [f], std=0.1)
    y = b.op("Conv", x, wt, bias, stride=[s, s], pads=[p, p], groups=1)
    y = b.op("Relu", y)
    b.output(y)
    return b.build()


@pytest.mark.gpu
@pytest.mark.parametrize("shape", [(1, 16, 20, 24, 32, 3, 1, 1), (1, 32, 17, 19, 48, 3, 2, 1), (2, 64, 14, 14, 160, 1, 1, 0),
                                   (1, 128, 28, 28, 128, 3, 1, 1), (1, 32, 30, 30, 64, 5, 2, 2),
                                   (1, 32, 16, 32, 3, 9, 1, 4), (2, 16, 8, 16, 48, 5, 1, 2)])
def test_conv_igemm_every_variant(ctx, shape):
    """tcgen05 implicit-GEMM convolution (KB6): every launch variant of every conv
    candidate (conv alone, + bias, + bias + ReLU), strides, zero padding, filter / pixel
    tails, batch > 1, cluster split-K, and the 16-byte unaligned row reads of stride-1
    convolutions with OW % 8 == 0 (9x9 / 5x5 windows: groups at the padded edges fall
    back to element loads)."""
    c = Case(ctx, _conv_graph(*shape))
    convs = [x for x in c.cands if x["klass"] == "gemm"]
    assert convs, "conv candidates must be accepted by the implicit-GEMM template"
    for x in convs:
        nv, _, _ = c.kg.variant_info(x["index"])
        for v in range(nv):
            c.kg.set_variant(x["index"], v)
            c.check(c.completion([x["index"]]))


@pytest.mark.gpu
@pytest.mark.parametrize("kw", [dict(), dict(batch=2, seq=64, hidden=256, heads=4), dict(seq=200, hidden=192, heads=3)])
def test_fused_attention_candidates(ctx, kw):
    """NEXT item N2: two-GEMM attention candidates (QK^T -> in-tile softmax ->
    P V, P kept in shared memory) against the oracle, and a BLP plan that may use them."""
    from paper_2406_09465_b200 import KorchGraph
    g = c2_vit_attention(**kw)
    c = Case(ctx, g)
    c.cands = c.kg.enumerate(attention_pairs=True)
    c.ref = candidates(c.G, convex_sets_from_states(execution_states(c.G)), 16, attention_pairs=True)
    assert [(tuple(x["members"]), x["output"]) for x in c.cands] == [(tuple(m), o) for m, o in c.ref]
    att = [x["index"] for x in c.cands if x["n_dense_linear"] == 2 and x["klass"] == "gemm"]
    if kw.get("seq", 128) % 64 == 0:
        assert att
    for i in att:
        nv, _, _ = c.kg.variant_info(i)   # one row per thread, and the 4-threads-per-row softmax
        for v in range(nv):
            c.kg.set_variant(i, v)
            c.check(c.completion([i]))
    costs = c.kg.profile()
    obj, sel = c.kg.select(costs)
    c.check(sel)


@pytest.mark.gpu
def test_c2_every_gemm_candidate(ctx):
    """Every tcgen05 GEMM candidate of the ViT attention layer (fused views + epilogues)."""
    c = Case(ctx, c2_vit_attention())
    gem = [x["index"] for x in c.cands if x["klass"] == "gemm"]
    assert len(gem) > 30
    for i in gem:
        c.check(c.completion([i]))


@pytest.mark.gpu
def test_c2_memory_bound_candidates(ctx):
    c = Case(ctx, c2_vit_attention())
    mb = [x["index"] for x in c.cands if x["klass"] in ("pw", "rr")]
    for i in mb:
        c.check(c.completion([i]))


@pytest.mark.gpu
@pytest.mark.parametrize("kw", [dict(), dict(batch=2, seq=64, hidden=256, heads=4), dict(seq=200, hidden=192, heads=3),
                                dict(rewrites=True), dict(batch=2, seq=64, hidden=256, heads=4, rewrites=True)])
def test_c2_pipeline(ctx, kw):
    """profile -> BLP -> execute for several attention shapes (batched, M tails), with and
    without the R1-R3 rewrites."""
    kw = dict(kw)
    rw = kw.pop("rewrites", False)
    g = c2_vit_attention(**kw)
    if rw:
        g["rewrites"] = True
    c = Case(ctx, g)
    costs = c.kg.profile()
    obj, sel = c.kg.select(costs)
    c.check(sel)
    if not rw:  # rewritten graphs no longer have one fragment per operator
        base = c.kg.operator_aligned()
        assert obj <= sum(costs[i] for i in base)
        c.check(base)
    c.check(c.kg.singletons())


@pytest.mark.gpu
@pytest.mark.parametrize("n", [160, 96])
def test_gemm_in_tile_layernorm_non_pow2_width(ctx, n):
    """GEMM whose epilogue reduces whole rows (Linear -> LayerNorm over N): one tile spans
    the row, TMEM allocation rounded up to a power of two (N = 160 -> 256 columns)."""
    b = GraphBuilder("bf16")
    x = b.input("x", [1, 200, 64])
    w = b.input("w", [64, n], std=0.125)
    bias = b.input("bias", [n], std=0.1)
    g_ = b.input("g", [n], mean=1.0, std=0.1)
    be = b.input("be", [n], std=0.1)
    y = b.op("Add", b.op("MatMul", x, w), bias)
    b.output(b.op("LayerNorm", y, g_, be, axis=-1, eps=1e-6))
    c = Case(ctx, b.build())
    gem = [x["index"] for x in c.cands if x["klass"] == "gemm" and len(x["members"]) >= 6]
    assert gem
    for i in gem:
        nv, _, _ = c.kg.variant_info(i)
        for v in range(nv):
            c.kg.set_variant(i, v)
            c.check(c.completion([i]))


@pytest.mark.gpu
def test_c2_batch64_bench_plan(ctx):
    """The bench's scaled workload at full size (C2, batch 64, M = 8192): profile, BLP,
    execute, whole output against the oracle (persistent / wide-tile GEMM variants are
    eligible at this size)."""
    c = Case(ctx, c2_vit_attention(batch=64))
    costs = c.kg.profile()
    _, sel = c.kg.select(costs)
    c.check(sel)


@pytest.mark.gpu
def test_c1_bandwidth_variant_sampled_rows(ctx):
    """The C1 bandwidth variant at its bench size (x[2^20, 128] fp32, 512 MiB in and out):
    the BLP-selected plan on the GPU, 4096 sampled rows checked against the oracle (rows
    are independent in softmax -> LayerNorm, so the oracle evaluates only those rows)."""
    import torch
    from paper_2406_09465_b200 import KorchGraph, torch_inputs
    rows = 1 << 20
    g = c1_softmax_layernorm(rows=rows)
    kg = KorchGraph(ctx, g)
    kg.enumerate()
    costs = kg.profile()
    _, sel = kg.select(costs)
    kg.set_orchestration(sel)
    ins = make_inputs(g, seed=0)
    dev = torch_inputs(g, {k: v[1] for k, v in ins.items()})
    outs, ws = kg.torch_outputs(), kg.torch_workspace()
    kg.execute(dev, outs, ws, torch.cuda.current_stream())
    torch.cuda.synchronize()
    pick = np.sort(np.random.default_rng(5).choice(rows, 4096, replace=False))
    got = outs[0][torch.as_tensor(pick, device=outs[0].device)].cpu().numpy().astype(np.float64)
    gs = c1_softmax_layernorm(rows=len(pick))
    vals = {k: v[0] for k, v in ins.items()}
    vals["x"] = vals["x"][pick]
    pg = fission(gs)
    want = eval_primitive_graph(pg, vals)[pg["outputs"][0]]
    err = np.max(np.abs(got - want)) / np.max(np.abs(want))
    assert err <= RTOL["f32"], err


@pytest.mark.gpu
def test_cold_l2_profile_is_finite(ctx):
    """Cold-L2 re-timing (flush + event-record nodes + kernel in one graph) returns a finite
    cost for the chosen variant and leaves the variant choice unchanged."""
    from paper_2406_09465_b200 import INF, KorchGraph
    kg = KorchGraph(ctx, c2_vit_attention())
    cands = kg.enumerate(attention_pairs=True)
    gem = [c["index"] for c in cands if c["klass"] == "gemm"][:3]
    warm = kg.profile(gem)
    chosen = [kg.variant_info(i)[1] for i in gem]
    cold = kg.profile(gem, flush_l2=True, tune=False)
    assert all(0 < c < INF for c in cold), cold
    assert [kg.variant_info(i)[1] for i in gem] == chosen
    assert all(c >= 0.5 * w for c, w in zip(cold, warm))


def _ieee_values(shape, rng):
    """Specials mixed into N(0,1): +-1000 (exp overflows in fp32 AND fp64, so fused
    fp32 intermediates and the oracle's fp64 ones agree), +-inf, NaN, +-0."""
    v = rng.standard_normal(shape)
    specials = np.array([1000.0, -1000.0, np.inf, -np.inf, np.nan, 0.0, -0.0])
    mask = rng.random(shape) < 0.25
    v[mask] = specials[rng.integers(0, len(specials), mask.sum())]
    return v


def _assert_ieee_equal(got, want, rtol):
    """NaN exactly where the oracle has NaN, +-inf where it has +-inf, finite values within
    rtol of the largest finite oracle magnitude."""
    np.testing.assert_array_equal(np.isnan(got), np.isnan(want))
    inf = np.isinf(want)
    np.testing.assert_array_equal(np.isinf(got), inf)
    np.testing.assert_array_equal(got[inf], want[inf])
    fin = np.isfinite(want)
    if fin.any():
        scale = max(np.max(np.abs(want[fin])), 1e-30)
        assert np.max(np.abs(got[fin] - want[fin])) <= rtol * scale


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_ieee_special_values_propagate(ctx, dtype):
    """korch.h promises IEEE propagation: x / 0 = +-inf, 0 / 0 = NaN, exp overflow = inf,
    the literal softmax (reading A9) turns an overflowing row into inf / inf = NaN, ReLU
    and sqrt keep NaN, sqrt(-1) = NaN.  Every candidate of the graph inside a feasible
    orchestration, element by element against the oracle."""
    from korch_workloads.inputs import bf16_bits_to_f32, bf16_round_bits
    from paper_2406_09465_b200 import torch_inputs
    b = GraphBuilder(dtype)
    x = b.input("x", [16, 64])
    y = b.input("y", [16, 64])
    b.output(b.op("Div", x, y))
    b.output(b.op("Softmax", x, axis=1))
    b.output(b.op("Relu", b.op("Exp", x)))
    b.output(b.op("Sqrt", b.op("Relu", x)))
    b.output(b.op("Sqrt", x))
    g = b.build()
    c = Case(ctx, g)
    rng = np.random.default_rng(11)
    xv = _ieee_values((16, 64), rng)
    yv = rng.standard_normal((16, 64))
    yv[rng.random((16, 64)) < 0.3] = 0.0
    vals, store = {}, {}
    for n, v in (("x", xv), ("y", yv)):
        v32 = v.astype(np.float32)
        if dtype == "bf16":
            bits = bf16_round_bits(v32)
            vals[n], store[n] = bf16_bits_to_f32(bits).astype(np.float64), bits
        else:
            vals[n], store[n] = v32.astype(np.float64), v32
    c.values = vals
    c.dev_in = torch_inputs(g, store)
    gen = [x_["index"] for x_ in c.cands if x_["klass"] != "rejected"]
    sels = {tuple(c.kg.singletons()), tuple(c.kg.operator_aligned())}
    sels |= {tuple(c.completion([i])) for i in gen}
    with np.errstate(all="ignore"):
        for sel in sorted(sels):
            got = c.run(list(sel))
            want = c.oracle(list(sel))
            for k, o in enumerate(c.kg.outputs):
                _assert_ieee_equal(got[k], want[o], RTOL[dtype])


@pytest.mark.gpu
@pytest.mark.parametrize("which", ["c1", "c2_small_pairs"])
def test_selection_on_measured_costs_equals_oracle_search(ctx, which):
    """P:377-413 on MEASURED costs: after on-device profiling, the product's selection
    (native exact search) and the HiGHS MILP both reach exactly the objective of the
    oracle's independent producer-assignment search on the same integer-ns cost vector,
    and the selection is feasible (Eq. 3/4) and accepted by the library."""
    from oracle.enumeration import candidate_inputs
    from oracle.orchestration import feasible, producer_search
    from paper_2406_09465_b200 import INF, solve_blp
    if which == "c1":
        g, kw = c1_softmax_layernorm(), {}
    else:
        g, kw = c2_vit_attention(seq=32, hidden=128, heads=2), {"attention_pairs": True}
    from paper_2406_09465_b200 import KorchGraph
    kg = KorchGraph(ctx, g)
    cands = kg.enumerate(**kw)
    costs = kg.profile()
    pg = fission(g)
    G = PGraph(pg)
    ref = candidates(G, convex_sets_from_states(execution_states(G)), attention_pairs=bool(kw))
    assert [(tuple(c["members"]), c["output"]) for c in cands] == [(tuple(m), o) for m, o in ref]
    gen = [i for i, c in enumerate(costs) if c < INF]
    sub = [ref[i] for i in gen]
    cin = [candidate_inputs(G, m) for m, _ in sub]
    best, _ = producer_search(sub, [costs[i] for i in gen], pg["outputs"], cin, G.topo_index)
    obj, sel = kg.select(costs)
    assert obj == best
    cin_all = [candidate_inputs(G, m) for m, _ in ref]
    assert feasible(ref, sel, pg["outputs"], cin_all)
    hi, hsel = solve_blp(cands, costs, kg.outputs, exact=False)
    assert hi == best and feasible(ref, hsel, pg["outputs"], cin_all)
    kg.set_orchestration(sel)


@pytest.mark.gpu
def test_execute_host_matches_execute(ctx):
    """korch_execute_host (H2D of the activation, the plan, D2H of the output in one graph
    replay) gives bitwise the same output as korch_execute on device buffers; repeated
    with a second input to check the copies are replayed, not cached."""
    import torch
    c = Case(ctx, c2_vit_attention())
    costs = c.kg.profile()
    _, sel = c.kg.select(costs)
    c.kg.set_orchestration(sel)
    ws = c.kg.torch_workspace()
    names = [s["name"] for s in c.graph["inputs"]]
    xi = names.index("x")
    for trial in range(2):
        x_host = (c.dev_in[xi].float() * (1 + trial)).to(c.dev_in[xi].dtype).cpu().pin_memory()
        dev = list(c.dev_in)
        dev[xi] = torch.empty_like(c.dev_in[xi])
        hin = [x_host if i == xi else None for i in range(len(names))]
        outs = c.kg.torch_outputs()
        host_out = [torch.empty_like(o, device="cpu").pin_memory() for o in outs]
        c.kg.execute_host(hin, dev, host_out, outs, ws, torch.cuda.current_stream())
        torch.cuda.synchronize()
        ref_in = list(c.dev_in)
        ref_in[xi] = x_host.cuda()
        ref = c.kg.torch_outputs()
        c.kg.execute(ref_in, ref, ws, torch.cuda.current_stream())
        torch.cuda.synchronize()
        assert torch.equal(host_out[0], ref[0].cpu())


@pytest.mark.gpu
def test_execute_host_back_to_back_distinct_inputs(ctx):
    """korch_execute_host called back to back with a different activation per call and no
    synchronisation in between: the plan's residual GEMM fetches x before its dependency
    wait, so it must not overlap the H2D copy of x.  Every call's output must
    equal korch_execute on that call's input."""
    import torch
    c = Case(ctx, c2_vit_attention())
    costs = c.kg.profile()
    _, sel = c.kg.select(costs)
    c.kg.set_orchestration(sel)
    ws = c.kg.torch_workspace()
    names = [s["name"] for s in c.graph["inputs"]]
    xi = names.index("x")
    gen = torch.Generator().manual_seed(7)
    xs = [torch.randn(c.dev_in[xi].shape, generator=gen).to(c.dev_in[xi].dtype).pin_memory() for _ in range(6)]
    dev = list(c.dev_in)
    dev[xi] = torch.empty_like(c.dev_in[xi])
    outs = c.kg.torch_outputs()
    host_out = torch.empty((len(xs),) + tuple(outs[0].shape), dtype=outs[0].dtype).pin_memory()
    stream = torch.cuda.current_stream()
    for rep in range(2):  # the second round replays the captured graphs
        for k, xh in enumerate(xs):
            hin = [xh if i == xi else None for i in range(len(names))]
            c.kg.execute_host(hin, dev, [host_out[k]], outs, ws, stream)
        torch.cuda.synchronize()
        for k, xh in enumerate(xs):
            ref_in = list(c.dev_in)
            ref_in[xi] = xh.cuda()
            ref = c.kg.torch_outputs()
            c.kg.execute(ref_in, ref, ws, stream)
            torch.cuda.synchronize()
            assert torch.equal(host_out[k], ref[0].cpu()), (rep, k)


def _gemm_graph(m, k, n, batch=1, act="Relu"):
    b = GraphBuilder("bf16")
    x = b.input("x", [batch, m, k])
    w = b.input("w", [k, n], std=k ** -0.5)
    bias = b.input("bias", [n], std=0.1)
    r = b.input("r", [batch, m, n])
    y = b.op("MatMul", x, w)
    y = b.op("Add", y, bias)
    y = b.op(act, y)
    y = b.op("Add", y, r)
    b.output(y)
    return b.build()


@pytest.mark.gpu
@pytest.mark.parametrize("m,k,n,batch", [(128, 768, 768, 1), (128, 768, 2304, 1), (200, 512, 256, 2),
                                         (128, 256, 196, 1), (160, 64, 676, 1), (64, 128, 100, 1)])
def test_every_gemm_variant(ctx, m, k, n, batch):
    """Every launch variant of every GEMM candidate: tile width, cluster split-K (K-slice
    partials reduced through distributed shared memory), column-lane epilogue, residual
    tile staged by TMA, ragged M / N / K, batch.  Each plan executes twice and both results
    must match the oracle (state left behind by a launch would corrupt the second)."""
    c = Case(ctx, _gemm_graph(m, k, n, batch))
    for x in c.cands:
        if x["klass"] != "gemm":
            continue
        nv, _, _ = c.kg.variant_info(x["index"])
        for v in range(nv):
            c.kg.set_variant(x["index"], v)
            sel = c.completion([x["index"]])
            c.check(sel)
            c.check(sel)


@pytest.mark.gpu
@pytest.mark.parametrize("m,k,n,batch", [(130, 192, 520, 40), (256, 64, 1024, 24)])
def test_persistent_gemm_every_variant(ctx, m, k, n, batch):
    """Grids of more than two waves also get the persistent variant (one CTA per SM walking
    the tiles, double-buffered TMEM accumulators, epilogue warps overlapping the next
    tile's main loop); every variant of every GEMM candidate, ragged M / N, batch."""
    c = Case(ctx, _gemm_graph(m, k, n, batch))
    seen = 0
    for x in c.cands:
        if x["klass"] != "gemm":
            continue
        nv, _, _ = c.kg.variant_info(x["index"])
        for v in range(nv):
            c.kg.set_variant(x["index"], v)
            seen += "persistent" in c.kg.variant_info(x["index"])[2]
            sel = c.completion([x["index"]])
            c.check(sel)
            c.check(sel)
    assert seen > 0


@pytest.mark.gpu
@pytest.mark.parametrize("m,k,n,batch", [(128, 64, 64, 1), (200, 96, 104, 1), (300, 320, 384, 2), (64, 16, 48, 3),
                                         (1024, 768, 2304, 1)])
def test_gemm_shapes(ctx, m, k, n, batch):
    """Ragged M (row mask), K (TMA zero fill), N (column mask), multi-tile grids, every
    generable candidate (GEMM with 0..3 fused epilogue primitives)."""
    c = Case(ctx, _gemm_graph(m, k, n, batch))
    for x in c.cands:
        if x["klass"] != "rejected":
            c.check(c.completion([x["index"]]))


def _dconv_graph(kind, dtype="bf16"):
    """Convolutions the direct-conv template (KB7 stencil) targets, with the operand chains
    and epilogues of the paper models: Candy's reflect-padded 9x9 layers (few input
    channels / few filters), an EfficientViT-style strided stem with HardSwish, YOLOX's
    Focus space-to-depth in front of its stem conv with SiLU, and a depthwise window on an
    elementwise input."""
    b = GraphBuilder(dtype)
    if kind == "candy_out":          # reflect pad -> 9x9 conv 16 -> 3 (+bias)
        x = b.input("x", [1, 16, 24, 32])
        h = b.op("Pad", x, pads=[[0, 0], [0, 0], [4, 4], [4, 4]], mode="reflect")
        y = b.op("Conv", h, b.input("w", [3, 16, 9, 9], std=0.03), b.input("bias", [3], std=0.1),
                 stride=[1, 1], pads=[0, 0], groups=1)
    elif kind == "candy_in":         # reflect pad -> 9x9 conv 3 -> 32 (+bias) -> relu
        x = b.input("x", [1, 3, 20, 40])
        h = b.op("Pad", x, pads=[[0, 0], [0, 0], [4, 4], [4, 4]], mode="reflect")
        y = b.op("Relu", b.op("Conv", h, b.input("w", [32, 3, 9, 9], std=0.06), b.input("bias", [32], std=0.1),
                              stride=[1, 1], pads=[0, 0], groups=1))
    elif kind == "stem":             # 3x3 s2 conv 3 -> 16 (+bias) -> hardswish, zero padding
        x = b.input("x", [2, 3, 34, 64])
        y = b.op("HardSwish", b.op("Conv", x, b.input("w", [16, 3, 3, 3], std=0.2), b.input("bias", [16], std=0.1),
                                   stride=[2, 2], pads=[1, 1], groups=1))
    elif kind == "focus":            # space-to-depth (reshape/transpose) -> 3x3 conv 12 -> 16 -> SiLU
        x = b.input("x", [1, 3, 32, 48])
        f = b.op("Reshape", x, shape=[1, 3, 16, 2, 24, 2])
        f = b.op("Transpose", f, perm=[0, 5, 3, 1, 2, 4])
        f = b.op("Reshape", f, shape=[1, 12, 16, 24])
        y = b.op("SiLU", b.op("Conv", f, b.input("w", [16, 12, 3, 3], std=0.1), b.input("bias", [16], std=0.1),
                              stride=[1, 1], pads=[1, 1], groups=1))
    elif kind == "candy_wide":       # reflect pad -> 9x9 conv 32 -> 3, two 128-pixel tiles per row (ragged)
        x = b.input("x", [1, 32, 6, 200])
        h = b.op("Pad", x, pads=[[0, 0], [0, 0], [4, 4], [4, 4]], mode="reflect")
        y = b.op("Conv", h, b.input("w", [3, 32, 9, 9], std=0.02), b.input("bias", [3], std=0.1),
                 stride=[1, 1], pads=[0, 0], groups=1)
    else:                            # hardswish -> depthwise 3x3 (+bias) -> hardswish
        x = b.input("x", [1, 40, 18, 32])
        y = b.op("HardSwish", b.op("Conv", b.op("HardSwish", x), b.input("w", [40, 1, 3, 3], std=0.3),
                                   b.input("bias", [40], std=0.1), stride=[1, 1], pads=[1, 1], groups=40))
    b.output(y)
    return b.build()


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("kind", ["candy_out", "candy_in", "stem", "focus"])
def test_direct_conv_every_variant(ctx, kind, dtype):
    """KB7 direct-convolution variants: for every candidate that carries them, each
    direct-conv launch variant inside a feasible orchestration matches the oracle (staged
    operand chains with reflect / zero padding and layout views, channel chunking, tails,
    epilogues)."""
    c = Case(ctx, _dconv_graph(kind, dtype))
    ran = 0
    for x in c.cands:
        if x["klass"] == "rejected":
            continue
        names = c.kg.variant_names(x["index"])
        for v, nm in enumerate(names):
            if not nm.startswith("korch_dconv"):
                continue
            c.kg.set_variant(x["index"], v)
            c.check(c.completion([x["index"]]))
            ran += 1
    assert ran >= 2


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["candy_out", "candy_in", "focus", "candy_wide"])
def test_tc_direct_conv_every_variant(ctx, kind):
    """KB6-D tensor-core direct convolution (descriptor-offset implicit GEMM over the staged
    input window): every candidate carrying it, inside a feasible orchestration, matches
    the oracle -- reflect / zero padding, Focus views, channel padding to 16, filters
    padded to N = 16 / 32, ragged 128-pixel row tiles."""
    c = Case(ctx, _dconv_graph(kind))
    ran = 0
    for x in c.cands:
        if x["klass"] == "rejected":
            continue
        for v, nm in enumerate(c.kg.variant_names(x["index"])):
            if not nm.startswith("korch_tconv"):
                continue
            c.kg.set_variant(x["index"], v)
            c.check(c.completion([x["index"]]))
            ran += 1
    assert ran >= 1


def _gather_b_graph(m, k, n, b_layout, dtype="bf16"):
    """MatMuls whose B view has no 16-byte-aligned row pitch (gather-B tcgen05 GEMM):
    'wn' = a [K, N] weight with odd N (SegFormer's 150-class classifier), 'chw' = the
    [C, HW] activation of a pointwise conv with HW = 196 / 676 (EfficientViT / YOLOX)."""
    b = GraphBuilder(dtype)
    if b_layout == "wn":
        x = b.input("x", [1, m, k])
        y = b.op("Add", b.op("MatMul", x, b.input("w", [k, n], std=k ** -0.5)), b.input("bias", [n], std=0.1))
    else:
        x = b.input("x", [1, k, n])                       # [1, C, HW]
        t = b.op("Reshape", x, shape=[k, n])
        y = b.op("SiLU", b.op("Add", b.op("MatMul", b.input("w", [m, k], std=k ** -0.5), t),
                                b.input("bias", [m, 1], std=0.1)))
    b.output(y)
    return b.build()


@pytest.mark.gpu
@pytest.mark.parametrize("m,k,n,lay", [(300, 256, 150, "wn"), (128, 64, 19, "wn"), (64, 128, 196, "chw"),
                                       (96, 64, 676, "chw"), (256, 1024, 49, "chw")])
def test_gather_b_gemm_every_variant(ctx, m, k, n, lay):
    """Gather-B GEMM (B gathered into the MN-major SW128 layout by four producer warps;
    8 consecutive columns per 16-byte unaligned read when B is N-contiguous): every
    launch variant of every GEMM candidate, ragged M / N tails."""
    c = Case(ctx, _gather_b_graph(m, k, n, lay))
    gg = [x for x in c.cands if x["klass"] == "gemm"]
    assert gg
    ran = 0
    for x in gg:
        nv, _, _ = c.kg.variant_info(x["index"])
        for v in range(nv):
            c.kg.set_variant(x["index"], v)
            c.check(c.completion([x["index"]]))
            ran += 1
    assert ran >= 2


def _skinny_mm_graph(cin, cout, hw, dtype="bf16"):
    """EfficientViT-style pointwise conv as MatMul over [C, HW] with few input channels
    (+bias, HardSwish, back to NCHW)."""
    b = GraphBuilder(dtype)
    x = b.input("x", [1, cin, hw, hw])
    t = b.op("Reshape", b.op("HardSwish", x), shape=[cin, hw * hw])
    t = b.op("Add", b.op("MatMul", b.input("w", [cout, cin], std=cin ** -0.5), t), b.input("bias", [cout, 1], std=0.1))
    b.output(b.op("HardSwish", b.op("Reshape", t, shape=[1, cout, hw, hw])))
    return b.build()


@pytest.mark.gpu
@pytest.mark.parametrize("cin,cout,hw", [(16, 64, 64), (32, 24, 40), (8, 200, 48)])
@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_skinny_k_matmul_every_variant(ctx, cin, cout, hw, dtype):
    """Skinny-K MatMul SIMT variants (K <= 64): every variant of every candidate carrying
    them, including an elementwise chain on the staged B operand and ragged row groups."""
    c = Case(ctx, _skinny_mm_graph(cin, cout, hw, dtype))
    ran = 0
    for x in c.cands:
        if x["klass"] == "rejected":
            continue
        for v, nm in enumerate(c.kg.variant_names(x["index"])):
            if nm.startswith("korch_skmm"):
                c.kg.set_variant(x["index"], v)
                c.check(c.completion([x["index"]]))
                ran += 1
    assert ran >= 2


def _ktv_graph(heads2=4, d=16, n=2048, dtype="bf16"):
    """EfficientViT's LiteMLA K^T V: relu(K)^T [d, n] x pad_ones(V) [n, d+1] per
    head over n tokens, K and V sliced out of a token-minor [2h, 3d, n] tensor."""
    b = GraphBuilder(dtype)
    x = b.input("x", [1, heads2, 3 * d, n])
    ms = b.op("Transpose", x, perm=[0, 1, 3, 2])                        # [1, 2h, n, 3d]
    k = b.op("Relu", b.op("Slice", ms, axis=3, start=d, end=2 * d))
    v = b.op("Slice", ms, axis=3, start=2 * d, end=3 * d)
    v = b.op("Pad", v, pads=[[0, 0], [0, 0], [0, 0], [0, 1]], mode="constant", value=1.0)
    kv = b.op("MatMul", b.op("Transpose", k, perm=[0, 1, 3, 2]), v)     # [1, 2h, d, d+1]
    b.output(b.op("MulC", kv, c=0.5))
    return b.build()


@pytest.mark.gpu
@pytest.mark.parametrize("n", [2048, 5000])
@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_split_k_contraction_every_variant(ctx, n, dtype):
    """KB8 cluster split-K contraction: every variant of every candidate carrying it
    (operand chains staged per token tile, ragged K slices, DSMEM combine)."""
    c = Case(ctx, _ktv_graph(n=n, dtype=dtype))
    ran = 0
    for x in c.cands:
        if x["klass"] == "rejected":
            continue
        for v, nm in enumerate(c.kg.variant_names(x["index"])):
            if nm.startswith("korch_kb8"):
                c.kg.set_variant(x["index"], v)
                c.check(c.completion([x["index"]]))
                ran += 1
    assert ran >= 1
