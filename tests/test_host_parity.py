"""Host-side parity of the library against the oracle (bit-exact, no GPU):
fission (primitive graph), Alg. 1 enumeration (candidate lists), BLP selection."""
import numpy as np
import pytest

from korch_workloads import c1_softmax_layernorm, c2_vit_attention
from korch_workloads.graphs import GraphBuilder
from oracle.enumeration import PGraph, candidate_inputs, candidates, convex_sets_from_states, execution_states
from oracle.fission import fission
from oracle.orchestration import feasible, producer_search

from paper_2406_09465_b200 import Context, KorchGraph, solve_blp


@pytest.fixture(scope="module")
def ctx():
    return Context(-1)


def _norm_ref(r):
    return ("input", r["input"]) if "input" in r else ("node", r["node"])


def _norm_attrs(kind, a):
    a = dict(a)
    if kind == "pad":
        a["pads"] = [list(p) for p in a["pads"]]
    if "c" in a:
        a["c"] = float(np.float64(a["c"]))
    return a


GRAPHS = {
    "c1": lambda: c1_softmax_layernorm(),
    "c1_noaffine": lambda: c1_softmax_layernorm(affine=False, eps=0.0),
    "c2": lambda: c2_vit_attention(),
    "c2_b2": lambda: c2_vit_attention(batch=2, seq=32, hidden=128, heads=4),
}


def _misc_graph():
    b = GraphBuilder("f32")
    x = b.input("x", [2, 16, 6, 6])
    w = b.input("w", [16, 16, 3, 3], std=0.1)
    g = b.input("g", [16], mean=1.0, std=0.1)
    be = b.input("be", [16], std=0.1)
    y = b.op("Conv", x, w, stride=[1, 1], pads=[1, 1], groups=1)
    y = b.op("InstanceNorm", y, g, be, eps=1e-5)
    y = b.op("Relu", y)
    y = b.op("Pad", y, pads=[[0, 0], [0, 0], [1, 1], [1, 1]], mode="reflect")
    y = b.op("GELU", y)
    z = b.op("Upsample2x", y)
    b.output(z)
    return b.build()


GRAPHS["misc"] = _misc_graph


def _rw(g):
    g["rewrites"] = True
    return g


def _cnn():
    from test_gpu_parity import _cnn_graph
    return _cnn_graph()


GRAPHS["cnn"] = _cnn
GRAPHS["c2_r1r3"] = lambda: _rw(c2_vit_attention())
GRAPHS["c2_b2_r1r3"] = lambda: _rw(c2_vit_attention(batch=2, seq=32, hidden=128, heads=4))


@pytest.mark.parametrize("name", sorted(GRAPHS))
def test_fission_matches_oracle(ctx, name):
    g = GRAPHS[name]()
    ours = KorchGraph(ctx, g).prim
    ref = fission(g)
    assert len(ours["nodes"]) == len(ref["nodes"])
    for a, b in zip(ours["nodes"], ref["nodes"]):
        assert a["id"] == b["id"]
        assert a["kind"] == b["kind"], (a, b)
        assert tuple(a["shape"]) == tuple(b["shape"])
        assert [_norm_ref(r) for r in a["inputs"]] == [tuple(r) for r in b["inputs"]]
        ra = _norm_attrs(a["kind"], a["attrs"])
        rb = _norm_attrs(b["kind"], b["attrs"])
        for k, v in rb.items():
            if k == "port_axes":
                assert {kk: list(vv) for kk, vv in ra[k].items()} == {kk: list(vv) for kk, vv in v.items()}
            else:
                assert ra[k] == v, (k, ra, rb)
    assert ours["outputs"] == ref["outputs"]


def _oracle_cands(g, max_prims=16):
    pg = fission(g)
    G = PGraph(pg)
    return G, candidates(G, convex_sets_from_states(execution_states(G)), max_prims=max_prims)


@pytest.mark.parametrize("name", sorted(GRAPHS))
def test_enumeration_matches_oracle(ctx, name):
    g = GRAPHS[name]()
    kg = KorchGraph(ctx, g)
    ours = kg.enumerate()
    G, ref = _oracle_cands(g)
    st = execution_states(G)
    assert kg.n_states == len(st)
    assert [(tuple(c["members"]), c["output"]) for c in ours] == [(tuple(m), o) for m, o in ref]
    for c in ours:
        assert c["inputs"] == candidate_inputs(G, c["members"])


def _random_op_graph(rng, n_ops):
    """Random DAG of elementwise / softmax / layout operators on [8, 32] tensors."""
    b = GraphBuilder("f32")
    refs = [b.input("x", [8, 32])]
    for _ in range(n_ops):
        k = int(rng.integers(0, 5))
        a = refs[int(rng.integers(0, len(refs)))]
        if k == 0:
            r = b.op("Exp", a)
        elif k == 1:
            r = b.op("Add", a, refs[int(rng.integers(0, len(refs)))])
        elif k == 2:
            r = b.op("Softmax", a, axis=1)
        elif k == 3:
            r = b.op("MulC", a, c=0.5)
        else:
            r = b.op("Relu", a)
        refs.append(r)
    used = set()
    for n in b.g["nodes"]:
        for r in n["inputs"]:
            if "node" in r:
                used.add(r["node"])
    for n in b.g["nodes"]:
        if n["id"] not in used:
            b.output({"node": n["id"]})
    return b.build()


def test_enumeration_random_graphs(ctx):
    rng = np.random.default_rng(3)
    for _ in range(25):
        g = _random_op_graph(rng, int(rng.integers(2, 7)))
        kg = KorchGraph(ctx, g)
        ours = kg.enumerate(max_prims=8)
        _, ref = _oracle_cands(g, max_prims=8)
        assert [(tuple(c["members"]), c["output"]) for c in ours] == [(tuple(m), o) for m, o in ref]


def test_blp_matches_exact_search_c1(ctx):
    """The product's HiGHS BLP reaches exactly the oracle's producer-assignment optimum."""
    g = c1_softmax_layernorm()
    kg = KorchGraph(ctx, g)
    cands = kg.enumerate()
    G, ref = _oracle_cands(g)
    cin = [candidate_inputs(G, m) for m, _ in ref]
    rng = np.random.default_rng(9)
    for _ in range(4):
        costs = [int(1500 + 100 * len(c["members"]) + rng.integers(0, 800)) for c in cands]
        obj, sel = solve_blp(cands, costs, kg.outputs)
        best, osel = producer_search(ref, costs, G.pg["outputs"], cin, G.topo_index)
        assert obj == best
        assert feasible(ref, sel, G.pg["outputs"], cin)
        kg.set_orchestration(sel)          # the library accepts it (Eq. 3/4)


def test_blp_pruning_exact_on_random_graphs(ctx):
    """The BLP's exact reductions (dominance, dead candidates) keep the optimum: random
    operator DAGs, costs drawn from 3 values (many ties, the hard case for dominance),
    objective == the oracle's producer-assignment search, selection feasible."""
    rng = np.random.default_rng(11)
    for _ in range(20):
        g = _random_op_graph(rng, int(rng.integers(2, 7)))
        kg = KorchGraph(ctx, g)
        cands = kg.enumerate(max_prims=8)
        G, ref = _oracle_cands(g, max_prims=8)
        cin = [candidate_inputs(G, m) for m, _ in ref]
        costs = [int(rng.integers(1, 4)) * 1000 for _ in cands]
        obj, sel = solve_blp(cands, costs, kg.outputs)
        best, _ = producer_search(ref, costs, G.pg["outputs"], cin, G.topo_index)
        assert obj == best
        assert feasible(ref, sel, G.pg["outputs"], cin)


def test_exact_solver_equals_highs_and_oracle(ctx):
    """The native A* search (libkorch_select.so) and the HiGHS MILP reach the same
    objective as the oracle's producer-assignment search on random DAGs and C1, with
    costs that tie often (3 values) and costs that rarely tie; the A* selection also has
    the fewest kernels among equal-cost optima (reading A8: the oracle's tie-break)."""
    from paper_2406_09465_b200.select import prune_dominated, solve_exact
    rng = np.random.default_rng(17)
    graphs = [_random_op_graph(rng, int(rng.integers(2, 7))) for _ in range(15)] + [c1_softmax_layernorm()]
    for gi, g in enumerate(graphs):
        kg = KorchGraph(ctx, g)
        mp = 16 if gi == len(graphs) - 1 else 8   # C1 at the default max_prims
        cands = kg.enumerate(max_prims=mp)
        G, ref = _oracle_cands(g, max_prims=mp)
        cin = [candidate_inputs(G, m) for m, _ in ref]
        for tie in (True, False):
            costs = [int(rng.integers(1, 4)) * 1000 if tie else int(rng.integers(1000, 9000)) for _ in cands]
            best, osel = producer_search(ref, costs, G.pg["outputs"], cin, G.topo_index)
            ex = solve_exact(cands, costs, kg.outputs)
            assert ex is not None
            assert ex[0] == best and feasible(ref, ex[1], G.pg["outputs"], cin)
            assert len(ex[1]) == len(osel)
            live = prune_dominated(cands, costs, range(len(cands)))
            ex2 = solve_exact(cands, costs, kg.outputs, live)
            assert ex2[0] == best and len(ex2[1]) == len(osel)
            hi, hsel = solve_blp(cands, costs, kg.outputs, exact=False)
            assert hi == best and feasible(ref, hsel, G.pg["outputs"], cin)


def test_exact_solver_whole_model_equals_highs(ctx):
    """Candy at its paper size (224^2, 2886 partitioned candidates): the exact A* search
    and HiGHS (proven optimal within its limit) agree on every part with analytic
    synthetic costs (bytes / 6.5 GB/ms + flops / 1.5 TFLOP/ms + 2 us + noise)."""
    import paper_2406_09465_b200.select as S
    from korch_workloads.models import candy
    kg = KorchGraph(ctx, candy())
    frag = {}
    for n in kg.prim["nodes"]:
        frag[n["op"]] = frag.get(n["op"], 0) + 1
    cands = kg.enumerate(partition_max=64, max_prims=max(12, max(frag.values())))
    rng = np.random.default_rng(0)
    costs = [S.INF if c["klass"] == "rejected" else
             int(2000 + c["bytes"] / 6.5 + c["flops"] / 1.5e6 + rng.integers(0, 800)) for c in cands]
    obj, sel = S.solve_partitioned(cands, costs, kg.outputs)
    assert S.LAST_SOLVER == "exact" and S.LAST_OPTIMAL
    kg.set_orchestration(sel)
    orig = S.solve_blp
    try:
        S.solve_blp = lambda c, co, o, tl=600.0: orig(c, co, o, tl, exact=False)
        obj2, sel2 = S.solve_partitioned(cands, costs, kg.outputs, time_limit=300)
        assert S.LAST_SOLVER == "highs" and S.LAST_OPTIMAL
    finally:
        S.solve_blp = orig
    assert obj == obj2 and len(sel) <= len(sel2)


@pytest.mark.parametrize("name,pm", [("c2", 8), ("c2", 12), ("c2_r1r3", 10), ("misc", 6), ("c1", 5)])
def test_partitioned_enumeration_matches_oracle(ctx, name, pm):
    from oracle.enumeration import candidates_partitioned, partition
    g = GRAPHS[name]()
    kg = KorchGraph(ctx, g)
    ours = kg.enumerate(partition_max=pm)
    G = PGraph(fission(g))
    parts = partition(G, pm)
    ref, n_states = candidates_partitioned(G, parts)
    assert [(tuple(c["members"]), c["output"]) for c in ours] == [(tuple(m), o) for m, o in ref]
    assert kg.n_states == n_states
    part_of = {v: i for i, p in enumerate(parts) for v in p}
    assert all(part_of[c["output"]] == c["part"] for c in ours)


def test_partitioned_blp_equals_global_optimum(ctx):
    """Per-part decomposition of Eq. 2-4 reaches the optimum of the whole (partitioned)
    candidate set (oracle producer-assignment search over all parts at once)."""
    g = c1_softmax_layernorm()
    kg = KorchGraph(ctx, g)
    ours = kg.enumerate(partition_max=5)
    assert len({c["part"] for c in ours}) > 1
    G = PGraph(fission(g))
    ref = [(tuple(c["members"]), c["output"]) for c in ours]
    cin = [candidate_inputs(G, m) for m, _ in ref]
    rng = np.random.default_rng(21)
    for _ in range(3):
        costs = [int(1500 + 90 * len(c["members"]) + rng.integers(0, 700)) for c in ours]
        obj, sel = kg.select(costs)
        best, _ = producer_search(ref, costs, G.pg["outputs"], cin, G.topo_index)
        assert obj == best
        assert feasible(ref, sel, G.pg["outputs"], cin)


@pytest.mark.parametrize("name", ["efficientvit", "candy", "segformer", "yolox"])
def test_models_fission_and_partitioned_enumeration(ctx, name):
    """Whole paper models (reduced sizes): primitive graph and partitioned candidate list
    bit-identical to the oracle's."""
    from korch_workloads.models import candy, efficientvit, segformer, yolox_nano
    from oracle.enumeration import candidates_partitioned, partition
    g = {"efficientvit": lambda: efficientvit(size=32, depths=(1, 1, 1, 1, 1)),
         "candy": lambda: candy(size=16, blocks=1),
         "segformer": lambda: segformer(size=32, depths=(1, 1, 1, 1)),
         "yolox": lambda: yolox_nano(size=64)}[name]()
    kg = KorchGraph(ctx, g)
    ref_pg = fission(g)
    assert [(n["kind"], tuple(n["shape"])) for n in kg.prim["nodes"]] == \
        [(n["kind"], tuple(n["shape"])) for n in ref_pg["nodes"]]
    ours = kg.enumerate(partition_max=32)
    G = PGraph(ref_pg)
    ref, n_states = candidates_partitioned(G, partition(G, 32))
    assert [(tuple(c["members"]), c["output"]) for c in ours] == [(tuple(m), o) for m, o in ref]
    assert kg.n_states == n_states
    assert len(kg.operator_aligned()) == len(g["nodes"])


def test_blp_with_rejections_and_baselines(ctx):
    g = c2_vit_attention()
    kg = KorchGraph(ctx, g)
    cands = kg.enumerate()
    base = kg.operator_aligned()
    assert len(base) == len(g["nodes"])
    singles = kg.singletons()
    assert len(singles) == kg.n_prims


# ------------------------------------------------------------------ N1 multi-output
@pytest.mark.parametrize("name", ["c1", "c1_noaffine", "c2_b2", "misc", "cnn"])
@pytest.mark.parametrize("max_outputs", [2, 3])
def test_multi_output_enumeration_matches_oracle(ctx, name, max_outputs):
    """N1 (reading A32): the library's (P', o, E) list equals the oracle's, in order."""
    from oracle.multi_output import multi_output_candidates
    g = GRAPHS[name]()
    kg = KorchGraph(ctx, g)
    ours = kg.enumerate(max_outputs=max_outputs)
    G, ref = _oracle_cands(g)
    want = multi_output_candidates(G, ref, max_outputs)
    assert len(want) > len(ref)
    assert [(tuple(c["members"]), c["output"], tuple(c["extra_outputs"])) for c in ours] == want
    for c in ours:
        assert c["inputs"] == candidate_inputs(G, c["members"])


def test_multi_output_random_graphs(ctx):
    from oracle.multi_output import multi_output_candidates
    rng = np.random.default_rng(9)
    for _ in range(20):
        g = _random_op_graph(rng, int(rng.integers(2, 7)))
        kg = KorchGraph(ctx, g)
        ours = kg.enumerate(max_prims=8, max_outputs=2)
        G, ref = _oracle_cands(g, max_prims=8)
        assert [(tuple(c["members"]), c["output"], tuple(c["extra_outputs"])) for c in ours] == \
            multi_output_candidates(G, ref, 2)


def test_multi_output_blp_equals_oracle_search_c1(ctx):
    """The product's selection (MILP with Eq. 4') reaches exactly the oracle's
    producer-assignment optimum on C1 with multi-output candidates and seeded costs."""
    from oracle.multi_output import feasible_mo, multi_output_candidates, producer_search_mo
    g = c1_softmax_layernorm()
    kg = KorchGraph(ctx, g)
    cands = kg.enumerate(max_outputs=2)
    G, ref = _oracle_cands(g)
    mo = multi_output_candidates(G, ref, 2)
    cin = [candidate_inputs(G, c[0]) for c in mo]
    rng = np.random.default_rng(17)
    for trial in range(4):
        costs = [int(rng.integers(500, 5000)) for _ in mo]
        costs = [c // 2 if mo[i][2] else c for i, c in enumerate(costs)]
        want, wsel = producer_search_mo(mo, costs, G.outputs, cin, G.topo_index)
        obj, sel = solve_blp(cands, costs, kg.outputs)
        assert obj == want
        assert feasible_mo(mo, sel, sorted(G.outputs), cin, G.topo_index)
        kg.set_orchestration(sel)          # the library accepts it (Eq. 3 / Eq. 4')


@pytest.mark.parametrize("name", ["c1", "c2", "misc", "cnn"])
def test_greedy_fusion_ablation_is_feasible_and_never_beats_blp(ctx, name):
    """Fission + greedy fusion (P:505-518 ablation; P:611-616 'fuse everything'): a
    feasible partition (oracle Eq. 3/4 check) whose cost is never below the BLP optimum."""
    from paper_2406_09465_b200.select import greedy_fusion
    g = GRAPHS[name]()
    kg = KorchGraph(ctx, g)
    cands = kg.enumerate()
    G, ref = _oracle_cands(g)
    cin = [candidate_inputs(G, m) for m, _ in ref]
    rng = np.random.default_rng(2)
    for _ in range(3):
        costs = [int(rng.integers(100, 5000)) if c["klass"] != "rejected" else (1 << 63) - 1 for c in cands]
        sel = greedy_fusion(cands, costs, kg.prim, kg.outputs)
        assert feasible(ref, sel, sorted(G.outputs), cin)
        members = sorted(m for i in sel for m in cands[i]["members"])
        assert members == list(range(kg.n_prims))          # a partition: no redundancy
        obj, _ = solve_blp(cands, costs, kg.outputs)
        assert obj <= sum(costs[i] for i in sel)


def test_greedy_fusion_fuses_c1_into_one_kernel(ctx):
    """C1's 15 primitives form one generable candidate; every producer's consumers end up
    in one kernel, so greedy fusion selects exactly that whole-block kernel."""
    from paper_2406_09465_b200.select import greedy_fusion
    kg = KorchGraph(ctx, c1_softmax_layernorm())
    cands = kg.enumerate()
    costs = [1000 if c["klass"] != "rejected" else (1 << 63) - 1 for c in cands]
    sel = greedy_fusion(cands, costs, kg.prim, kg.outputs)
    assert len(sel) == 1 and len(cands[sel[0]]["members"]) == kg.n_prims
