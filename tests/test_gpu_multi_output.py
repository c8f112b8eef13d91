"""GPU parity for multi-output candidate kernels (reading A32): every
(P', o, E) kernel the library generates runs inside a feasible orchestration and matches
the oracle's orchestration-aware evaluation element by element (A21
tolerances); the profile -> select -> execute pipeline with secondary outputs reaches
the oracle's exact optimum on the measured costs."""
import numpy as np
import pytest

from korch_workloads import c1_softmax_layernorm, make_inputs
from korch_workloads.graphs import GraphBuilder
from oracle.enumeration import PGraph, candidate_inputs, candidates, convex_sets_from_states, execution_states
from oracle.fission import fission
from oracle.multi_output import (eval_orchestration_mo, feasible_mo, multi_output_candidates, outputs_of,
                                 producer_search_mo)

torch = pytest.importorskip("torch")

RTOL = {"f32": 1e-4, "bf16": 2e-2}


@pytest.fixture(scope="module")
def ctx():
    from paper_2406_09465_b200 import Context
    return Context(0)


def residual_ln_graph(dtype="bf16", n=64, c=64):
    """x -> t = x + Linear(x) -> y = LN(t) -> u = t + Linear(y): t feeds both the
    LayerNorm and the second residual (SegFormer / ViT block shape), so a GEMM-epilogue
    kernel can emit {LN(t), t}."""
    b = GraphBuilder(dtype)
    x = b.input("x", [1, n, c])
    w1 = b.input("w1", [c, c], std=c ** -0.5)
    b1 = b.input("b1", [c], std=0.02)
    w2 = b.input("w2", [c, c], std=c ** -0.5)
    b2 = b.input("b2", [c], std=0.02)
    g = b.input("g", [c], mean=1.0, std=0.1)
    be = b.input("be", [c], std=0.1)
    t = b.op("Add", x, b.op("Add", b.op("MatMul", x, w1), b1))
    y = b.op("LayerNorm", t, g, be, axis=-1, eps=1e-6)
    u = b.op("Add", t, b.op("Add", b.op("MatMul", y, w2), b2))
    b.output(u)
    return b.build()


class MOCase:
    def __init__(self, ctx, graph, max_outputs=2, seed=0):
        from paper_2406_09465_b200 import KorchGraph, torch_inputs
        self.graph = graph
        self.kg = KorchGraph(ctx, graph)
        self.cands = self.kg.enumerate(max_outputs=max_outputs)
        self.pg = fission(graph)
        self.G = PGraph(self.pg)
        single = candidates(self.G, convex_sets_from_states(execution_states(self.G)))
        self.ref = multi_output_candidates(self.G, single, max_outputs)
        assert [(tuple(c["members"]), c["output"], tuple(c["extra_outputs"])) for c in self.cands] == self.ref
        self.cin = [candidate_inputs(self.G, c[0]) for c in self.ref]
        ins = make_inputs(graph, seed=seed)
        self.values = {k: v[0] for k, v in ins.items()}
        self.dev_in = torch_inputs(graph, {k: v[1] for k, v in ins.items()})
        self.storage = graph["dtype"]

    def completion(self, must, use_extras):
        """`must` plus single-output producers (smallest first) for every tensor still
        needed; with use_extras the secondary outputs of `must` count as materialised."""
        prod = {}
        for c in self.cands:
            if c["klass"] != "rejected" and not c["extra_outputs"]:
                prod.setdefault(c["output"], []).append(c["index"])
        for o in prod:
            prod[o].sort(key=lambda i: (len(self.cands[i]["members"]), i))
        have = set(outputs_of(self.ref[must])) if use_extras else {self.ref[must][1]}
        sel = [must]
        need = list(self.cin[must]) + list(self.kg.outputs)
        while need:
            t = need.pop()
            if t in have:
                continue
            i = prod[t][0]
            sel.append(i)
            have.add(t)
            need.extend(self.cin[i])
        return sorted(set(sel))

    def check(self, sel):
        self.kg.set_orchestration(sel)
        outs = self.kg.torch_outputs()
        ws = self.kg.torch_workspace()
        self.kg.execute(self.dev_in, outs, ws, torch.cuda.current_stream())
        torch.cuda.synchronize()
        want = eval_orchestration_mo(self.pg, self.ref, sel, self.values, self.G.topo_index, self.storage)
        for k, o in enumerate(self.kg.outputs):
            got = outs[k].float().cpu().numpy().astype(np.float64)
            err = np.max(np.abs(got - want[o]))
            scale = np.max(np.abs(want[o]))
            assert err <= RTOL[self.storage] * scale, f"sel={sel}: err {err:.3e} vs {scale:.3e}"


def _every_multi_output_candidate(c):
    mo = [i for i, x in enumerate(c.ref) if x[2]]
    assert mo
    ran = 0
    for i in mo:
        if c.cands[i]["klass"] == "rejected":
            continue
        for use in (True, False):
            sel = c.completion(i, use)
            if not feasible_mo(c.ref, sel, sorted(c.G.outputs), c.cin, c.G.topo_index):
                continue
            c.check(sel)
            ran += 1
    return ran


@pytest.mark.gpu
def test_c1_every_multi_output_candidate(ctx):
    c = MOCase(ctx, c1_softmax_layernorm())
    assert _every_multi_output_candidate(c) >= 19


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_gemm_epilogue_secondary_outputs(ctx, dtype):
    """GEMM epilogues (tcgen05 template) that also store an intermediate, e.g. the
    residual sum t next to LN(t)."""
    c = MOCase(ctx, residual_ln_graph(dtype))
    gem = [i for i, x in enumerate(c.ref) if x[2] and c.cands[i]["klass"] == "gemm"]
    if dtype == "bf16":   # fp32 MatMuls run on the SIMT row template
        assert gem, "no generable multi-output GEMM candidate"
    assert _every_multi_output_candidate(c) >= len(gem)


@pytest.mark.gpu
@pytest.mark.parametrize("which", ["c1", "residual_ln"])
def test_multi_output_pipeline_on_measured_costs(ctx, which):
    """profile -> select (MILP with Eq. 4') -> execute: the selection's objective equals the
    oracle's exact multi-output search on the same measured integer-ns costs, never exceeds
    the single-output optimum, and its output matches the oracle."""
    from paper_2406_09465_b200 import INF
    g = c1_softmax_layernorm() if which == "c1" else residual_ln_graph()
    c = MOCase(ctx, g)
    costs = c.kg.profile()
    gen = [i for i, x in enumerate(costs) if x < INF]
    sub = [c.ref[i] for i in gen]
    best, _ = producer_search_mo(sub, [costs[i] for i in gen], sorted(c.G.outputs), [c.cin[i] for i in gen],
                                 c.G.topo_index)
    obj, sel = c.kg.select(costs)
    assert obj == best
    assert feasible_mo(c.ref, sel, sorted(c.G.outputs), c.cin, c.G.topo_index)
    single = [i for i in gen if not c.ref[i][2]]
    s_best, _ = producer_search_mo([c.ref[i] for i in single], [costs[i] for i in single], sorted(c.G.outputs),
                                   [c.cin[i] for i in single], c.G.topo_index)
    assert obj <= s_best
    c.check(sel)
