"""Whole paper models through the C ABI at reduced sizes: Candy (IN/ReLU/pad
CNN) and SegFormer (LN/attention transformer), partitioned (reading A17), executed with
the operator-aligned orchestration and with a BLP-selected orchestration over profiled
candidates; outputs against the oracle's orchestration-aware fp64 evaluation of the
same orchestration (bf16 storage, rtol 2e-2 of the output's max norm)."""
import numpy as np
import pytest

from korch_workloads import make_inputs
from korch_workloads.models import candy, segformer
from oracle.enumeration import PGraph
from oracle.evaluate import eval_orchestration
from oracle.fission import fission

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def ctx():
    from paper_2406_09465_b200 import Context
    return Context(0)


def _run_and_check(ctx, graph, max_members=2, rtol=2e-2):
    from paper_2406_09465_b200 import KorchGraph, torch_inputs
    kg = KorchGraph(ctx, graph)
    cands = kg.enumerate(partition_max=64)
    pg = fission(graph)
    G = PGraph(pg)
    ref_cands = [(tuple(c["members"]), c["output"]) for c in cands]
    ins = make_inputs(graph, seed=0)
    vals = {k: v[0] for k, v in ins.items()}
    dev = torch_inputs(graph, {k: v[1] for k, v in ins.items()})
    small = [c["index"] for c in cands if len(c["members"]) <= max_members and c["klass"] != "rejected"]
    base = kg.operator_aligned()
    prof = sorted(set(small) | set(base))
    costs = [(1 << 63) - 1] * len(cands)
    for i, ns in zip(prof, kg.profile(prof)):
        costs[i] = ns
    obj, sel = kg.select(costs)
    assert obj <= sum(costs[i] for i in base)
    for orch in (base, sel):
        kg.set_orchestration(orch)
        outs, ws = kg.torch_outputs(), kg.torch_workspace()
        kg.execute(dev, outs, ws, torch.cuda.current_stream())
        torch.cuda.synchronize()
        want = eval_orchestration(pg, ref_cands, orch, vals, G.topo_index, graph["dtype"])
        for k, o in enumerate(kg.outputs):
            got = outs[k].float().cpu().numpy().astype(np.float64)
            r = want[o]
            assert np.isfinite(got).all()
            err = np.max(np.abs(got - r)) / np.max(np.abs(r))
            assert err <= rtol, f"rel err {err:.3e}"
    return len(cands), len(sel), len(base)


@pytest.mark.gpu
@pytest.mark.timeout(1200)
def test_candy_small(ctx):
    n, k_sel, k_base = _run_and_check(ctx, candy(size=32, blocks=1))
    assert n > 500


@pytest.mark.gpu
@pytest.mark.timeout(1200)
def test_efficientvit_small(ctx):
    from korch_workloads.models import efficientvit
    n, k_sel, k_base = _run_and_check(ctx, efficientvit(size=64, depths=(1, 1, 1, 1, 1)))
    assert n > 500


@pytest.mark.gpu
@pytest.mark.timeout(1200)
def test_yolox_small(ctx):
    from korch_workloads.models import yolox_nano
    n, k_sel, k_base = _run_and_check(ctx, yolox_nano(size=64))
    assert n > 1000


@pytest.mark.gpu
@pytest.mark.timeout(1200)
def test_segformer_small(ctx):
    n, k_sel, k_base = _run_and_check(ctx, segformer(size=64, depths=(1, 1, 1, 1)))
    assert n > 1000


@pytest.mark.gpu
@pytest.mark.timeout(1200)
def test_concurrent_branches_bitwise_equal_sequential(ctx):
    """N4: replaying the plan with independent steps on up to 4 capture streams (event
    joins for RAW / WAR / WAW hazards on reused workspace ranges) gives bitwise the outputs
    of the sequential chain, over repeated back-to-back replays (a missing hazard edge
    would let a later step overwrite a buffer still being read)."""
    import os
    from korch_workloads.models import yolox_nano
    from paper_2406_09465_b200 import KorchGraph, torch_inputs
    graph = yolox_nano(size=64)
    kg = KorchGraph(ctx, graph)
    cands = kg.enumerate(partition_max=64)
    base = kg.operator_aligned()                  # many kernels, parallel head branches
    ins = make_inputs(graph, seed=0)
    dev = torch_inputs(graph, {k: v[1] for k, v in ins.items()})
    res = {}
    old = os.environ.get("KORCH_STREAMS")
    try:
        for ns in ("1", "4"):
            os.environ["KORCH_STREAMS"] = ns
            kg.set_orchestration(base)
            outs, ws = kg.torch_outputs(), kg.torch_workspace()
            for _ in range(20):
                kg.execute(dev, outs, ws, torch.cuda.current_stream())
            torch.cuda.synchronize()
            res[ns] = [o.clone() for o in outs]
    finally:
        if old is None:
            os.environ.pop("KORCH_STREAMS", None)
        else:
            os.environ["KORCH_STREAMS"] = old
    assert all(torch.equal(a, b) for a, b in zip(res["1"], res["4"]))


@pytest.mark.gpu
@pytest.mark.timeout(1800)
@pytest.mark.parametrize("name", ["candy", "efficientvit", "yolox", "segformer"])
def test_paper_size_model_plan_matches_oracle(ctx, name):
    """Each paper model at its paper input size executing the orchestration
    the bench runs (exact Eq. 2-4 optimum on the costs of the committed tuning database,
    profiles/tuning_db; candidates missing from it are profiled live), against the
    oracle's orchestration-aware fp64 evaluation of the same orchestration (reading A36:
    relative L2 error <= 2e-2 and max-norm error <= 5e-2 for whole bf16 models)."""
    import os
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from bench import TUNING_DB, model_enum_opts, model_graph
    from paper_2406_09465_b200 import KorchGraph, torch_inputs, tunedb
    graph = model_graph(name)
    kg = KorchGraph(ctx, graph)
    opts = model_enum_opts(kg)
    cands = kg.enumerate(**opts)
    db = tunedb.load(os.path.join(TUNING_DB, f"{name}_b1.json"))
    ok, why = tunedb.usable(db, graph, opts)
    if ok:
        costs, missing = tunedb.apply(kg, db)
        for i, c in zip(missing, kg.profile(missing) if missing else []):
            costs[i] = c
    else:
        costs = kg.profile()
    obj, sel = kg.select(costs)
    kg.set_orchestration(sel)
    ins = make_inputs(graph, seed=0)
    dev = torch_inputs(graph, {k: v[1] for k, v in ins.items()})
    outs, ws = kg.torch_outputs(), kg.torch_workspace()
    kg.execute(dev, outs, ws, torch.cuda.current_stream())
    torch.cuda.synchronize()
    pg = fission(graph)
    G = PGraph(pg)
    want = eval_orchestration(pg, [(tuple(c["members"]), c["output"]) for c in cands], sel,
                              {k: v[0] for k, v in ins.items()}, G.topo_index, graph["dtype"])
    for k, o in enumerate(kg.outputs):
        got = outs[k].float().cpu().numpy().astype(np.float64)
        r = want[o]
        assert np.isfinite(got).all()
        l2 = np.linalg.norm(got - r) / np.linalg.norm(r)
        mx = np.max(np.abs(got - r)) / np.max(np.abs(r))
        assert l2 <= 2e-2 and mx <= 5e-2, f"{name}: rel L2 {l2:.3e}, max-norm {mx:.3e}"


@pytest.mark.gpu
@pytest.mark.timeout(1800)
@pytest.mark.parametrize("name", ["candy", "efficientvit", "yolox"])
def test_batched_models_small(ctx, name):
    """The batched model graphs of the C3 / C5 batch sweep (batch 2; batched pointwise
    convolutions as token-major MatMuls) through the library, operator-aligned and
    BLP-selected orchestrations against the oracle."""
    from korch_workloads.models import efficientvit, yolox_nano
    g = {"candy": lambda: candy(size=32, blocks=1, batch=2),
         "efficientvit": lambda: efficientvit(size=64, depths=(1, 1, 1, 1, 1), batch=2),
         "yolox": lambda: yolox_nano(size=64, batch=2)}[name]()
    n, k_sel, k_base = _run_and_check(ctx, g)
    assert n > 500
