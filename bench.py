#!/usr/bin/env python
"""Benchmark: end-to-end latency of the Korch-orchestrated executable (bs=1) on B200.

A "step" is one inference of the selected orchestration (H10 in SURVEY.md §8(a)): the
whole primitive graph executed as the BLP-chosen fused kernels (one CUDA-graph replay).
The one-time tuning (load -> fission -> enumerate -> NVRTC -> on-device profiling ->
HiGHS BLP -> accept) runs before the warm-up and is reported under "tuning".

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl korch|reference]

N > 1 runs under torchrun: every rank runs its own bs=1 replica (the path does not
shard below one image), timings are gathered over NCCL and the
max over ranks is reported.  Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BASELINE = json.load(open(os.path.join(ROOT, "BASELINE.json")))
METRIC = BASELINE["metric"]


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"],
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained"), "source": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "source": "fallback"}


def config_graph(name: str, batch: int = 1):
    from korch_workloads import c1_softmax_layernorm, c2_vit_attention
    if name == "c1":
        return c1_softmax_layernorm(rows=4 * batch), {"workload": "C1 softmax+LayerNorm 4x128 fp32 (BASELINE configs[0])"}
    if name == "c1_bw":
        return c1_softmax_layernorm(rows=1 << 20), {"workload": "C1 bandwidth variant x[2^20,128] fp32"}
    if name == "c2":
        return c2_vit_attention(batch=batch), {
            "workload": "C2 ViT-B pre-LN MHSA layer, seq 128, hidden 768, 12 heads, bf16 (BASELINE configs[1])"}
    raise ValueError(name)


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.samples = []
        if not self.proc:
            return
        self.proc.terminate()
        out, _ = self.proc.communicate()
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 7:
                self.samples.append(f)

    def summary(self):
        if not getattr(self, "samples", None):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for s in self.samples:
            for n, v in zip(names, s[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.samples)}


def load_ncu_traffic(kernel_name: str):
    """dram bytes per launch for `kernel_name` from a committed ncu --set full summary."""
    d = os.path.join(ROOT, "profiles")
    if not os.path.isdir(d):
        return None
    for f in sorted(os.listdir(d)):
        if f.endswith("_ncu_full.json"):
            try:
                j = json.load(open(os.path.join(d, f)))
            except Exception:
                continue
            k = j.get("kernels", {}).get(kernel_name)
            if k and "dram_bytes" in k:
                return k["dram_bytes"]
    return None


def oracle_baseline(graph, sel_cands, sel, budget_s=15.0):
    """The oracle as it stands (fp64 numpy) executing the same orchestration on the host."""
    import numpy as np
    from korch_workloads import make_inputs
    from oracle.enumeration import PGraph
    from oracle.evaluate import eval_orchestration
    from oracle.fission import fission
    pg = fission(graph)
    G = PGraph(pg)
    ins = {k: v[0] for k, v in make_inputs(graph, seed=0).items()}
    n, t0 = 0, time.perf_counter()
    while True:
        eval_orchestration(pg, sel_cands, sel, ins, G.topo_index, graph["dtype"])
        n += 1
        el = time.perf_counter() - t0
        if el > budget_s or n >= 2000:
            break
    cores = len(os.sched_getaffinity(0))
    try:
        import threadpoolctl
        info = threadpoolctl.threadpool_info()
        blas = max((x.get("num_threads", 1) for x in info), default=1)
    except Exception:
        blas = cores
    res = {"value": el / n * 1e3, "unit": "ms", "cores": int(blas), "host_cores": cores, "kind": "oracle",
           "sample": f"{n} inferences of the selected orchestration (fp64 numpy, bf16/fp32 rounding at kernel outputs), {el:.1f} s"}
    # SURVEY.md §8(d) oracle tasks: the same at one BLAS thread, and the unfissioned
    # operator interpreter
    from oracle.operators import eval_operator_graph

    def timed(fn, budget):
        k, t = 0, time.perf_counter()
        while True:
            fn()
            k += 1
            if time.perf_counter() - t > budget or k >= 2000:
                return (time.perf_counter() - t) / k * 1e3, k
    try:
        import threadpoolctl
        with threadpoolctl.threadpool_limits(1):
            res["single_thread_ms"], _ = timed(
                lambda: eval_orchestration(pg, sel_cands, sel, ins, G.topo_index, graph["dtype"]), budget_s / 3)
    except Exception as e:
        res["single_thread_ms"] = f"unavailable: {e}"[:120]
    res["operator_interpreter_ms"], _ = timed(lambda: eval_operator_graph(graph, ins), budget_s / 3)
    return res


def time_plan(kg, sel, dev_in, steps=20, flush_mb=512):
    """Mean device ms per execution of orchestration `sel` (CUDA events on the launch
    stream, L2 flushed between steps outside the events)."""
    import torch
    kg.set_orchestration(sel)
    outs, ws = kg.torch_outputs(), kg.torch_workspace()
    stream = torch.cuda.current_stream()
    flush = torch.empty(flush_mb << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        kg.execute(dev_in, outs, ws, stream)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    torch.cuda.synchronize()
    for i, (a, e) in enumerate(ev):
        flush.fill_(i & 0xFF)
        a.record(stream)
        kg.execute(dev_in, outs, ws, stream)
        e.record(stream)
    torch.cuda.synchronize()
    return statistics.mean(a.elapsed_time(e) for a, e in ev), outs


MODEL_MAX_PRIMS = 12  # SPEC S:393's default; whole models only (reading A5)
DEFAULT_MODELS = ["candy", "efficientvit", "yolox", "segformer", "efficientvit2048"]
TUNING_DB = os.path.join(ROOT, "profiles", "tuning_db")


def model_graph(name: str, batch: int = 1):
    from korch_workloads.models import MODELS
    return MODELS[name]() if batch == 1 else MODELS[name](batch=batch)


def model_enum_opts(kg) -> dict:
    """Enumeration options for whole models: partitioned (reading A17, <= 64 primitives
    per part) and max_prims = 12, raised to the largest operator fragment so
    the one-kernel-per-operator baseline stays in the candidate set (reading A5)."""
    frag = {}
    for n in kg.prim["nodes"]:
        frag[n["op"]] = frag.get(n["op"], 0) + 1
    return {"partition_max": 64, "max_prims": max(MODEL_MAX_PRIMS, max(frag.values()))}


def timed_steps(fn, stream, steps, flush):
    """Per-step device ms (CUDA events on `stream`), L2 flushed between steps outside the
    events."""
    import torch
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    torch.cuda.synchronize()
    for i, (a, e) in enumerate(ev):
        flush.fill_(i & 0xFF)
        a.record(stream)
        fn()
        e.record(stream)
    torch.cuda.synchronize()
    return [a.elapsed_time(e) for a, e in ev]


def dist_summary(ts):
    qs = sorted(ts)

    def pct(q):
        return qs[min(len(qs) - 1, int(round(q * (len(qs) - 1))))]
    return {"mean": statistics.mean(ts), "p10": pct(0.1), "p50": statistics.median(ts), "p90": pct(0.9)}


# FP32 FMA peak of the SIMT kernels (direct convolution, skinny-K MatMul, SIMT
# contractions): 148 SMs x 128 FP32 lanes x 2 flop x 1.965 GHz (B200_PROFILING.md unit
# counts and the max SM clock)
FP32_SIMT_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12


def linear_flops(kg, members):
    """2 x multiply-adds of the dense linear members (Conv2d, MatMul) of a candidate, from the
    primitive graph's shapes: the flops of a window / contraction kernel whose template did
    not record them (a row-template plan carrying a direct-convolution variant)."""
    nodes = {n["id"]: n for n in kg.prim["nodes"]}
    ins = {x["name"]: x["shape"] for x in kg.prim["inputs"]}

    def shape(ref):
        return ins[ref["input"]] if "input" in ref else nodes[ref["node"]]["shape"]
    f = 0.0
    for m in members:
        n = nodes[m]
        if n["kind"] == "conv2d":
            w = shape(n["inputs"][1])                     # [F, C / groups, R, S]
            f += 2.0 * math.prod(n["shape"]) * w[1] * w[2] * w[3]
        elif n["kind"] == "matmul":
            a = shape(n["inputs"][0])
            f += 2.0 * math.prod(n["shape"]) * a[-1]
    return f


def roofline_of(kg, cands, i, cold_ns, pk):
    """Roofline of candidate i from its algorithmic bytes / flops and a cold-L2 time:
    tcgen05 kernels (GEMMs, attention, the KB6-D tensor-core direct convolution) against
    the bf16 tensor peak or HBM, SIMT kernels with flops (direct conv, skinny-K MatMul)
    against the FP32 FMA peak ("alu") or HBM."""
    c = dict(cands[i])
    name = kg.kernel_name(i)
    if c["flops"] <= 0:
        c["flops"] = linear_flops(kg, c["members"])
    tensor = (name.startswith("korch_gemm") or name.startswith("korch_pgemm") or name.startswith("korch_conv")
              or name.startswith("korch_gg") or name.startswith("korch_attn") or name.startswith("korch_tconv"))
    simt = not tensor
    if simt and c["flops"] > 0 and c["flops"] / (FP32_SIMT_TFLOPS * 1e12) > c["bytes"] / (pk["hbm_gbs"] * 1e9):
        ach = c["flops"] / (cold_ns * 1e-9) / 1e12
        r = {"bound": "alu", "achieved": ach, "peak": FP32_SIMT_TFLOPS, "unit": "TFLOP/s",
             "peak_source": "148 SM x 128 FP32 lanes x 2 x 1.965 GHz"}
        r["frac"] = r["achieved"] / r["peak"]
        r.update({"traffic": load_ncu_traffic(name), "candidate": i, "class": c["klass"], "members": len(c["members"]),
                  "algorithmic_bytes": c["bytes"], "flops": c["flops"], "ns_cold_l2": cold_ns, "name": name,
                  "variant": kg.variant_info(i)[2]})
        return r
    ridge = pk["bf16_tflops"] * 1e12 / (pk["hbm_gbs"] * 1e9)
    ai = c["flops"] / max(1, c["bytes"]) if tensor else 0.0
    if ai > ridge:
        ach = c["flops"] / (cold_ns * 1e-9) / 1e12
        r = {"bound": "tensor", "achieved": ach, "peak": pk["bf16_tflops"], "unit": "TFLOP/s"}
    else:
        ach = c["bytes"] / (cold_ns * 1e-9) / 1e9
        r = {"bound": "hbm", "achieved": ach, "peak": pk["hbm_gbs"], "unit": "GB/s"}
    r["frac"] = r["achieved"] / r["peak"]
    r.update({"traffic": load_ncu_traffic(name), "candidate": i, "class": c["klass"], "members": len(c["members"]),
              "algorithmic_bytes": c["bytes"], "flops": c["flops"], "ns_cold_l2": cold_ns, "name": name,
              "variant": kg.variant_info(i)[2]})
    return r


def run_model(K, name, pk, steps=50, oracle_check=True, retune=False, db_dir=TUNING_DB, flush=None):
    """One paper model at its paper input size, bs 1: partitioned enumeration,
    costs from the tuning database (tunedb.py; recorded on a B200 by tools/tune_models.py,
    P:629) or profiled live, exact Eq. 2-4 selection, then the chosen orchestration and the
    operator-aligned one (one kernel per unfused operator) timed end to end with L2 flushed
    between steps and clocks sampled; output checked against the fp64 oracle."""
    import numpy as np
    import torch
    import paper_2406_09465_b200.select as S
    from korch_workloads import make_inputs
    from paper_2406_09465_b200 import tunedb
    t0 = time.perf_counter()
    graph = model_graph(name)
    ctx = K.Context(torch.cuda.current_device())
    kg = K.KorchGraph(ctx, graph)
    opts = model_enum_opts(kg)
    cands = kg.enumerate(**opts)
    t_enum = time.perf_counter() - t0
    db_path = os.path.join(db_dir, f"{name}_b1.json")
    db = None if retune else tunedb.load(db_path)
    ok, why = tunedb.usable(db, graph, opts)
    t1 = time.perf_counter()
    if ok:
        costs, missing = tunedb.apply(kg, db)
        if missing:
            live = kg.profile(missing)
            for i, c in zip(missing, live):
                costs[i] = c
        tuning = {"source": f"tuning database {os.path.relpath(db_path, ROOT)} (recorded {db.get('created')} on "
                            f"{db.get('device')}, {len(db['kernels'])} kernels)", "profiled_live": len(missing),
                  "recorded_tuning_s": db.get("tuning_s")}
    else:
        kg.compile()
        costs = kg.profile()
        tuning = {"source": f"profiled live ({why})", "profiled_live": len(cands)}
    tuning["profile_s"] = time.perf_counter() - t1
    t1 = time.perf_counter()
    obj, sel = kg.select(costs)
    tuning.update({"enumerate_s": t_enum, "select_s": time.perf_counter() - t1, "solver": S.LAST_SOLVER,
                   "search_states": S.LAST_EXPANDED})
    blp_optimal, blp_gap = S.LAST_OPTIMAL, S.LAST_GAP
    base = kg.operator_aligned()
    ins = make_inputs(graph, seed=0)
    dev = K.torch_inputs(graph, {k: v[1] for k, v in ins.items()})
    stream = torch.cuda.current_stream()
    if flush is None:
        flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    res = {"input": graph["inputs"][0]["shape"], "n_prims": kg.n_prims, "n_candidates": len(cands),
           "n_generable": len(kg.generable()), "n_states": kg.n_states, "parts": len({c["part"] for c in cands})}

    def measure(plan):
        kg.set_orchestration(plan)
        outs, ws = kg.torch_outputs(), kg.torch_workspace()
        for _ in range(5):
            kg.execute(dev, outs, ws, stream)
        with Clocks(torch.cuda.current_device()) as clk:
            ts = timed_steps(lambda: kg.execute(dev, outs, ws, stream), stream, steps, flush)
            # keep the GPU busy until the sampler has seen the load
            t_end = time.perf_counter()
            while time.perf_counter() - t_end < 0.25:
                for _ in range(20):
                    kg.execute(dev, outs, ws, stream)
                torch.cuda.synchronize()
        return dist_summary(ts), clk.summary(), outs, ws
    lat, clocks, outs, ws = measure(sel)
    got = [o.float().cpu().numpy().astype(np.float64) for o in outs]
    order = kg.plan()
    # e2e through korch_execute_host: the image H2D from pinned memory, the plan, and the
    # output written straight into pinned host memory, every step
    xi = [s["name"] for s in graph["inputs"]].index("x")
    host_x = dev[xi].cpu().pin_memory()
    host_out = [torch.empty_like(o, device="cpu").pin_memory() for o in outs]
    hin = [host_x if i == xi else None for i in range(len(dev))]
    dev_e2e = list(dev)
    dev_e2e[xi] = torch.empty_like(dev[xi])
    for _ in range(3):
        kg.execute_host(hin, dev_e2e, host_out, outs, ws, stream)
    e2e = timed_steps(lambda: kg.execute_host(hin, dev_e2e, host_out, outs, ws, stream), stream, max(10, steps // 2),
                      flush)
    torch.cuda.synchronize()
    e2e_match = all(torch.equal(h, g.cpu()) or torch.equal(h.float(), torch.from_numpy(r).to(h.dtype).float())
                    for h, g, r in zip(host_out, outs, got))
    # plan roofline T*(u) = sum_i max(B_i / BW, F_i / P)
    t_star = sum(max(cands[i]["bytes"] / pk["hbm_gbs"], cands[i]["flops"] / (pk["bf16_tflops"] * 1e3)) for i in order)
    dom = max(order, key=lambda i: costs[i])
    dom_cold = kg.profile([dom], flush_l2=True, trials=7, tune=False)[0]
    kinds = {n["id"]: n["kind"] for n in kg.prim["nodes"]}
    top = [{"cand": i, "ns": costs[i], "class": cands[i]["klass"], "bytes": cands[i]["bytes"],
            "flops": cands[i]["flops"], "kinds": [kinds[m] for m in cands[i]["members"]],
            "variant": kg.variant_info(i)[2], "name": kg.kernel_name(i)}
           for i in sorted(order, key=lambda i: -costs[i])[:5]]
    base_lat, base_clocks, _, _ = measure(base)
    # fission + greedy fusion without the BLP (P:505-518 ablation, reading A35), same costs
    greedy = S.greedy_fusion(cands, costs, kg.prim, kg.outputs)
    try:
        g_lat, _, _, _ = measure(greedy)
        res["greedy_fusion"] = {"latency_ms": g_lat["p50"], "kernels": len(greedy),
                                "objective_ns": sum(costs[i] for i in greedy)}
    except Exception as e:  # reported, never silently replaced
        res["greedy_fusion"] = {"error": f"{type(e).__name__}: {e}"[:300], "kernels": len(greedy)}
    # N1 (reading A32): the same model with multi-output candidates, when a tuning database
    # recorded with them exists (profiles/tuning_db/<model>_b1_mo2.json)
    mo_db = tunedb.load(os.path.join(db_dir, f"{name}_b1_mo2.json"))
    if mo_db is not None:
        try:
            mopts = dict(opts, max_outputs=2)
            kg2 = K.KorchGraph(ctx, graph)
            c2 = kg2.enumerate(**mopts)
            ok2, why2 = tunedb.usable(mo_db, graph, mopts)
            if ok2:
                costs2, missing2 = tunedb.apply(kg2, mo_db)
                for i, c in zip(missing2, kg2.profile(missing2) if missing2 else []):
                    costs2[i] = c
                obj2, sel2 = kg2.select(costs2, time_limit=60.0)
                kg2.set_orchestration(sel2)
                o2, w2 = kg2.torch_outputs(), kg2.torch_workspace()
                for _ in range(5):
                    kg2.execute(dev, o2, w2, stream)
                t2 = timed_steps(lambda: kg2.execute(dev, o2, w2, stream), stream, steps, flush)
                same = all(torch.allclose(a.float(), b.float(), rtol=5e-2, atol=5e-2) for a, b in zip(o2, outs))
                res["multi_output"] = {"latency_ms": statistics.median(t2), "kernels": len(kg2.plan()),
                                       "objective_ns": obj2, "n_candidates": len(c2),
                                       "kernels_with_secondary_outputs": sum(1 for i in sel2 if c2[i]["extra_outputs"]),
                                       "blp_optimal": S.LAST_OPTIMAL, "profiled_live": len(missing2),
                                       "outputs_close_to_single_output_plan": same}
            else:
                res["multi_output"] = {"skipped": why2}
            del kg2
        except Exception as e:  # reported, never silently replaced
            res["multi_output"] = {"error": f"{type(e).__name__}: {e}"[:300]}
    res.update({"latency_ms": lat["p50"], "latency_ms_dist": lat, "clocks": clocks, "kernels": len(order),
                "e2e_ms": statistics.median(e2e), "e2e_h2d_bytes": host_x.numel() * host_x.element_size(),
                "e2e_d2h_bytes": sum(t.numel() * t.element_size() for t in host_out), "e2e_output_matches": e2e_match,
                "operator_aligned_ms": base_lat["p50"], "operator_aligned_ms_dist": base_lat,
                "operator_aligned_kernels": len(base), "operator_aligned_clocks": base_clocks,
                "speedup_vs_operator_aligned": base_lat["p50"] / lat["p50"],
                "blp_objective_ns": obj, "operator_aligned_objective_ns": sum(costs[i] for i in base),
                "blp_optimal": blp_optimal, "blp_max_rel_gap": blp_gap,
                "plan_roofline": {"t_star_us": t_star / 1e3, "frac_of_t_star": t_star / (lat["p50"] * 1e6),
                                  "bytes": sum(cands[i]["bytes"] for i in order),
                                  "flops": sum(cands[i]["flops"] for i in order)},
                "dominant": roofline_of(kg, cands, dom, dom_cold, pk), "slowest_selected": top,
                "tuning": tuning})
    if oracle_check:
        from oracle.enumeration import PGraph
        from oracle.evaluate import eval_orchestration
        from oracle.fission import fission
        t1 = time.perf_counter()
        pg = fission(graph)
        G = PGraph(pg)
        want = eval_orchestration(pg, [(tuple(c["members"]), c["output"]) for c in cands], sel,
                                  {k: v[0] for k, v in ins.items()}, G.topo_index, graph["dtype"])
        errs = [float(np.max(np.abs(g - want[o])) / np.max(np.abs(want[o]))) for g, o in zip(got, kg.outputs)]
        l2s = [float(np.linalg.norm(g - want[o]) / np.linalg.norm(want[o])) for g, o in zip(got, kg.outputs)]
        res["oracle_rel_err"] = max(errs)
        res["oracle_rel_l2"] = max(l2s)
        # reading A36: whole bf16 models, relative L2 <= 2e-2 and max-norm <= 5e-2
        res["oracle_tol"] = {"rel_l2": 2e-2, "max_norm": 5e-2} if graph["dtype"] == "bf16" else 1e-4
        res["oracle_s"] = time.perf_counter() - t1
    res["wall_s"] = time.perf_counter() - t0
    print("[models] " + json.dumps({name: {k: res[k] for k in ("latency_ms", "operator_aligned_ms", "kernels",
                                                             "blp_optimal", "wall_s")}}), file=sys.stderr, flush=True)
    del kg, outs, dev, ws
    ctx.close()
    torch.cuda.empty_cache()
    return res


SCALING_MODELS = ["efficientvit", "yolox", "candy"]   # BASELINE configs C3 (EfficientViT) and C5 (YOLOX / Candy)
SCALING_GLOBAL_BATCH = 8


def model_batch_throughput(K, name, pk, global_batch=SCALING_GLOBAL_BATCH, steps=20, flush=None, coll_dev=None,
                           db_dir=TUNING_DB):
    """BASELINE C3 / C5: a paper model at a global batch sharded over the
    ranks.  Each rank runs the orchestration selected for its LOCAL batch (reading A26;
    costs from the tuning database recorded at that batch, else profiled live with the
    candidates shared round-robin across ranks and MIN-all-reduced, G1), with no
    communication on the data path; the step time is the max over ranks (G4) and the
    output shards are all-gathered afterwards (G3, outside the timed region)."""
    import torch
    import torch.distributed as dist
    import paper_2406_09465_b200.select as S
    from korch_workloads import make_inputs
    from paper_2406_09465_b200 import tunedb
    from paper_2406_09465_b200.dist import max_over_ranks, merge_costs, my_share, shard, world
    rank, ws_, _ = world()
    lo, hi = shard(global_batch, rank, ws_)
    batch = hi - lo
    graph = model_graph(name, batch)
    ctx = K.Context(torch.cuda.current_device())
    kg = K.KorchGraph(ctx, graph)
    opts = model_enum_opts(kg)
    cands = kg.enumerate(**opts)
    t0 = time.perf_counter()
    db_path = os.path.join(db_dir, f"{name}_b{batch}.json")
    db = tunedb.load(db_path)
    ok, why = tunedb.usable(db, graph, opts)
    if ok:
        costs, missing = tunedb.apply(kg, db)
        if missing:
            for i, c in zip(missing, kg.profile(missing)):
                costs[i] = c
        source = f"tuning database {os.path.relpath(db_path, ROOT)} ({len(missing)} profiled live)"
    else:
        # No database at this local batch: a BOUNDED live search keeps the benchmark within
        # minutes -- the operator-aligned kernels plus every candidate of <= 2 primitives
        # (the full search is tools/tune_models.py --batch B, minutes to tens of minutes per
        # model); the remaining candidates are left out (cost = INF), so the selection is
        # optimal over this subset only and is reported as such.
        base = set(kg.operator_aligned())
        pool = [i for i in kg.generable() if i in base or len(cands[i]["members"]) <= 2]
        kg.compile(pool)
        costs = [K.INF] * len(cands)
        if ws_ > 1 and global_batch % ws_ == 0:
            mine = [pool[j] for j in my_share(len(pool), rank, ws_)]
            part = kg.profile(mine)
            merged, variants = merge_costs(mine, part, [kg.variant_info(i)[1] for i in mine], len(cands),
                                           device=coll_dev)
            for i in pool:
                costs[i] = merged[i]
                if variants[i] >= 0:
                    kg.set_variant(i, variants[i])
            source = f"bounded live search, sharded over {ws_} ranks ({why}): {len(pool)} candidates"
        else:
            for i, c in zip(pool, kg.profile(pool)):
                costs[i] = c
            source = f"bounded live search ({why}): {len(pool)} of {len(cands)} candidates"
    obj, sel = kg.select(costs)
    t_tune = time.perf_counter() - t0
    ins = make_inputs(graph, seed=100 + rank)
    dev = K.torch_inputs(graph, {k: v[1] for k, v in ins.items()})
    stream = torch.cuda.current_stream()
    if flush is None:
        flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    kg.set_orchestration(sel)
    outs, wsb = kg.torch_outputs(), kg.torch_workspace()
    for _ in range(5):
        kg.execute(dev, outs, wsb, stream)
    if ws_ > 1:
        dist.barrier()
    ts = timed_steps(lambda: kg.execute(dev, outs, wsb, stream), stream, steps, flush)
    ms = statistics.median(ts)
    ms_max, = max_over_ranks([ms], device=coll_dev)
    gather_ms = None
    if ws_ > 1:
        o = outs[0].contiguous() if coll_dev else outs[0].float().cpu()
        bufs = [torch.empty_like(o) for _ in range(ws_)]
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        dist.all_gather(bufs, o)
        torch.cuda.synchronize()
        gather_ms = (time.perf_counter() - t1) * 1e3
    res = {"global_batch": global_batch, "local_batch": batch, "n_gpus": ws_, "ms": ms_max, "ms_rank0": ms,
           "throughput": {"value": global_batch / (ms_max * 1e-3), "unit": "images/s"},
           "kernels": len(kg.plan()), "blp_objective_ns": obj, "blp_optimal": S.LAST_OPTIMAL, "tuning": source,
           "tune_s": t_tune, "output_gather_ms_host_timed": gather_ms}
    del kg, outs, dev, wsb
    ctx.close()
    torch.cuda.empty_cache()
    return res


def scaled_variant(K, pk, global_batch=64, steps=10, coll_dev=None):
    """C2 at global batch 64 (M = 8192 tokens; SURVEY.md §8(d) C2 scale list) sharded over
    the ranks (§8(e)): each rank tunes and selects for its LOCAL batch (reading A26), runs
    its shard with no communication, and the step time is the max over ranks (G4); the
    output shards are then all-gathered (G3, timed separately).  The dominant kernel is
    re-timed cold against the tensor (or HBM) roofline."""
    import torch
    import torch.distributed as dist
    from korch_workloads import make_inputs
    from paper_2406_09465_b200.dist import (broadcast_selection, max_over_ranks, merge_costs, my_share, shard,
                                            world)
    rank, ws_, _ = world()
    lo, hi = shard(global_batch, rank, ws_)
    batch = hi - lo
    graph, cfg = config_graph("c2", batch)
    ctx = K.Context(torch.cuda.current_device())
    kg = K.KorchGraph(ctx, graph)
    cands = kg.enumerate(attention_pairs=True)
    t0 = time.perf_counter()
    if ws_ > 1 and global_batch % ws_ == 0:
        # equal shards -> identical graphs: profile a share each, MIN all-reduce (G1)
        mine = my_share(len(cands), rank, ws_)
        part = kg.profile(mine)
        costs, variants = merge_costs(mine, part, [kg.variant_info(i)[1] for i in mine], len(cands),
                                      device=coll_dev)
        for i, v in enumerate(variants):
            if v >= 0:
                kg.set_variant(i, v)
        obj, sel = kg.select(costs)
        sel = broadcast_selection(sel, src=0, device=coll_dev)
    else:
        costs = kg.profile()
        obj, sel = kg.select(costs)
    t_tune = time.perf_counter() - t0
    ins = make_inputs(graph, seed=1000 + rank)
    dev = K.torch_inputs(graph, {k: v[1] for k, v in ins.items()})
    if ws_ > 1:
        dist.barrier()
    ms, outs = time_plan(kg, sel, dev, steps=steps)
    ms_max, = max_over_ranks([ms], device=coll_dev)
    gather_ms = None
    if ws_ > 1:
        o = outs[0].contiguous() if coll_dev else outs[0].float().cpu()
        bufs = [torch.empty_like(o) for _ in range(ws_)]
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        for _ in range(3):
            dist.all_gather(bufs, o)
        torch.cuda.synchronize()
        gather_ms = (time.perf_counter() - t1) / 3 * 1e3
    order = kg.plan()
    dom = max(order, key=lambda i: costs[i])
    cold = kg.profile([dom], flush_l2=True, trials=7, tune=False)[0]
    dc = cands[dom]
    flops = sum(cands[i]["flops"] for i in order)
    res = {"workload": f"C2 ViT-B MHSA layer, global batch {global_batch} x seq 128 sharded over {ws_} GPU(s), "
                       f"local batch {batch} (M = {batch * 128}), bf16",
           "ms": ms_max, "ms_rank0": ms, "local_batch": batch, "kernels": len(order),
           "throughput": {"value": global_batch / (ms_max * 1e-3), "unit": "sequences/s (seq 128)"},
           "tflops_plan": flops / (ms * 1e-3) / 1e12, "tune_s": t_tune, "output_gather_ms_host_timed": gather_ms,
           "plan_members": [cands[i]["members"] for i in order],
           "dominant": {"candidate": dom, "class": dc["klass"], "members": len(dc["members"]),
                        "ns_cold_l2": cold, "variant": kg.variant_info(dom)[2], "name": kg.kernel_name(dom)}}
    if dc["flops"] > 0:
        t = dc["flops"] / (cold * 1e-9) / 1e12
        res["dominant"].update({"bound": "tensor", "achieved_tflops": t, "peak_tflops": pk["bf16_tflops"],
                                "frac": t / pk["bf16_tflops"]})
    else:
        gbs = dc["bytes"] / cold
        res["dominant"].update({"bound": "hbm", "achieved_gbs": gbs, "peak_gbs": pk["hbm_gbs"],
                                "frac": gbs / pk["hbm_gbs"]})
    ctx.close()
    return res


def bandwidth_variant(K, pk, steps=10):
    """C1 at x[2^20,128] fp32 (SURVEY.md §8(d) C1 bandwidth variant): enumerate, profile
    (cold, inputs > L2), BLP-select, execute; achieved GB/s of the plan and of its
    dominant kernel against the measured HBM peak."""
    import torch
    graph, cfg = config_graph("c1_bw")
    ctx = K.Context(torch.cuda.current_device())
    kg = K.KorchGraph(ctx, graph)
    cands = kg.enumerate()
    costs = kg.profile(warmup=1, launches=2, trials=3)
    obj, sel = kg.select(costs)
    kg.set_orchestration(sel)
    order = kg.plan()
    x = torch.randn(graph["inputs"][0]["shape"], device="cuda")
    g = 1 + 0.1 * torch.randn(graph["inputs"][1]["shape"], device="cuda")
    b = 0.1 * torch.randn(graph["inputs"][2]["shape"], device="cuda")
    outs, ws = kg.torch_outputs(), kg.torch_workspace()
    stream = torch.cuda.current_stream()
    for _ in range(2):
        kg.execute([x, g, b], outs, ws, stream)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    torch.cuda.synchronize()
    for a, e in ev:
        a.record(stream)
        kg.execute([x, g, b], outs, ws, stream)
        e.record(stream)
    torch.cuda.synchronize()
    ms = statistics.median(a.elapsed_time(e) for a, e in ev)
    plan_bytes = sum(cands[i]["bytes"] for i in order)
    dom = max(order, key=lambda i: costs[i])
    res = {"workload": cfg["workload"], "kernels": len(order), "ms": ms, "plan_bytes": plan_bytes,
           "achieved_gbs": plan_bytes / (ms * 1e-3) / 1e9, "peak_gbs": pk["hbm_gbs"],
           "frac": plan_bytes / (ms * 1e-3) / 1e9 / pk["hbm_gbs"],
           "dominant": {"candidate": dom, "members": len(cands[dom]["members"]), "class": cands[dom]["klass"],
                        "bytes": cands[dom]["bytes"], "ns": costs[dom],
                        "gbs": cands[dom]["bytes"] / costs[dom], "variant": kg.variant_info(dom)[2],
                        "name": cands[dom]["signature"]},
           "blp_objective_ns": obj,
           "operator_aligned_ns": sum(costs[i] for i in kg.operator_aligned())}
    del x, outs, ws
    ctx.close()
    return res


def run_reference(args):
    """--impl reference: the oracle (the paper has no runnable reference here), timed on the
    host cores on this arm's workload, bounded to a few minutes."""
    import numpy as np
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    graph, cfg = config_graph(args.config)
    from korch_workloads import make_inputs
    from oracle.operators import eval_operator_graph
    ins = {k: v[0] for k, v in make_inputs(graph, seed=0).items()}
    for _ in range(args.warmup):
        eval_operator_graph(graph, ins)
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        eval_operator_graph(graph, ins)
        ts.append((time.perf_counter() - t0) * 1e3)
    ms = statistics.mean(ts)
    cores = len(os.sched_getaffinity(0))
    line = {"impl": "reference", "metric": METRIC, "value": ms, "unit": "ms", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": dict(cfg, batch=1),
            "cpu_baseline": {"value": ms, "unit": "ms", "cores": cores, "kind": "oracle",
                             "sample": f"{args.steps} unfissioned fp64 operator-graph evaluations"},
            "e2e": {"value": ms, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def spawn_ranks(n: int) -> int:
    """`bench.py --gpus N` started without a launcher: start N ranks (one process per GPU)
    the way the driver does, `torch.distributed.run` on 127.0.0.1, with the same
    arguments; rank 0 prints the JSON line."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default=os.environ.get("KORCH_BENCH_CONFIG", "c2"))
    ap.add_argument("--impl", default="korch", choices=["korch", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-bw-variant", action="store_true", help="skip the C1 x[2^20,128] bandwidth measurement")
    ap.add_argument("--models", default=",".join(DEFAULT_MODELS),
                    help="comma list of whole paper models to time at bs 1 ('' = none)")
    ap.add_argument("--retune", action="store_true", help="profile the models live instead of using the tuning database")
    ap.add_argument("--scaling-models", default=",".join(SCALING_MODELS),
                    help="models timed at --scaling-batch global batch, sharded over the ranks ('' = none)")
    ap.add_argument("--scaling-batch", type=int, default=SCALING_GLOBAL_BATCH)
    ap.add_argument("--no-scaled", action="store_true", help="skip the C2 batch-64 measurement")
    ap.add_argument("--no-attention-pairs", action="store_true",
                    help="paper-faithful P:626 prune only (no fused two-GEMM attention candidates)")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--save-selection", default=None, help="write the chosen plan (for tools/replay.py)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args.gpus)
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    # one process per GPU; KORCH_DIST_BACKEND=gloo + more ranks than GPUs is a test mode
    # that exercises the multi-rank logic on one device
    backend = os.environ.get("KORCH_DIST_BACKEND", "nccl")
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    coll_dev = "cuda" if backend == "nccl" else None
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)

    import paper_2406_09465_b200 as K
    from korch_workloads import make_inputs

    graph, cfg = config_graph(args.config)
    pk = peaks()
    t_all = time.perf_counter()
    ctx = K.Context(local)
    kg = K.KorchGraph(ctx, graph)
    t0 = time.perf_counter()
    # NEXT item N2: two-GEMM attention candidates join the search
    cands = kg.enumerate(attention_pairs=not args.no_attention_pairs)
    t_enum = time.perf_counter() - t0
    t0 = time.perf_counter()
    kg.compile()
    t_compile = time.perf_counter() - t0
    t0 = time.perf_counter()
    from paper_2406_09465_b200.dist import broadcast_selection, merge_costs, my_share
    if world > 1:
        # profiling sharded across the GPUs (G1: MIN all-reduce of costs + variants)
        mine = my_share(len(cands), rank, world)
        local = kg.profile(mine)
        costs, variants = merge_costs(mine, local, [kg.variant_info(i)[1] for i in mine], len(cands),
                                      device=coll_dev)
        for i, v in enumerate(variants):
            if v >= 0:
                kg.set_variant(i, v)
    else:
        costs = kg.profile()
    t_prof = time.perf_counter() - t0
    t0 = time.perf_counter()
    obj, sel = kg.select(costs)
    if world > 1:
        sel = broadcast_selection(sel, src=0, device=coll_dev)   # G2: rank 0's selection
        obj = sum(costs[i] for i in sel)
    t_sel = time.perf_counter() - t0
    base = kg.operator_aligned()
    base_obj = sum(costs[i] for i in base) if all(costs[i] < K.INF for i in base) else None
    kg.set_orchestration(sel)
    order = kg.plan()
    if args.save_selection:
        json.dump({"config": args.config, "batch": 1, "selection": sel,
                   "attention_pairs": not args.no_attention_pairs,
                   "variants": {str(i): kg.variant_info(i)[1] for i in order},
                   "tags": {str(i): kg.variant_info(i)[2] for i in order},
                   "kernels": {str(i): cands[i]["signature"] for i in order},
                   "costs_ns": {str(i): costs[i] for i in order},
                   "all_costs_ns": costs,
                   "all_variants": [kg.variant_info(i)[1] for i in range(len(cands))]},
                  open(args.save_selection, "w"), indent=1)
    tuning = {"enumerate_s": t_enum, "compile_s": t_compile, "profile_s": t_prof, "select_s": t_sel,
              "total_s": time.perf_counter() - t_all, "n_candidates": len(cands), "n_states": kg.n_states,
              "n_generable": len(kg.generable()), "n_prims": kg.n_prims}

    ins = make_inputs(graph, seed=0)
    dev_in = K.torch_inputs(graph, {k: v[1] for k, v in ins.items()})
    outs = kg.torch_outputs()
    ws = kg.torch_workspace()
    stream = torch.cuda.current_stream()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2

    def step():
        kg.execute(dev_in, outs, ws, stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # device-timed steps, L2 flushed between steps (flush outside the events)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        # keep the GPU busy with the same workload until the sampler has produced samples,
        # then run the timed steps (each bracketed by events, L2 flushed in between)
        t_start = time.perf_counter()
        while time.perf_counter() - t_start < 0.6:
            for _ in range(50):
                step()
            torch.cuda.synchronize()
        for i in range(args.steps):
            flush.fill_(i & 0xFF)
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
        torch.cuda.synchronize()
        t_end = time.perf_counter()
        while time.perf_counter() - t_end < 0.3:
            for _ in range(50):
                step()
            torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    times = [a.elapsed_time(b) for a, b in ev]
    ms = statistics.mean(times)
    qs = sorted(times)

    def pct(q):
        return qs[min(len(qs) - 1, int(round(q * (len(qs) - 1))))]
    dist_ms = {"mean": ms, "median": statistics.median(times), "p10": pct(0.1), "p90": pct(0.9)}

    # warm back-to-back replays (context: the regime the profiler measures in)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    warm_ms = e0.elapsed_time(e1) / args.steps

    # e2e through the public API with host buffers: H2D of the activation input(s),
    # execute, D2H of the output, every step
    act_names = [s["name"] for s in graph["inputs"] if s["name"] == "x"]
    host_in = {n: dev_in[[s["name"] for s in graph["inputs"]].index(n)].cpu().pin_memory() for n in act_names}
    host_out = [torch.empty_like(o, device="cpu").pin_memory() for o in outs]
    h2d = sum(t.numel() * t.element_size() for t in host_in.values())
    d2h = sum(t.numel() * t.element_size() for t in host_out)
    idx_of = {s["name"]: i for i, s in enumerate(graph["inputs"])}
    # korch_execute_host: the H2D copies, the plan and the D2H copies in one graph replay
    hin = [host_in.get(s["name"]) for s in graph["inputs"]]

    def e2e_step():
        kg.execute_host(hin, dev_in, host_out, outs, ws, stream)
    for _ in range(args.warmup):
        e2e_step()
    torch.cuda.synchronize()
    ee = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for i in range(args.steps):
        flush.fill_(i & 0xFF)
        ee[i][0].record(stream)
        e2e_step()
        ee[i][1].record(stream)
    torch.cuda.synchronize()
    e2e_ms = statistics.mean(a.elapsed_time(b) for a, b in ee)

    # dominant kernel: largest profiled cost in the plan; re-time it cold-L2 on its stream
    dom = max(order, key=lambda i: costs[i])
    dom_cold = kg.profile([dom], flush_l2=True, trials=9, tune=False)[0]
    dc = cands[dom]
    if dc["klass"] == "gemm" and dc["flops"] > 0:
        # compute-class kernel: report against the bf16 tensor peak if it is compute bound
        ai = dc["flops"] / max(1, dc["bytes"])
        ridge = pk["bf16_tflops"] * 1e12 / (pk["hbm_gbs"] * 1e9)
    else:
        ai, ridge = 0.0, 1.0
    if ai > ridge:
        ach = dc["flops"] / (dom_cold * 1e-9) / 1e12
        roof = {"bound": "tensor", "achieved": ach, "peak": pk["bf16_tflops"], "unit": "TFLOP/s"}
    else:
        ach = dc["bytes"] / (dom_cold * 1e-9) / 1e9
        roof = {"bound": "hbm", "achieved": ach, "peak": pk["hbm_gbs"], "unit": "GB/s"}
    roof["frac"] = roof["achieved"] / roof["peak"]
    kname = kg.kernel_name(dom)
    roof["traffic"] = load_ncu_traffic(kname)
    roof["kernel"] = {"candidate": dom, "class": dc["klass"], "members": len(dc["members"]),
                      "algorithmic_bytes": dc["bytes"], "flops": dc["flops"], "ns_cold_l2": dom_cold,
                      "ns_warm": costs[dom], "name": kname, "peak_source": pk["source"]}

    # plan roofline: T*(u) = sum_i max(B_i / BW, F_i / P) over the selected
    # kernels, and the launch floor n_kernels * t_min + T*(u), t_min = the cheapest profiled
    # candidate of this graph (one launch of a near-empty kernel in graph replay)
    t_star_ns = sum(max(cands[i]["bytes"] / pk["hbm_gbs"], cands[i]["flops"] / (pk["bf16_tflops"] * 1e3))
                    for i in order)
    t_min_ns = min(c for c in costs if c < K.INF)
    plan_roof = {"t_star_us": t_star_ns / 1e3, "t_min_kernel_us": t_min_ns / 1e3,
                 "floor_us": (len(order) * t_min_ns + t_star_ns) / 1e3,
                 "frac_of_t_star": t_star_ns / (ms * 1e6), "frac_of_floor": (len(order) * t_min_ns + t_star_ns) / (ms * 1e6),
                 "bytes": sum(cands[i]["bytes"] for i in order), "flops": sum(cands[i]["flops"] for i in order)}

    # gather max over ranks (G4): a step takes as long as its slowest rank
    from paper_2406_09465_b200.dist import max_over_ranks
    ms_max, e2e_max = max_over_ranks([ms, e2e_ms], device=coll_dev)
    # G3: gather every replica's output (outside the timed region); identical inputs and an
    # identical orchestration must give bitwise-identical outputs on every GPU
    replicas_agree = None
    if world > 1:
        o0 = outs[0].contiguous() if coll_dev else outs[0].float().cpu()
        gathered = [torch.empty_like(o0) for _ in range(world)]
        dist.all_gather(gathered, o0)
        replicas_agree = all(torch.equal(gathered[0], x) for x in gathered[1:])

    # the operator-aligned orchestration measured end to end (BASELINE target)
    base_ms = None
    if base_obj is not None:
        base_ms, _ = time_plan(kg, base, dev_in, steps=args.steps)
        kg.set_orchestration(sel)
    models = None
    if args.models:
        # every rank runs every model (bs 1 does not shard: replicas); the reported latency
        # is the max over ranks of each rank's median step (G4)
        models = {}
        for m in [m for m in args.models.split(",") if m]:
            try:
                models[m] = run_model(K, m, pk, steps=max(20, args.steps), retune=args.retune, flush=flush,
                                      oracle_check=rank == 0)
                lat = models[m]["latency_ms"]
            except Exception as e:  # reported, never silently replaced
                models[m] = {"error": f"{type(e).__name__}: {e}"[:400]}
                lat = float("nan")
            if world > 1:
                lat_max, = max_over_ranks([lat], device=coll_dev)
                models[m]["latency_ms_rank0"] = models[m].get("latency_ms")
                models[m]["latency_ms"] = lat_max
    model_scaling = None
    if args.scaling_models:
        model_scaling = {}
        for m in [m for m in args.scaling_models.split(",") if m]:
            try:
                model_scaling[m] = model_batch_throughput(K, m, pk, global_batch=args.scaling_batch, flush=flush,
                                                          coll_dev=coll_dev)
            except Exception as e:  # reported, never silently replaced
                model_scaling[m] = {"error": f"{type(e).__name__}: {e}"[:400]}
    scaled = None
    if not args.no_scaled and args.config == "c2":
        try:
            scaled = scaled_variant(K, pk, coll_dev=coll_dev)
            # P:610-620 / SURVEY N3: is the optimal orchestration batch dependent?
            scaled["plan_differs_from_bs1"] = sorted(scaled["plan_members"]) != sorted(cands[i]["members"]
                                                                                       for i in order)
        except Exception as e:
            scaled = {"error": str(e)[:300]}
    bw = None
    if rank == 0 and world == 1 and not args.no_bw_variant:
        try:
            bw = bandwidth_variant(K, pk)
        except Exception as e:  # reported, never silently replaced
            bw = {"error": str(e)[:300]}
    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            cpu = oracle_baseline(graph, [(tuple(c["members"]), c["output"]) for c in cands], sel, args.cpu_budget)
        line = {
            "metric": METRIC, "value": ms_max, "unit": "ms", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": graph["dtype"], "data": "synthetic (seeded PCG64, random-init weights)",
            "config": dict(cfg, batch_per_gpu=1, global_batch=world, l2="flushed between steps (512 MiB write)",
                           parallelism=f"replicas x{world}"),
            "throughput": {"value": world * 1e3 / ms_max, "unit": "inferences/s"},
            "multi_gpu": {"profiling": "sharded round-robin over ranks, MIN all-reduce of costs (G1), "
                                       "rank-0 selection broadcast (G2)" if world > 1 else "single GPU",
                          "replica_outputs_identical": replicas_agree},
            "warm_l2_ms_per_step": warm_ms,
            "latency_ms_rank0": dist_ms,
            "plan_roofline": plan_roof,
            "e2e": {"value": e2e_max, "unit": "ms", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "call": "korch_execute_host (pinned host buffers; H2D copy kernel over mapped memory, plan, "
                            "output written by its kernel straight into mapped host memory; one graph replay; "
                            "weights resident)"},
            "gpu_launches": len(order) * args.steps,
            "kernels_per_step": len(order),
            "selection": {"blp_objective_ns": obj, "operator_aligned_ns": base_obj,
                          "operator_aligned_kernels": len(base), "kernels": order,
                          "operator_aligned_ms": base_ms,
                          "speedup_vs_operator_aligned": (base_ms / ms_max) if base_ms else None},
            "models": models,
            "roofline": roof,
            "bandwidth_variant": bw,
            "scaled_variant": scaled,
            "model_batch_throughput": model_scaling,
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
            "tuning": tuning,
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
