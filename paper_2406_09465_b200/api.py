"""Python front end of the C ABI (argument marshalling + the host-side BLP).

    ctx = Context(0)
    kg  = KorchGraph(ctx, graph_dict)          # korch_graph_load (fission inside)
    kg.enumerate()                              # Alg. 1 + templates
    costs = kg.profile()                        # on-device PROFILING, ns
    sel = kg.select(costs)                      # Eq. 2-4 BLP (HiGHS)
    kg.set_orchestration(sel)                   # Eq. 3/4 check, buffer plan
    kg.execute(inputs, outputs, workspace, stream)   # CUDA-graph replay

Device buffers are torch tensors (PyTorch is used for memory, streams and
process groups only).
"""
from __future__ import annotations

import ctypes as C
import json
import os

from . import _lib
from ._lib import LIB, check
from .select import INF, operator_aligned, singletons, solve_blp, solve_partitioned

DTYPE_BYTES = {"f32": 4, "bf16": 2}


class Context:
    def __init__(self, device: int = 0):
        self.h = C.c_void_p()
        check(LIB.korch_create(int(device), C.byref(self.h)))
        self.device = device

    def close(self):
        if self.h:
            LIB.korch_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


class KorchGraph:
    def __init__(self, ctx: Context, graph):
        self.ctx = ctx
        text = graph if isinstance(graph, str) else json.dumps(graph)
        b = text.encode()
        self.h = C.c_void_p()
        check(LIB.korch_graph_load(ctx.h, b, len(b), C.byref(self.h)))
        self.cands = None
        self.n_states = None
        self.prim = self.dump()
        self.inputs = self.prim["inputs"]
        self.outputs = self.prim["outputs"]
        self.workspace_bytes = None

    def __del__(self):  # pragma: no cover
        try:
            if self.h:
                LIB.korch_graph_free(self.h)
        except Exception:
            pass

    # ---------------------------------------------------------------- graph
    def dump(self) -> dict:
        need = C.c_size_t()
        LIB.korch_graph_dump(self.h, None, 0, C.byref(need))
        buf = C.create_string_buffer(need.value)
        check(LIB.korch_graph_dump(self.h, buf, need.value, C.byref(need)))
        return json.loads(buf.value.decode())

    def validate(self) -> str:
        buf = C.create_string_buffer(1 << 16)
        check(LIB.korch_validate(self.h, buf, len(buf)))
        return buf.value.decode()

    @property
    def n_prims(self):
        return len(self.prim["nodes"])

    def output_shape(self, k=0):
        return tuple(self.prim["nodes"][self.outputs[k]]["shape"])

    # ---------------------------------------------------------------- candidates
    def enumerate(self, max_prims: int = 16, keep_multi_linear: bool = False, max_states: int = 1_000_000,
                  partition_max: int = 0, attention_pairs: bool = False, max_outputs: int = 1):
        o = _lib.EnumOpts(max_prims, int(keep_multi_linear), max_states, partition_max, int(attention_pairs),
                          int(max_outputs))
        nc, ns = C.c_int64(), C.c_int64()
        check(LIB.korch_enumerate(self.h, C.byref(o), C.byref(nc), C.byref(ns)))
        self.n_states = ns.value
        self.cands = [self.candidate(i) for i in range(nc.value)]
        topo = self.topo_index()
        for c in self.cands:
            c["sink_topo"] = topo[c["output"]]   # the kernel's place in the schedule (A6)
        return self.cands

    def topo_index(self):
        """Position of every primitive in the library's topological order (Kahn, smallest
        id first; the order kernels run in, reading A6)."""
        import heapq
        nodes = self.prim["nodes"]
        preds = [sorted({r["node"] for r in nd["inputs"] if "node" in r}) for nd in nodes]
        succ = [[] for _ in nodes]
        for v, ps in enumerate(preds):
            for u in ps:
                succ[u].append(v)
        indeg = [len(p) for p in preds]
        ready = [v for v in range(len(nodes)) if not indeg[v]]
        heapq.heapify(ready)
        pos = [0] * len(nodes)
        k = 0
        while ready:
            v = heapq.heappop(ready)
            pos[v] = k
            k += 1
            for w in succ[v]:
                indeg[w] -= 1
                if not indeg[w]:
                    heapq.heappush(ready, w)
        return pos

    def candidate(self, i: int) -> dict:
        d = _lib.CandDesc()
        check(LIB.korch_candidate(self.h, i, C.byref(d)))
        return {
            "index": i,
            "members": [d.members[k] for k in range(d.n_members)],
            "output": d.output,
            "extra_outputs": [d.extra_outputs[k] for k in range(d.n_extra_outputs)],
            "inputs": [d.inputs[k] for k in range(d.n_inputs)],
            "graph_inputs": [d.graph_inputs[k] for k in range(d.n_graph_inputs)],
            "klass": _lib.CLASS_NAMES[d.klass],
            "n_dense_linear": d.n_dense_linear,
            "bytes": d.bytes,
            "flops": d.flops,
            "signature": d.signature.decode(),
            "part": d.part,
        }

    def source(self, i: int) -> str:
        need = C.c_size_t()
        LIB.korch_candidate_source(self.h, i, None, 0, C.byref(need))
        buf = C.create_string_buffer(max(1, need.value))
        check(LIB.korch_candidate_source(self.h, i, buf, len(buf), C.byref(need)))
        return buf.value.decode()

    def kernel_name(self, i: int) -> str:
        """Name of the chosen (else first) launch variant's kernel of candidate i (the name
        ncu reports)."""
        import re
        _, ch, _ = self.variant_info(i)
        names = re.findall(r"__global__ void __launch_bounds__\([^)]*\) (korch_\w+)\(", self.source(i))
        return names[max(ch, 0)] if names else ""

    def generable(self):
        return [c["index"] for c in self.cands if c["klass"] != "rejected"]

    # ---------------------------------------------------------------- compile / profile
    def compile(self, idx=None, threads: int = 0, cache_dir: str | None = None):
        idx = self.generable() if idx is None else list(idx)
        arr = _lib.i64_array(idx)
        ok = (C.c_int32 * max(1, len(idx)))()
        cd = cache_dir.encode() if cache_dir else None
        st = LIB.korch_compile(self.h, arr, len(idx), threads, cd, ok)
        flags = [ok[k] for k in range(len(idx))]
        if st == _lib.KORCH_E_NVRTC:
            # candidates with no compiled variant are "cannot be generated": the
            # profiler gives them cost INF; the failures are kept for inspection
            self.compile_failures = [(i, LIB.korch_last_error().decode()) for i, f in zip(idx, flags) if not f]
        else:
            check(st)
            self.compile_failures = []
        return flags

    def profile(self, idx=None, warmup=3, launches=20, trials=5, flush_l2=False, tune=True,
                compile_threads=0):
        """PROFILING: median per-launch ns per candidate; INF if not generable."""
        allidx = list(range(len(self.cands))) if idx is None else list(idx)
        arr = _lib.i64_array(allidx)
        out = (C.c_int64 * max(1, len(allidx)))()
        o = _lib.ProfOpts(warmup, launches, trials, int(flush_l2), compile_threads, 0 if tune else -1)
        check(LIB.korch_profile(self.h, arr, len(allidx), C.byref(o), out))
        costs = [out[k] for k in range(len(allidx))]
        if idx is None:
            self.costs = costs
        return costs

    # ---------------------------------------------------------------- orchestration
    def select(self, costs=None, time_limit=600.0):
        """Eq. 2-4 optimum (per partition part when the graph was partitioned)."""
        costs = self.costs if costs is None else costs
        return solve_partitioned(self.cands, costs, self.outputs, time_limit=time_limit)

    def operator_aligned(self):
        return operator_aligned(self.cands, self.prim)

    def singletons(self):
        return singletons(self.cands, self.n_prims)

    def variant_info(self, i: int):
        """(number of launch variants, chosen variant or -1, tag of the chosen/first one)."""
        nv, ch = C.c_int32(), C.c_int32()
        buf = C.create_string_buffer(512)
        check(LIB.korch_variant_info(self.h, i, C.byref(nv), C.byref(ch), buf, len(buf)))
        return nv.value, ch.value, buf.value.decode()

    def variant_costs(self, i: int):
        """[(tag, ns)] for every launch variant of candidate i (ns = -1 if not profiled)."""
        nv, _, _ = self.variant_info(i)
        out = []
        for v in range(nv):
            ns = C.c_int64()
            check(LIB.korch_variant_cost(self.h, i, v, C.byref(ns)))
            out.append(ns.value)
        return out

    def variant_names(self, i: int):
        """Kernel names of every launch variant of candidate i (tuning-database keys)."""
        nv, _, _ = self.variant_info(i)
        buf = C.create_string_buffer(128)
        need = C.c_size_t()
        out = []
        for v in range(nv):
            check(LIB.korch_variant_name(self.h, i, v, buf, len(buf), C.byref(need)))
            out.append(buf.value.decode())
        return out

    def set_variant(self, i: int, v: int):
        check(LIB.korch_select_variant(self.h, i, v))

    def set_orchestration(self, sel, variants=None) -> int:
        """Accept selection `sel`; `variants` ({cand: variant}) pins launch variants."""
        for i, v in (variants or {}).items():
            self.set_variant(int(i), int(v))
        arr = _lib.i64_array(list(sel))
        ws = C.c_size_t()
        check(LIB.korch_set_orchestration(self.h, arr, len(sel), C.byref(ws)))
        self.workspace_bytes = ws.value
        return ws.value

    def plan(self):
        n = C.c_int64()
        check(LIB.korch_plan(self.h, C.byref(n), None))
        arr = (C.c_int64 * max(1, n.value))()
        check(LIB.korch_plan(self.h, C.byref(n), arr))
        return [arr[k] for k in range(n.value)]

    # ---------------------------------------------------------------- execution
    def execute(self, inputs, outputs, workspace, stream=None):
        """inputs/outputs: sequences of device pointers (int) or torch tensors."""
        def ptr(t):
            return t if isinstance(t, int) else t.data_ptr()
        n_in, n_out = len(self.inputs), len(self.outputs)
        if len(inputs) != n_in or len(outputs) != n_out:
            raise ValueError("wrong number of inputs/outputs")
        ia = (C.c_void_p * max(1, n_in))(*[ptr(t) for t in inputs])
        oa = (C.c_void_p * max(1, n_out))(*[ptr(t) for t in outputs])
        ws = ptr(workspace) if workspace is not None else 0
        s = stream if isinstance(stream, int) or stream is None else stream.cuda_stream
        check(LIB.korch_execute(self.h, ia, oa, C.c_void_p(ws), C.c_void_p(s or 0)))

    def execute_host(self, host_inputs, dev_inputs, host_outputs, dev_outputs, workspace, stream=None):
        """End-to-end call (korch_execute_host): host_inputs[i] (pinned tensor / pointer, or
        None = already resident on the device) are copied into dev_inputs[i], the plan runs,
        and dev_outputs[j] are copied back into host_outputs[j] (None = not copied); one
        CUDA-graph replay on `stream`."""
        def ptr(t):
            return 0 if t is None else t if isinstance(t, int) else t.data_ptr()
        n_in, n_out = len(self.inputs), len(self.outputs)
        if not (len(host_inputs) == len(dev_inputs) == n_in and len(host_outputs) == len(dev_outputs) == n_out):
            raise ValueError("wrong number of inputs/outputs")
        arr = lambda xs, n: (C.c_void_p * max(1, n))(*[ptr(t) for t in xs])  # noqa: E731
        ws = ptr(workspace) if workspace is not None else 0
        s = stream if isinstance(stream, int) or stream is None else stream.cuda_stream
        check(LIB.korch_execute_host(self.h, arr(host_inputs, n_in), arr(dev_inputs, n_in), arr(host_outputs, n_out),
                                     arr(dev_outputs, n_out), C.c_void_p(ws), C.c_void_p(s or 0)))

    # helpers for torch-resident buffers
    def torch_outputs(self, device="cuda"):
        import torch
        dt = {"f32": torch.float32, "bf16": torch.bfloat16}[self.prim["dtype"]]
        return [torch.empty(self.prim["nodes"][o]["shape"], dtype=dt, device=device) for o in self.outputs]

    def torch_workspace(self, device="cuda"):
        import torch
        return torch.empty(max(256, self.workspace_bytes or 0), dtype=torch.uint8, device=device)


def torch_inputs(graph: dict, arrays: dict, device="cuda"):
    """Move seeded storage arrays (float32 or uint16 bf16 bits) to the device, in graph order."""
    import numpy as np
    import torch
    out = []
    for spec in graph["inputs"]:
        a = arrays[spec["name"]]
        if spec["dtype"] == "bf16":
            t = torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).view(torch.bfloat16)
        else:
            t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32))
        out.append(t.to(device))
    return out
