"""Primitive-graph and orchestration-aware evaluation (test infrastructure only).

eval_primitive_graph: evaluate every primitive in float64 in topological order.
eval_orchestration:   execute a selection kernel by kernel, as the executable
  generator stitches them: kernels in the order of the topological
  index of their output (reading A6), each kernel computing its members in float64
  from its materialised inputs; only the kernel's single output is materialised,
  rounded to the storage dtype (bf16 round-to-nearest-even, or fp32) — reading A25.
  Duplicate producers of a tensor: the earliest one binds (A7).
"""
from __future__ import annotations

import numpy as np

from .primitives import eval_primitive
from .operators import kahn_order


def round_to_storage(x: np.ndarray, dtype: str) -> np.ndarray:
    """float64 -> storage dtype -> float64 (fp32: IEEE RNE; bf16: RNE of the fp32 value)."""
    if dtype == "f64":
        return np.asarray(x, dtype=np.float64)
    x32 = np.asarray(x, dtype=np.float64).astype(np.float32)
    if dtype == "f32":
        return x32.astype(np.float64)
    if dtype == "bf16":
        u = x32.view(np.uint32).astype(np.uint64)
        r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
        y = r.astype(np.uint32).view(np.float32).astype(np.float64)
        y = np.where(np.isnan(x32), np.nan, y)
        return y
    raise ValueError(dtype)


def _args(nd, env, inputs):
    return [env[r[1]] if r[0] == "node" else inputs[r[1]] for r in nd["inputs"]]


def eval_primitive_graph(pg: dict, inputs: dict, all_nodes=False):
    """inputs: {name: float64 array}. Returns {output id: array} (or every node)."""
    nodes = pg["nodes"]
    order = kahn_order(nodes, lambda nd: [r[1] for r in nd["inputs"] if r[0] == "node"])
    env = {}
    for i in order:
        nd = nodes[i]
        env[i] = eval_primitive(nd["kind"], nd["attrs"], _args(nd, env, inputs), nd["shape"])
    return env if all_nodes else {o: env[o] for o in pg["outputs"]}


def eval_orchestration(pg: dict, cands, sel, inputs: dict, topo_index, storage=None):
    """Evaluate the orchestration `sel` (indices into cands = [(members, output)])."""
    storage = storage or pg["dtype"]
    nodes = pg["nodes"]
    order = sorted(sel, key=lambda i: (topo_index[cands[i][1]], i))
    mat = {}                                   # materialised tensors (rounded)
    for k in order:
        members, out = cands[k]
        if out in mat:                         # A7: earliest producer binds
            continue
        mset = set(members)
        local = {}
        for v in sorted(members, key=lambda v: topo_index[v]):
            nd = nodes[v]
            args = []
            for r in nd["inputs"]:
                if r[0] == "input":
                    args.append(inputs[r[1]])
                elif r[1] in mset:
                    args.append(local[r[1]])
                else:
                    if r[1] not in mat:
                        raise ValueError(f"kernel {k} input p{r[1]} not materialised")
                    args.append(mat[r[1]])
            local[v] = eval_primitive(nd["kind"], nd["attrs"], args, nd["shape"])
        mat[out] = round_to_storage(local[out], storage)
    return {o: mat[o] for o in pg["outputs"]}
