"""Tuning database: profiled candidate costs kept on disk (the paper keeps MetaSchedule's
tuning records in a database and can halt and resume tuning).

One JSON file per (graph, enumeration options): for every candidate kernel signature
(the generated kernel's name, a hash of its source: shapes, strides, program, launch
configuration) the median cost in ns of every launch variant and the fastest variant.
Records are valid only for the same code generator (korch_version() carries the
prelude/template/NVRTC salt) and the same GPU model; `apply` ignores a file recorded
under another version or device, so a stale database can never feed a selection.

This is caller-side bookkeeping (argument marshalling over korch_profile /
korch_select_variant); every measurement comes from the library's on-device profiler.
"""
from __future__ import annotations

import hashlib
import json
import os
import time

from ._lib import LIB
from .select import INF


def graph_key(graph: dict, enum_opts: dict) -> str:
    text = json.dumps(graph, sort_keys=True) + json.dumps(enum_opts, sort_keys=True)
    return hashlib.sha256(text.encode()).hexdigest()[:16]


def device_name(device: int = 0) -> str:
    try:
        import torch
        return torch.cuda.get_device_name(device)
    except Exception:
        return "unknown"


def record(kg, costs, graph: dict, enum_opts: dict, extra: dict | None = None) -> dict:
    """Database of the costs just profiled on `kg`: every launch variant of every
    generable candidate, keyed by its kernel name (korch_variant_name)."""
    kernels = {}
    for i, c in enumerate(kg.cands):
        if c["klass"] == "rejected":
            continue
        # called right after a full profile: every variant was attempted, so "not
        # timed" (-1: did not compile / failed to launch) is recorded as a failure
        for name, ns in zip(kg.variant_names(i), kg.variant_costs(i)):
            if name not in kernels:
                kernels[name] = None if ns < 0 or ns >= INF else int(ns)
    db = {"version": LIB.korch_version().decode(), "device": device_name(), "graph_key": graph_key(graph, enum_opts),
          "enum_opts": enum_opts, "created": time.strftime("%Y-%m-%d %H:%M:%S"), "kernels": kernels}
    db.update(extra or {})
    return db


def save(path: str, db: dict):
    os.makedirs(os.path.dirname(os.path.abspath(path)), exist_ok=True)
    tmp = path + ".tmp"
    with open(tmp, "w") as f:
        json.dump(db, f, separators=(",", ":"))
    os.replace(tmp, path)


def load(path: str):
    try:
        with open(path) as f:
            return json.load(f)
    except (OSError, ValueError):
        return None


def prelude_salt(version: str) -> str:
    """The part of korch_version()'s codegen salt that kernel names do NOT cover (shared
    prelude, NVRTC options and version).  Kernel names hash the generated body (and the
    GEMM template for tcgen05 kernels), so with this salt unchanged a record whose kernel
    name still occurs describes exactly the kernel that would run; kernels whose
    generator changed get new names and are simply not found (profiled live)."""
    tail = version.rsplit("codegen ", 1)[-1]
    return tail.split("-")[0]


def usable(db, graph: dict, enum_opts: dict) -> tuple[bool, str]:
    if db is None:
        return False, "no database"
    if prelude_salt(db.get("version", "")) != prelude_salt(LIB.korch_version().decode()):
        return False, f"recorded by {db.get('version')}"
    if db.get("graph_key") != graph_key(graph, enum_opts):
        return False, "different graph / enumeration options"
    if db.get("device") != device_name():
        return False, f"recorded on {db.get('device')}"
    return True, "ok"


def apply(kg, db) -> tuple[list, list]:
    """Costs from the database: a candidate's cost is its fastest recorded launch variant
    (pinned as its choice, as korch_profile would); returns (costs, indices of candidates
    with a variant the database does not cover -- the caller profiles those live)."""
    costs, missing = [], []
    rec = db["kernels"]
    for i, c in enumerate(kg.cands):
        if c["klass"] == "rejected":
            costs.append(INF)
            continue
        names = kg.variant_names(i)
        if any(n not in rec for n in names):
            costs.append(INF)
            missing.append(i)
            continue
        ns = [INF if rec[n] is None else rec[n] for n in names]
        v = min(range(len(ns)), key=lambda k: (ns[k], k))
        costs.append(ns[v])
        if ns[v] < INF:
            kg.set_variant(i, v)
    return costs, missing
