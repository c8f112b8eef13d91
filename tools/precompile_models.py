#!/usr/bin/env python
"""Ahead-of-time NVRTC compilation (sm_100a, no GPU needed) of every generable candidate
kernel of the whole-model workloads, into the in-tree model cache that bench.py --models
uses (it travels to the GPU box with the snapshot)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["KORCH_CACHE_DIR"] = os.path.join(ROOT, "paper_2406_09465_b200", "kcache_models")
os.makedirs(os.environ["KORCH_CACHE_DIR"], exist_ok=True)

import paper_2406_09465_b200 as K  # noqa: E402
from bench import MODEL_MAX_PRIMS  # noqa: E402
from korch_workloads.models import MODELS  # noqa: E402

names = sys.argv[1:] or list(MODELS)
ctx = K.Context(-1)
for n in names:
    t = time.time()
    kg = K.KorchGraph(ctx, MODELS[n]())
    kg.enumerate(partition_max=64, max_prims=MODEL_MAX_PRIMS)
    ok = kg.compile()
    print(n, sum(ok), len(ok), f"{time.time() - t:.0f}s", flush=True)
