"""korch-b200: B200-native kernel-orchestrated primitive-graph executor (Korch, arXiv 2406.09465).

The hot path lives in libkorch.so (C ABI in include/korch.h) and the sm_100a
kernels it generates; this package is the thin Python binding plus the
host-side BLP selection.
"""
from .api import Context, KorchGraph, torch_inputs  # noqa: F401
from .select import INF, operator_aligned, singletons, solve_blp  # noqa: F401
