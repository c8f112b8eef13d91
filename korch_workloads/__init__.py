"""Shared workload descriptions and seeded input generators.

This package is the ONLY code shared between the oracle (`oracle/`) and the
product path (`paper_2406_09465_b200/`).  It holds no arithmetic of the method:
it describes operator-level computation graphs (the *input* to Korch, P:121
"The input to Korch is a tensor program ... represented as a computation
graph") as JSON-able dicts, and draws seeded synthetic tensors for their
inputs (SURVEY.md §8(d) "Synthetic inputs").
"""
from .graphs import (  # noqa: F401
    c1_softmax_layernorm,
    c2_vit_attention,
    chain_graph,
    CONFIGS,
)
from .inputs import make_inputs, bf16_round_bits, bf16_bits_to_f32  # noqa: F401
