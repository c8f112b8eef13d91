"""Seeded synthetic inputs (SURVEY.md §8(d) "Synthetic inputs").

Every graph input is drawn, in the order the graph lists them, from one
numpy Generator(PCG64(seed)) as N(mean, std) (or all-ones).  bf16 inputs are
produced by round-to-nearest-even from the fp32 draw, so the GPU and the
oracle receive identical bits.  No arithmetic of the method lives here.
"""
from __future__ import annotations

import numpy as np


def bf16_round_bits(x32: np.ndarray) -> np.ndarray:
    """fp32 array -> uint16 bf16 bit patterns, round-to-nearest-even (NaN kept quiet)."""
    u = np.ascontiguousarray(x32, dtype=np.float32).view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    r = ((u + 0x7FFF + lsb) >> 16).astype(np.uint16)
    nan = np.isnan(x32)
    if nan.any():
        r = r.copy()
        r[nan] = 0x7FC0
    return r


def bf16_bits_to_f32(b16: np.ndarray) -> np.ndarray:
    return (b16.astype(np.uint32) << 16).view(np.float32)


def make_inputs(graph: dict, seed: int = 0):
    """Return {name: (values_f64, storage_array)} for every graph input.

    values_f64 is the exact value of the stored element in float64; the
    storage array is float32 for "f32" and uint16 bf16 bits for "bf16".
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    out = {}
    for spec in graph["inputs"]:
        shape = tuple(spec["shape"])
        init = spec.get("init", {"dist": "normal", "mean": 0.0, "std": 1.0})
        if init["dist"] == "ones":
            v32 = np.ones(shape, dtype=np.float32)
        elif init["dist"] == "normal":
            v32 = (rng.standard_normal(shape) * init.get("std", 1.0)
                   + init.get("mean", 0.0)).astype(np.float32)
        else:
            raise ValueError(f"unknown init {init}")
        if spec["dtype"] == "bf16":
            bits = bf16_round_bits(v32)
            out[spec["name"]] = (bf16_bits_to_f32(bits).astype(np.float64), bits)
        elif spec["dtype"] == "f32":
            out[spec["name"]] = (v32.astype(np.float64), v32)
        else:
            raise ValueError(f"unknown dtype {spec['dtype']}")
    return out
