"""ctypes binding of include/korch.h — argument marshalling only.

Every step of the hot path runs inside libkorch.so (host C++) and the sm_100a
kernels it generates; nothing here computes.  If the library is missing the
import fails loudly: there is no Python or CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libkorch.so")
# in-tree cubin cache (git-ignored, travels to the GPU box with the snapshot)
CACHE_DIR = os.path.join(HERE, "kcache")
os.makedirs(CACHE_DIR, exist_ok=True)
os.environ.setdefault("KORCH_CACHE_DIR", CACHE_DIR)

KORCH_OK = 0
ERRORS = {
    -1: "KORCH_E_ARG", -2: "KORCH_E_PARSE", -3: "KORCH_E_SHAPE", -4: "KORCH_E_CYCLE",
    -5: "KORCH_E_STATE_EXPLOSION", -6: "KORCH_E_INFEASIBLE", -7: "KORCH_E_NOT_SCHEDULABLE",
    -8: "KORCH_E_NVRTC", -9: "KORCH_E_CUDA", -10: "KORCH_E_OOM", -11: "KORCH_E_UNSUPPORTED",
}
KORCH_E_NVRTC = -8
CLASS_NAMES = {0: "rejected", 1: "pw", 2: "rr", 3: "gemm"}
INT64_MAX = (1 << 63) - 1

# every symbol include/korch.h declares (checked by tests/test_abi.py)
EXPORTS = [
    "korch_version", "korch_last_error", "korch_create", "korch_destroy", "korch_graph_load",
    "korch_graph_free", "korch_graph_info", "korch_graph_dump", "korch_validate", "korch_enumerate",
    "korch_candidate", "korch_candidate_source", "korch_compile", "korch_profile",
    "korch_set_orchestration", "korch_plan", "korch_execute", "korch_variant_info", "korch_select_variant",
    "korch_variant_cost", "korch_execute_host", "korch_variant_name",
]


class KorchError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code


class EnumOpts(C.Structure):
    _fields_ = [("max_prims", C.c_int32), ("keep_multi_linear", C.c_int32), ("max_states", C.c_int64),
                ("partition_max", C.c_int32), ("attention_pairs", C.c_int32), ("max_outputs", C.c_int32)]


class CandDesc(C.Structure):
    _fields_ = [("n_members", C.c_int32), ("members", C.POINTER(C.c_int32)), ("output", C.c_int32),
                ("n_inputs", C.c_int32), ("inputs", C.POINTER(C.c_int32)),
                ("n_graph_inputs", C.c_int32), ("graph_inputs", C.POINTER(C.c_int32)),
                ("klass", C.c_int32), ("n_dense_linear", C.c_int32), ("bytes", C.c_int64),
                ("flops", C.c_double), ("signature", C.c_char_p), ("part", C.c_int32),
                ("n_extra_outputs", C.c_int32), ("extra_outputs", C.POINTER(C.c_int32))]


class ProfOpts(C.Structure):
    _fields_ = [("warmup", C.c_int32), ("launches", C.c_int32), ("trials", C.c_int32),
                ("flush_l2", C.c_int32), ("compile_threads", C.c_int32), ("tune", C.c_int32)]


def load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(LIB_PATH)
    P, I32, I64, SZ = C.c_void_p, C.c_int32, C.c_int64, C.c_size_t
    sig = {
        "korch_version": ([], C.c_char_p),
        "korch_last_error": ([], C.c_char_p),
        "korch_create": ([I32, C.POINTER(P)], I32),
        "korch_destroy": ([P], I32),
        "korch_graph_load": ([P, C.c_char_p, SZ, C.POINTER(P)], I32),
        "korch_graph_free": ([P], I32),
        "korch_graph_info": ([P, C.POINTER(I32), C.POINTER(I32), C.POINTER(I32)], I32),
        "korch_graph_dump": ([P, C.c_char_p, SZ, C.POINTER(SZ)], I32),
        "korch_validate": ([P, C.c_char_p, SZ], I32),
        "korch_enumerate": ([P, C.POINTER(EnumOpts), C.POINTER(I64), C.POINTER(I64)], I32),
        "korch_candidate": ([P, I64, C.POINTER(CandDesc)], I32),
        "korch_candidate_source": ([P, I64, C.c_char_p, SZ, C.POINTER(SZ)], I32),
        "korch_compile": ([P, C.POINTER(I64), I64, I32, C.c_char_p, C.POINTER(I32)], I32),
        "korch_profile": ([P, C.POINTER(I64), I64, C.POINTER(ProfOpts), C.POINTER(I64)], I32),
        "korch_set_orchestration": ([P, C.POINTER(I64), I64, C.POINTER(SZ)], I32),
        "korch_plan": ([P, C.POINTER(I64), C.POINTER(I64)], I32),
        "korch_execute": ([P, C.POINTER(P), C.POINTER(P), P, P], I32),
        "korch_execute_host": ([P, C.POINTER(P), C.POINTER(P), C.POINTER(P), C.POINTER(P), P, P], I32),
        "korch_variant_info": ([P, I64, C.POINTER(I32), C.POINTER(I32), C.c_char_p, SZ], I32),
        "korch_select_variant": ([P, I64, I32], I32),
        "korch_variant_cost": ([P, I64, I32, C.POINTER(I64)], I32),
        "korch_variant_name": ([P, I64, I32, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)], I32),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    return lib


LIB = load()


def check(status):
    if status != KORCH_OK:
        raise KorchError(status, LIB.korch_last_error().decode())
    return status


def i64_array(vals):
    arr = (C.c_int64 * max(1, len(vals)))(*vals)
    return arr
