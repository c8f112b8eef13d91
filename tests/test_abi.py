"""The C-ABI library loads and exports every symbol include/korch.h declares; host-only
contexts load graphs, enumerate, generate and compile (no GPU compute)."""
import ctypes
import json
import os
import re

import pytest

from korch_workloads import c1_softmax_layernorm, c2_vit_attention

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    text = open(os.path.join(ROOT, "include", "korch.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(korch_[a-z_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2406_09465_b200 import _lib
    lib = ctypes.CDLL(_lib.LIB_PATH)
    declared = _header_functions()
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(lib, name), f"{name} declared in korch.h but not exported"
    assert sorted(_lib.EXPORTS) == declared


def test_version_and_error_strings():
    from paper_2406_09465_b200._lib import LIB
    assert b"sm_100a" in LIB.korch_version()
    assert LIB.korch_last_error() is not None


def test_host_only_context_and_errors():
    from paper_2406_09465_b200 import Context, KorchGraph
    from paper_2406_09465_b200._lib import KorchError
    ctx = Context(-1)
    kg = KorchGraph(ctx, c1_softmax_layernorm())
    assert kg.n_prims == 15
    assert kg.validate() == "ok"
    with pytest.raises(KorchError, match="KORCH_E_PARSE"):
        KorchGraph(ctx, "{not json")
    bad = c1_softmax_layernorm()
    bad["nodes"][0]["kind"] = "FFT"
    with pytest.raises(KorchError, match="KORCH_E_UNSUPPORTED"):
        KorchGraph(ctx, bad)
    cyc = c1_softmax_layernorm()
    cyc["nodes"][0]["inputs"] = [{"node": 1}]
    with pytest.raises(KorchError, match="KORCH_E_CYCLE"):
        KorchGraph(ctx, cyc)
    shp = c1_softmax_layernorm()
    shp["inputs"][1]["shape"] = [7]
    with pytest.raises(KorchError, match="KORCH_E_SHAPE"):
        KorchGraph(ctx, shp)
    kg.enumerate()
    with pytest.raises(KorchError, match="KORCH_E_CUDA"):
        kg.profile([0])
    # execute before an accepted orchestration
    with pytest.raises(KorchError, match="KORCH_E_ARG"):
        kg.execute([0, 0, 0], [0], 0)


def test_set_orchestration_checks_eq3_eq4():
    from paper_2406_09465_b200 import Context, KorchGraph
    from paper_2406_09465_b200._lib import KorchError
    ctx = Context(-1)
    kg = KorchGraph(ctx, c1_softmax_layernorm())
    cands = kg.enumerate()
    out = kg.outputs[0]
    last = [c["index"] for c in cands if c["output"] == out and len(c["members"]) == 1][0]
    with pytest.raises(KorchError, match="KORCH_E_INFEASIBLE"):
        kg.set_orchestration([last])             # inputs of the last kernel never produced (Eq. 4)
    with pytest.raises(KorchError, match="KORCH_E_INFEASIBLE"):
        kg.set_orchestration([0])                # output not produced (Eq. 3)
    whole = [c["index"] for c in cands if len(c["members"]) == 15][0]
    ws = kg.set_orchestration([whole])
    assert ws == 0 and kg.plan() == [whole]
    ws = kg.set_orchestration(kg.singletons())
    assert ws > 0 and len(kg.plan()) == 15


def test_host_only_compile_c1():
    """NVRTC cross-compiles every C1 candidate for sm_100a without a GPU."""
    from paper_2406_09465_b200 import Context, KorchGraph
    ctx = Context(-1)
    kg = KorchGraph(ctx, c1_softmax_layernorm())
    cands = kg.enumerate()
    ok = kg.compile(threads=8)
    assert all(ok) and len(ok) == len(cands)
    src = kg.source(cands[-1]["index"])
    assert "__global__" in src and "__shfl_xor_sync" in src
