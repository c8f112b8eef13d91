"""Pins for oracle/rewrites.py (R1-R3): the rewritten graph computes the same
function (fp64), has the structure Fig. 2b describes, and each rule's identity holds."""
import numpy as np

from korch_workloads import c1_softmax_layernorm, c2_vit_attention, make_inputs
from oracle.evaluate import eval_primitive_graph
from oracle.fission import fission
from oracle.operators import eval_operator_graph, softmax
from oracle.primitives import eval_primitive

RNG = np.random.default_rng(77)


def _rw(g):
    g["rewrites"] = True
    return g


def test_rewritten_attention_equals_operator_graph():
    for kw in (dict(seq=16, hidden=64, heads=4), dict(batch=2, seq=24, hidden=96, heads=3)):
        g = _rw(c2_vit_attention(**kw))
        ins = {k: v[0] for k, v in make_inputs(g, seed=4).items()}
        ref = list(eval_operator_graph(g, ins).values())[0]
        got = list(eval_primitive_graph(fission(g), ins).values())[0]
        np.testing.assert_allclose(got, ref, rtol=1e-11, atol=1e-11)


def test_rewrite_structure_fig2b():
    """Fig. 2b: the softmax reduce disappears into a MatMul with a padded operand; the
    divide moves after the MatMul (34 -> 37 primitives, one fewer reduce)."""
    plain = fission(c2_vit_attention())
    rw = fission(_rw(c2_vit_attention()))
    kinds = [n["kind"] for n in rw["nodes"]]
    assert len(plain["nodes"]) == 34 and len(rw["nodes"]) == 37
    red = lambda pg: sum(1 for n in pg["nodes"] if n["kind"] == "reduce" and n["attrs"]["op"] == "sum")
    assert red(plain) - red(rw) == 1
    assert kinds.count("pad") == 1 and kinds.count("slice") == 3 + 2
    pad = [n for n in rw["nodes"] if n["kind"] == "pad"][0]
    assert pad["attrs"]["value"] == 1.0 and pad["shape"][-1] == 64 + 16
    mm = [n for n in rw["nodes"] if n["kind"] == "matmul" and ("node", pad["id"]) in n["inputs"]][0]
    div = [n for n in rw["nodes"] if n["kind"] == "div"]
    assert len(div) == 2                       # LN's divide + the moved softmax divide
    assert any(n["id"] > mm["id"] for n in div)


def test_rules_hold_individually():
    e = RNG.standard_normal((3, 5, 7)) ** 2
    v = RNG.standard_normal((3, 7, 4))
    ones = np.ones((7, 1))
    # R1: reduce_sum(e, last) == matmul(e, ones)[..., 0]
    np.testing.assert_allclose(eval_primitive("reduce", {"axis": 2, "op": "sum"}, [e]),
                               eval_primitive("matmul", {}, [e, ones])[..., 0], rtol=1e-13)
    # R2: matmul(e / b(s), v) == matmul(e, v) / b(s)
    s = e.sum(2)
    lhs = np.matmul(e / s[..., None], v)
    rhs = np.matmul(e, v) / s[..., None]
    np.testing.assert_allclose(lhs, rhs, rtol=1e-12)
    # R3: [matmul(e, v) | matmul(e, ones)] == matmul(e, pad(v, ones))
    vh = eval_primitive("pad", {"pads": [[0, 0], [0, 0], [0, 16]], "value": 1.0}, [v])
    mm = np.matmul(e, vh)
    np.testing.assert_allclose(mm[..., :4], np.matmul(e, v), rtol=1e-13)
    np.testing.assert_allclose(mm[..., 4:], np.repeat(e.sum(2)[..., None], 16, axis=2), rtol=1e-13)
    # composition = softmax(x) @ v
    x = RNG.standard_normal((3, 5, 7))
    ex = np.exp(x)
    mm = np.matmul(ex, eval_primitive("pad", {"pads": [[0, 0], [0, 0], [0, 16]], "value": 1.0}, [v]))
    np.testing.assert_allclose(mm[..., :4] / mm[..., 4:5], np.matmul(softmax(x, 2), v), rtol=1e-12)


def test_no_site_no_change():
    """C1 has a softmax but no MatMul after it: the rewrite leaves it alone."""
    a = fission(c1_softmax_layernorm())
    b = fission(_rw(c1_softmax_layernorm()))
    assert [n["kind"] for n in a["nodes"]] == [n["kind"] for n in b["nodes"]]
