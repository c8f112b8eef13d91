"""Pins for the oracle's operator and primitive interpreters and fission rules.

Each test checks the oracle against something other than itself: values the paper
fixes, closed forms, invariants, brute-force loops, or independent library routines.
"""
import json
import math
import os

import numpy as np
import pytest
from scipy import signal, stats

from korch_workloads import c1_softmax_layernorm, c2_vit_attention, make_inputs
from korch_workloads.graphs import GraphBuilder
from oracle import operators as O
from oracle.evaluate import eval_primitive_graph, round_to_storage
from oracle.fission import fission
from oracle.primitives import eval_primitive

GOLD = os.path.join(os.path.dirname(__file__), "golden")
RNG = np.random.default_rng(1234)


def test_softmax_golden_values():
    cases = json.load(open(os.path.join(GOLD, "softmax_examples.json")))["cases"]
    for c in cases:
        x = np.array(c["x"])
        if "softmax" in c:
            np.testing.assert_allclose(O.softmax(x, 0), c["softmax"], rtol=0, atol=1e-15)
        else:
            e = eval_primitive("exp", {}, [x])
            assert abs(eval_primitive("reduce", {"axis": 0, "op": "sum"}, [e]) - c["exp_sum"]) < 1e-15


def test_softmax_rows_sum_to_one_and_shift_invariance():
    x = RNG.standard_normal((7, 33)) * 5
    s = O.softmax(x, 1)
    np.testing.assert_allclose(s.sum(1), 1.0, atol=1e-12)
    assert (s > 0).all()
    # softmax(x + c) == softmax(x): a dropped/wrong-axis normaliser breaks this
    np.testing.assert_allclose(O.softmax(x + 3.0, 1), s, rtol=1e-12)
    # two-class softmax is the logistic function (closed form)
    x2 = RNG.standard_normal((50, 2))
    np.testing.assert_allclose(O.softmax(x2, 1)[:, 1], 1 / (1 + np.exp(x2[:, 0] - x2[:, 1])), rtol=1e-12)


@pytest.mark.parametrize("eps", [0.0, 1e-5, 0.3])
def test_layernorm_invariants(eps):
    x = RNG.standard_normal((9, 64)) * 2 + 1
    y = O.layernorm(x, None, None, eps)
    np.testing.assert_allclose(y.mean(-1), 0.0, atol=1e-12)
    var = x.var(-1)                                 # numpy population variance
    np.testing.assert_allclose(y.var(-1), var / (var + eps), rtol=1e-12)
    # affine: gamma scales, beta shifts
    g, b = RNG.standard_normal(64), RNG.standard_normal(64)
    np.testing.assert_allclose(O.layernorm(x, g, b, eps), y * g + b, rtol=1e-12)


def test_instancenorm_invariants_and_constant_input():
    x = RNG.standard_normal((2, 3, 5, 4))
    y = O.instancenorm(x, np.ones(3), np.zeros(3), eps=0.0)
    np.testing.assert_allclose(y.mean((2, 3)), 0, atol=1e-12)
    np.testing.assert_allclose(y.var((2, 3)), 1, rtol=1e-12)
    c = np.full((1, 2, 3, 3), 4.2)
    assert np.all(O.instancenorm(c, np.ones(2), np.zeros(2), eps=1e-5) == 0)


def test_gelu_against_normal_cdf():
    x = np.linspace(-6, 6, 101)
    np.testing.assert_allclose(O.gelu(x), x * stats.norm.cdf(x), rtol=1e-12, atol=1e-15)  # 1+erf cancels for x<0
    assert O.gelu(np.array([0.0]))[0] == 0.0


def test_matmul_brute_force():
    a, b = RNG.standard_normal((2, 3, 4)), RNG.standard_normal((4, 5))
    ref = np.zeros((2, 3, 5))
    for i in range(2):
        for m in range(3):
            for n in range(5):
                ref[i, m, n] = sum(a[i, m, k] * b[k, n] for k in range(4))
    np.testing.assert_allclose(eval_primitive("matmul", {}, [a, b]), ref, rtol=1e-13)


def test_conv2d_brute_force_and_scipy():
    x, w = RNG.standard_normal((1, 4, 6, 5)), RNG.standard_normal((6, 2, 3, 3))
    got = O.conv2d(x, w, stride=(2, 1), pads=(1, 1), groups=2)
    xp = np.pad(x, ((0, 0), (0, 0), (1, 1), (1, 1)))
    oh, ow = (6 + 2 - 3) // 2 + 1, 5
    ref = np.zeros((1, 6, oh, ow))
    for f in range(6):
        g = f // 3
        for i in range(oh):
            for j in range(ow):
                ref[0, f, i, j] = sum(xp[0, g * 2 + c, 2 * i + r, j + s] * w[f, c, r, s]
                                      for c in range(2) for r in range(3) for s in range(3))
    np.testing.assert_allclose(got, ref, rtol=1e-12)
    # single channel, stride 1: scipy's correlate2d
    x1, w1 = RNG.standard_normal((1, 1, 7, 7)), RNG.standard_normal((1, 1, 3, 3))
    np.testing.assert_allclose(O.conv2d(x1, w1, pads=(1, 1))[0, 0],
                               signal.correlate2d(x1[0, 0], w1[0, 0], mode="same"), rtol=1e-12)


def test_maxpool_brute_force():
    x = RNG.standard_normal((1, 2, 5, 5))
    got = O.maxpool(x, 3, 2, 1)
    xp = np.pad(x, ((0, 0), (0, 0), (1, 1), (1, 1)), constant_values=-np.inf)
    for c in range(2):
        for i in range(3):
            for j in range(3):
                assert got[0, c, i, j] == xp[0, c, 2 * i:2 * i + 3, 2 * j:2 * j + 3].max()


@pytest.mark.parametrize("kind,attrs,shapes", [
    ("matmul", {}, [(3, 4), (4, 5)]),
    ("matmul", {}, [(2, 3, 4), (2, 4, 5)]),
    ("conv2d", {"stride": [1, 1], "pads": [1, 1], "groups": 1}, [(1, 3, 5, 5), (4, 3, 3, 3)]),
])
def test_linear_primitives_are_linear(kind, attrs, shapes):
    """additivity and homogeneity in every input."""
    args = [RNG.standard_normal(s) for s in shapes]
    base = eval_primitive(kind, attrs, args)
    for k in range(len(args)):
        y, z, alpha = RNG.standard_normal(shapes[k]), RNG.standard_normal(shapes[k]), 1.7
        a1 = list(args); a1[k] = y
        a2 = list(args); a2[k] = z
        a3 = list(args); a3[k] = y + z
        np.testing.assert_allclose(eval_primitive(kind, attrs, a3),
                                   eval_primitive(kind, attrs, a1) + eval_primitive(kind, attrs, a2),
                                   rtol=1e-10, atol=1e-10)
        a4 = list(args); a4[k] = alpha * y
        np.testing.assert_allclose(eval_primitive(kind, attrs, a4),
                                   alpha * eval_primitive(kind, attrs, a1), rtol=1e-10, atol=1e-10)
    assert base.shape


def test_reduce_broadcast_definitions():
    x = np.array([[1.0, 2, 3], [4, 5, 6]])
    np.testing.assert_array_equal(eval_primitive("reduce", {"axis": 1, "op": "sum"}, [x]), [6, 15])
    np.testing.assert_array_equal(eval_primitive("broadcast", {"axis": 1, "size": 2}, [np.array([7.0, 9])]),
                                  [[7, 7], [9, 9]])
    y = eval_primitive("broadcast", {"axis": 0, "size": 4}, [x])
    assert y.shape == (4, 2, 3) and all((y[i] == x).all() for i in range(4))


def test_layout_primitives_are_permutations():
    x = RNG.standard_normal((3, 4, 5))
    for kind, attrs in [("transpose", {"perm": [2, 0, 1]}), ("reshape", {"shape": [12, 5]})]:
        y = eval_primitive(kind, attrs, [x])
        np.testing.assert_array_equal(np.sort(y.ravel()), np.sort(x.ravel()))
    y = eval_primitive("transpose", {"perm": [2, 0, 1]}, [x])
    assert y[4, 1, 2] == x[1, 2, 4]


def _single_op_graph(kind, in_shapes, attrs, computed_ops=0):
    b = GraphBuilder("f32")
    refs = [b.input(f"in{i}", s) for i, s in enumerate(in_shapes)]
    r = b.op(kind, *refs, **attrs)
    b.output(r)
    return b.build()


@pytest.mark.parametrize("kind,shapes,attrs", [
    ("Softmax", [(5, 17)], {"axis": 1}),
    ("Softmax", [(2, 3, 9)], {"axis": 1}),
    ("LayerNorm", [(6, 32), (32,), (32,)], {"axis": -1, "eps": 1e-5}),
    ("LayerNorm", [(6, 32)], {"axis": -1, "eps": 0.0}),
    ("InstanceNorm", [(2, 3, 4, 5), (3,), (3,)], {"eps": 1e-5}),
    ("GELU", [(4, 10)], {}),
    ("SiLU", [(4, 10)], {}),
    ("Mish", [(4, 10)], {}),
    ("Conv", [(1, 3, 6, 6), (4, 3, 3, 3), (4,)], {"stride": [1, 1], "pads": [1, 1], "groups": 1}),
    ("Upsample2x", [(1, 2, 3, 4)], {}),
])
def test_fission_equals_operator(kind, shapes, attrs):
    """Fission rules are functionally equivalent to the operator (P:221 'functionally
    equivalent primitive graph'), float64, <= 1e-12 relative."""
    g = _single_op_graph(kind, shapes, attrs)
    ins = {f"in{i}": RNG.standard_normal(s) for i, s in enumerate(shapes)}
    ref = O.eval_operator_graph(g, ins)
    pg = fission(g)
    got = eval_primitive_graph(pg, ins)
    for (oid, r), (pid, v) in zip(sorted(ref.items()), sorted(got.items())):
        assert v.shape == r.shape
        np.testing.assert_allclose(v, r, rtol=1e-12, atol=1e-12)


def test_fission_rule_shapes_match_paper():
    """Fig. 5: softmax -> exp, reduce, broadcast, div."""
    pg = fission(_single_op_graph("Softmax", [(4, 8)], {"axis": 1}))
    assert [n["kind"] for n in pg["nodes"]] == ["exp", "reduce", "broadcast", "div"]
    pg = fission(c1_softmax_layernorm())
    assert len(pg["nodes"]) == 15
    pg = fission(c2_vit_attention())
    assert len(pg["nodes"]) == 34


@pytest.mark.parametrize("builder", [c1_softmax_layernorm, lambda: c2_vit_attention(seq=16, hidden=64, heads=4)])
def test_fissioned_config_equals_operator_graph(builder):
    g = builder()
    ins = {k: v[0] for k, v in make_inputs(g, seed=0).items()}
    ref = O.eval_operator_graph(g, ins)
    got = eval_primitive_graph(fission(g), ins)
    for r, v in zip(ref.values(), got.values()):
        np.testing.assert_allclose(v, r, rtol=1e-11, atol=1e-11)


def test_fissioned_layernorm_invariant_on_c1():
    """BASELINE north star: LayerNorm outputs have mean 0 and variance 1 (eps=0, no affine);
    with eps>0 the variance is sigma^2/(sigma^2+eps) (reading A10)."""
    for eps in (0.0, 1e-5):
        g = c1_softmax_layernorm(rows=4, cols=128, affine=False, eps=eps)
        ins = {k: v[0] for k, v in make_inputs(g, seed=3).items()}
        y = list(eval_primitive_graph(fission(g), ins).values())[0]
        s = O.softmax(ins["x"], 1)
        np.testing.assert_allclose(y.mean(1), 0, atol=1e-12)
        np.testing.assert_allclose(y.var(1), s.var(1) / (s.var(1) + eps), rtol=1e-9)


def test_round_to_storage_bf16():
    # exact bf16 values survive; halfway cases round to even; ulp spacing 2^-7 near 1
    v = np.array([1.0, 1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8, -2.5, 3.0e38])
    r = round_to_storage(v, "bf16")
    assert r[0] == 1.0 and r[1] == 1.0 and r[2] == 1.0 + 2 ** -6 and r[3] == -2.5
    assert math.isfinite(r[4]) or math.isinf(r[4])
    x = RNG.standard_normal(1000)
    np.testing.assert_allclose(round_to_storage(x, "bf16"), x, rtol=2 ** -8)
