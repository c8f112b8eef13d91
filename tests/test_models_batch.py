"""Batched model graphs (BASELINE configs C3-C5 batch sweeps) compute, image by image,
exactly what the batch-1 graphs compute: evaluated by the oracle's operator interpreter
(fp64) with the batch-1 weights (pointwise weights transposed where the batched graph
stores W^T), every image of a batch-2 run equals the batch-1 run on that image."""
import numpy as np
import pytest

from korch_workloads import make_inputs
from korch_workloads.models import candy, efficientvit, segformer, yolox_nano
from oracle.operators import eval_operator_graph

MODELS = {"candy": lambda b: candy(size=32, blocks=2, batch=b),
          "segformer": lambda b: segformer(size=64, depths=(1, 1, 1, 1), batch=b),
          "efficientvit": lambda b: efficientvit(size=64, depths=(1, 1, 1, 1, 1), batch=b),
          "yolox": lambda b: yolox_nano(size=64, batch=b)}


@pytest.mark.parametrize("name", sorted(MODELS))
def test_batch2_equals_two_batch1_runs(name):
    g1, g2 = MODELS[name](1), MODELS[name](2)
    ins_a = {k: v[0] for k, v in make_inputs(g1, seed=0).items()}
    ins_b = {k: v[0] for k, v in make_inputs(g1, seed=1).items()}
    shapes2 = {s["name"]: tuple(s["shape"]) for s in g2["inputs"]}
    ins2 = {}
    for k, v in ins_a.items():
        if k == "x":
            ins2[k] = np.concatenate([ins_a["x"], ins_b["x"]], axis=0)
        elif k + "T" in shapes2:                                # pointwise W [Cout,Cin] -> W^T
            ins2[k + "T"] = v.T
        elif v.shape == shapes2[k]:
            ins2[k] = v
        else:                                                   # bias [Cout,1] -> [Cout]
            assert v.size == int(np.prod(shapes2[k])), (k, v.shape, shapes2[k])
            ins2[k] = v.reshape(shapes2[k])
    assert set(ins2) == set(shapes2)
    ins_b = {k: (ins_b["x"] if k == "x" else v) for k, v in ins_a.items()}
    (o1a,) = eval_operator_graph(g1, ins_a).values()
    (o1b,) = eval_operator_graph(g1, ins_b).values()
    (o2,) = eval_operator_graph(g2, ins2).values()
    assert o2.shape[0] == 2 and o2.shape[1:] == o1a.shape[1:]
    np.testing.assert_allclose(o2[0], o1a[0], rtol=1e-10, atol=1e-10)
    np.testing.assert_allclose(o2[1], o1b[0], rtol=1e-10, atol=1e-10)
