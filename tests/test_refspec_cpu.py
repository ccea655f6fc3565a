"""refspec (the reference's ModelSpec front end) on the CPU: names, order, shapes, shape-composition errors,
and initial values bit-identical to the reference's build_model (nn.py:492-509) — against the golden fixtures'
``p0`` arrays (the reference's build_model at seed 3) and, when the reference tree is present, against it
directly."""
import os
import sys

import numpy as np
import pytest
import torch

from paper_2110_12484_b200 import refspec as R
from paper_2110_12484_b200.errors import ShapeCompositionError
from tests.golden_io import load_json, load_npz

MODELS = ["convbn_ce", "conv_ce", "mlp_mse", "seg_bce_dice", "bn1_tail"]


@pytest.mark.parametrize("name", MODELS)
def test_init_matches_reference_fixture(name):
    meta = load_json("e2e.json")[name]
    a = load_npz("e2e.npz")
    m = R.RefModel(meta["spec"], tuple(meta["input_shape"]))
    vals = R.init_values(m, 3)                                   # make_golden.py builds these models at seed 3
    assert list(vals) == meta["param_names"]
    assert [n for n, _ in m.named_parameters()] == meta["param_names"]
    for n in meta["param_names"]:
        assert np.array_equal(vals[n], a[f"{name}/p0/{n}"]), n   # float64, bit for bit
    assert R.spec_parameter_count(meta["spec"]) == sum(v.size for v in vals.values())
    R.load_reference_params(m, vals)
    for n, p in m.named_parameters():
        assert torch.equal(p, torch.from_numpy(vals[n]).float())  # one rounding to fp32


def test_shape_composition_errors():
    with pytest.raises(ShapeCompositionError, match="layer 0: dense expects per-sample shape"):
        R.RefModel([R.Dense(5, 3)], (4,))
    with pytest.raises(ShapeCompositionError, match="layer 1: conv2d"):
        R.RefModel([R.Conv2d(3, 4, 3), R.Conv2d(5, 4, 3)], (3, 8, 8))
    with pytest.raises(ShapeCompositionError, match="layer 1: maxpool2d kernel 9"):
        R.RefModel([R.Conv2d(3, 4, 3), R.MaxPool2d(9)], (3, 8, 8))
    with pytest.raises(ShapeCompositionError, match="layer 0"):
        R.RefModel([R.Relu()], (0, 3))
    with pytest.raises(TypeError):
        R.RefModel([{"type": "Attention"}], (3,))


def test_batchnorm_relu_fusion_and_eval_forward_cpu():
    spec = [R.Conv2d(3, 4, 3, 1, 1), R.BatchNorm(4), R.Relu(), R.MaxPool2d(2), R.Flatten(), R.Dense(64, 5)]
    m = R.RefModel(spec, (3, 8, 8))
    R.load_reference_params(m, R.init_values(m, 11))
    assert m.layer1.fuse_relu and m.layer2.fused
    m.eval()                                                     # running statistics (0, 1): eval runs anywhere
    x = torch.randn(2, 3, 8, 8)
    w = dict(m.named_parameters())
    h = torch.nn.functional.conv2d(x, w["layer0.weight"], w["layer0.bias"], 1, 1)
    h = torch.relu(h / np.sqrt(1 + 1e-5) * w["layer1.gamma"].view(1, -1, 1, 1) + w["layer1.beta"].view(1, -1, 1, 1))
    h = torch.nn.functional.max_pool2d(h, 2).reshape(2, -1)
    torch.testing.assert_close(m(x), h @ w["layer5.weight"] + w["layer5.bias"], rtol=1e-5, atol=1e-6)
    m.train()
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        m(x)


REF = "/root/reference/pkg/src"


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference tree not present (GPU box)")
def test_init_matches_reference_directly():
    sys.path.insert(0, REF)
    from mbstream import nn as RN
    spec = [RN.Conv2d(3, 8, 3, 1, 1), RN.BatchNorm(8), RN.Relu(), RN.MaxPool2d(2), RN.Flatten(),
            RN.Dense(8 * 4 * 4, 16), RN.Relu(), RN.Dense(16, 5, bias=False)]
    for seed in (0, 7):
        rp, rm = RN.build_model(spec, (3, 8, 8), seed)
        m = R.RefModel(spec, (3, 8, 8))                         # the reference's own descriptor instances
        vals = R.init_values(m, seed)
        ra = rp.arrays()
        assert list(vals) == list(ra)
        for n in ra:
            assert np.array_equal(vals[n], ra[n]), n
        assert R.spec_parameter_count(spec) == RN.spec_parameter_count(spec)
        R.load_reference_params(m, rp)                          # a reference ParameterSet loads directly
