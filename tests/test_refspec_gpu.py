"""refspec on the GPU: the reference's own ModelSpec + seed -> our module (reference parameter names and
layouts, K5 batchnorm with the reference's biased running variance, K6 max-pool) -> the B200 MBS loop, checked
against the reference's own mini_batch_gradient / train_mini_batch outputs (golden fixtures, reference names
compared directly — no name mapping). Tolerances as tests/test_engine_gpu.py."""
import numpy as np
import pytest
import torch

import paper_2110_12484_b200 as mbs
from paper_2110_12484_b200 import refspec as R
from tests.golden_io import fhex, load_json, load_npz
from tests.gpu_util import rel_l2

pytestmark = pytest.mark.gpu

MODELS = ["convbn_ce", "conv_ce", "mlp_mse", "seg_bce_dice"]
GRAD_TOL = {"convbn_ce": 1e-4, "conv_ce": 1e-5, "mlp_mse": 1e-5, "seg_bce_dice": 1e-5}


@pytest.fixture(autouse=True)
def _no_tf32(monkeypatch):
    monkeypatch.setattr(torch.backends.cuda.matmul, "allow_tf32", False)
    monkeypatch.setattr(torch.backends.cudnn, "allow_tf32", False)


def _xy(a, name, meta, lo, hi, cuda):
    x = torch.from_numpy(a[f"{name}/x"][lo:hi]).float().to(cuda)
    y = torch.from_numpy(a[f"{name}/y"][lo:hi])
    y = (y if meta["loss_kind"] == "cross_entropy" else y.float()).to(cuda)
    return x, y


@pytest.mark.parametrize("name", MODELS)
@pytest.mark.parametrize("mode", ["paper_faithful", "exact_weighted"])
def test_reference_spec_gradient_and_step(cuda, name, mode):
    meta = load_json("e2e.json")[name]
    a = load_npz("e2e.npz")
    params, model = R.build_model(meta["spec"], tuple(meta["input_shape"]), 3, device=cuda)
    assert params.names() == meta["param_names"]
    for n in meta["param_names"]:                                # reference init, one fp32 rounding
        assert torch.equal(params[n].detach().cpu(), torch.from_numpy(a[f"{name}/p0/{n}"]).float()), n
    n_b = meta["n_b"]
    plan = mbs.plan_split(n_b, meta["n_mu"])
    x, y = _xy(a, name, meta, 0, n_b, cuda)
    total, stats = mbs.mini_batch_gradient(model, params, x, y, plan, mode, meta["loss_kind"])
    got = np.concatenate([total[n].detach().double().cpu().numpy().ravel() for n in meta["param_names"]])
    want = np.concatenate([a[f"{name}/{mode}/grad0/{n}"].ravel() for n in meta["param_names"]])
    assert rel_l2(got, want) <= GRAD_TOL[name]
    ms = meta["modes"][mode][0]
    assert stats.loss == pytest.approx(fhex(ms["loss"]), rel=1e-5)
    np.testing.assert_allclose(stats.losses_raw, [fhex(v) for v in ms["losses_raw"]], rtol=1e-5)

    # one optimizer step from the reference's initial weights: the reference's post-step weights
    params2, model2 = R.build_model(meta["spec"], tuple(meta["input_shape"]), 3, device=cuda)
    st = mbs.sgd_state(0.01, 0.9, 5e-4) if meta["optimizer"] == "sgd" else mbs.adam_state(0.01, 5e-4)
    mbs.train_mini_batch(model2, params2, (x, y), plan, mode, meta["loss_kind"], st)
    w = R.reference_arrays(params2)
    got = np.concatenate([w[n].ravel() for n in meta["param_names"]])
    want = np.concatenate([a[f"{name}/{mode}/p1/{n}"].ravel() for n in meta["param_names"]])
    assert rel_l2(got, want) <= 1e-5


def test_batchnorm_running_stats_use_the_biased_variance(cuda):
    """nn.py:320-327: running_var <- (1-m) running_var + m var_biased(micro-batch), per channel."""
    spec = [R.Conv2d(3, 4, 3, 1, 1), R.BatchNorm(4, momentum=0.3), R.Relu(), R.Flatten(), R.Dense(4 * 6 * 6, 2)]
    params, model = R.build_model(spec, (3, 6, 6), 5, device=cuda)
    x = torch.randn(3, 3, 6, 6, device=cuda)
    with torch.no_grad():
        h = torch.nn.functional.conv2d(x.double(), model.layer0.weight.double(), model.layer0.bias.double(), 1, 1)
    model.train()
    model(x)
    mean = h.mean(dim=(0, 2, 3))
    var_b = h.var(dim=(0, 2, 3), unbiased=False)
    torch.testing.assert_close(model.layer1.running_mean.double(), 0.3 * mean, rtol=1e-5, atol=1e-6)
    torch.testing.assert_close(model.layer1.running_var.double(), 0.7 + 0.3 * var_b, rtol=1e-5, atol=1e-6)
