"""BASELINE-size checks (C2: ResNet-50 @224, mini 1024 / micro 128) through size-independent properties.

* K1 over the real ResNet-50 parameter layout (P = 23,717,030, 161 segments,
  channels_last) for a full 8-micro mini-batch vs the float64 oracle
  accumulator (fp32 rounding only), plus linearity and the grad-norm.
* K2 + streamer: a full shuffled 1024-sample uint8 mini-batch streamed from
  pinned host memory is bit-identical to x[order[...]].to(bf16, channels_last).
* K3: one SGD step over the full flat buffer vs the oracle.
"""
import numpy as np
import pytest
import torch

import paper_2110_12484_b200 as mbs
from oracle import mbs_oracle as O
from paper_2110_12484_b200.streamer import Staging
from paper_2110_12484_b200.workloads import WORKLOADS, build_model
from tests.gpu_util import rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def r50(cuda):
    model = build_model(WORKLOADS["c2"]).to(cuda).to(memory_format=torch.channels_last)
    return model, mbs.ParameterSet(model)


def test_k1_full_resnet50_layout(cuda, r50):
    model, params = r50
    assert params.layout.n_params == 23_717_030 and len(params.layout.names) == 161
    plan = mbs.plan_split(1024, 128)
    acc = mbs.GradientAccumulator(params)
    acc.begin(plan.n_s_mu)
    oacc = np.zeros(params.layout.total)
    gen = torch.Generator(device=cuda).manual_seed(0)
    for k in range(plan.n_s_mu):
        f = mbs.normalization_factor(plan, k, "exact_weighted")
        flat = torch.randn(params.layout.total, device=cuda, generator=gen)
        grads = [params.layout.view(flat, i) for i in range(len(params.layout.names))]
        acc.add_tensors(grads, f, last=(k == plan.n_s_mu - 1))
        mask = torch.zeros_like(flat)
        for i in range(len(params.layout.names)):
            params.layout.view(mask, i).fill_(1.0)
        oacc += f * (flat * mask).double().cpu().numpy()
    st = acc.finalize(1024)
    got = acc.flat.double().cpu().numpy()
    assert rel_l2(got, oacc) <= 1e-6
    assert np.sqrt(float(st[0])) == pytest.approx(np.linalg.norm(oacc), rel=1e-6)
    # padding between segments never written
    assert float(acc.flat.abs().sum()) == pytest.approx(float(np.abs(got).sum()), rel=1e-6)


def test_k3_full_sgd_step(cuda, r50):
    model, params = r50
    w0 = params.flat.double().cpu().numpy()
    g = torch.randn(params.layout.total, device=cuda) * 1e-2
    gs = mbs.GradientSet(params.layout.views(g), flat=g, layout=params.layout)
    st = mbs.sgd_state(0.01, 0.9, 5e-4)
    mbs.apply_update(params, gs, st)
    ost = O.OptState("sgd", 0.01, 0.9, 5e-4)
    w = {"w": w0.copy()}
    O.apply_update(w, {"w": g.double().cpu().numpy()}, ost)
    assert rel_l2(params.flat.double().cpu().numpy(), w["w"]) <= 1e-7


def test_streamer_full_minibatch_bit_exact(cuda):
    w = WORKLOADS["c2"]
    n = 1536
    x = torch.randint(0, 256, (n,) + w.sample_shape, dtype=torch.uint8).pin_memory()
    y = torch.randint(0, 102, (n,), dtype=torch.int64).pin_memory()
    order = O.epoch_order(n, 0, 0)
    plan = O.plan_split(1024, 128)
    jobs = [(O.micro_batch_rows(order, 0, plan, k), 0, plan.sizes[k]) for k in range(plan.n_s_mu)]
    streamer = mbs.make_streamer(x, y, 128)
    outs = list(streamer.stream(x, y, jobs, Staging(torch.bfloat16, channels_last=True), prefetch=True))
    for (rows, _, _), (xk, yk) in zip(jobs, outs):
        ri = torch.from_numpy(rows.astype(np.int64))
        want = x[ri].to(cuda).to(torch.bfloat16).contiguous(memory_format=torch.channels_last)
        assert torch.equal(xk, want)
        assert torch.equal(yk.cpu(), y[ri])
    streamer.close()
