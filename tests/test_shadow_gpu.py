"""bf16 shadow-weight mode: K1 accumulating bf16 gradients, K3 writing the bf16 shadow, and whole
bf16-autocast training equal to the fp32-master + autocast-cast path."""
import copy

import numpy as np
import pytest
import torch

import paper_2110_12484_b200 as mbs
from paper_2110_12484_b200 import _native as N
from tests.gpu_util import Bag, rel_l2

pytestmark = pytest.mark.gpu


def test_k1_typed_bf16_equals_fp32_of_the_same_values(cuda):
    shapes = [(64, 3, 7, 7), (64,), (128, 64, 3, 3), (10, 2048), (10,), (5, 5, 1, 1)]
    a = mbs.ParameterSet(Bag(shapes, cuda, seed=1))
    b = mbs.ParameterSet(Bag(shapes, cuda, seed=1))
    acc_a, acc_b = mbs.GradientAccumulator(a), mbs.GradientAccumulator(b)
    g = torch.Generator(device=cuda).manual_seed(2)
    acc_a.begin(3)
    acc_b.begin(3)
    for k in range(3):
        grads16 = [torch.randn(s, device=cuda, generator=g).to(torch.bfloat16) for s in shapes]
        grads16[1] = grads16[1].float()                     # mixed: some segments fp32
        acc_a.add_tensors(grads16, 0.25 + k, last=(k == 2))
        acc_b.add_tensors([t.float() for t in grads16], 0.25 + k, last=(k == 2))
    assert torch.equal(acc_a.flat, acc_b.flat)
    sa, sb = acc_a.finalize(8), acc_b.finalize(8)
    assert torch.equal(sa[0], sb[0])                        # identical grad-norm partials


@pytest.mark.parametrize("opt", ["sgd", "adam"])
def test_k3_writes_the_rounded_shadow(cuda, opt):
    net = torch.nn.Sequential(torch.nn.Conv2d(3, 16, 3), torch.nn.Flatten(), torch.nn.Linear(16 * 6 * 6, 4)).to(cuda)
    params = mbs.ParameterSet(net, shadow=torch.bfloat16)
    assert net[0].weight.dtype == torch.bfloat16 and net[0].bias.dtype == torch.float32
    assert params["0.weight"].dtype == torch.float32
    assert torch.equal(params.shadow, params.flat.to(torch.bfloat16))
    acc = mbs.GradientAccumulator(params)
    acc.begin(1)
    acc.add_tensors([torch.randn_like(params[n]) for n in params.names()], 1.0, last=True)
    acc.finalize(1)
    st = mbs.sgd_state(0.1, 0.9, 5e-4) if opt == "sgd" else mbs.adam_state(0.01, 5e-4)
    mbs.apply_update(params, acc.as_gradient_set(), st)
    assert torch.equal(params.shadow, params.flat.to(torch.bfloat16))
    assert torch.equal(net[0].weight.detach(), params["0.weight"].detach().to(torch.bfloat16))


@pytest.mark.parametrize("cfg", ["c1", "c3"])
def test_shadow_training_equals_autocast_training(cuda, cfg, monkeypatch):
    """Same native model trained for 2 mini-batches with bf16 autocast: fp32 masters cast by autocast
    vs bf16 shadows refreshed by K3 — the same bf16 weights and the same exactly-widened gradients."""
    from paper_2110_12484_b200 import graphs
    from paper_2110_12484_b200.streamer import Staging
    from paper_2110_12484_b200.workloads import WORKLOADS, build_model, synthetic_data
    w = WORKLOADS[cfg]
    torch.manual_seed(0)
    torch.backends.cudnn.deterministic = True
    base = build_model(w, ops="native").to(cuda).to(memory_format=torch.channels_last)
    n, n_mu = (32, 8) if cfg == "c1" else (6, 4)
    shape = (3, 32, 32)
    x = torch.randint(0, 256, (n,) + shape, dtype=torch.uint8, generator=torch.Generator().manual_seed(1)).to(cuda)
    if w.target == "classes":
        y = torch.randint(0, w.n_classes, (n,), generator=torch.Generator().manual_seed(2)).to(cuda)
    else:
        y = (torch.rand((n, 1) + shape[1:], generator=torch.Generator().manual_seed(2)) < 0.5).float().to(cuda)
    res = {}
    for shadow in (None, torch.bfloat16):
        graphs.clear()
        net = copy.deepcopy(base)
        params = mbs.ParameterSet(net, shadow=shadow)
        st = mbs.sgd_state(0.01, 0.9, 5e-4) if w.optimizer == "sgd" else mbs.adam_state(0.01, 5e-4)
        es = mbs.train_epoch(net, params, x, y, mini_batch_size=n // 2, micro_batch_size=n_mu,
                             normalization="exact_weighted", loss_kind=w.loss_kind, optimizer_state=st, seed=0,
                             epoch_index=0, staging=Staging(torch.bfloat16, True), autocast_dtype=torch.bfloat16)
        res[shadow] = (params.flat.detach().double().cpu().numpy(), es.mini_losses,
                       {k: v.clone() for k, v in net.state_dict().items() if "running" in k})
    torch.backends.cudnn.deterministic = False
    a, b = res[None], res[torch.bfloat16]
    assert rel_l2(b[0], a[0]) <= 1e-6, rel_l2(b[0], a[0])
    assert np.allclose(a[1], b[1], rtol=1e-4)
    for k in a[2]:
        assert torch.allclose(a[2][k], b[2][k], rtol=1e-4, atol=1e-5), k
    graphs.clear()
