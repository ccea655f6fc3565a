"""Micro-batch auto-sizing on measured HBM (memory.py:88-101 rule, measured inputs)."""
import pytest
import torch

import paper_2110_12484_b200 as mbs
from paper_2110_12484_b200 import memory

pytestmark = pytest.mark.gpu


def test_measure_budget_and_fit(cuda):
    torch.manual_seed(0)
    net = torch.nn.Sequential(torch.nn.Conv2d(3, 32, 3, padding=1), torch.nn.ReLU(),
                              torch.nn.Conv2d(32, 32, 3, padding=1), torch.nn.AdaptiveAvgPool2d(1),
                              torch.nn.Flatten(), torch.nn.Linear(32, 10)).to(cuda)
    params = mbs.ParameterSet(net)

    def make_batch(n):
        return torch.randn(n, 3, 64, 64, device=cuda), torch.randint(0, 10, (n,), device=cuda)

    b = memory.measure_budget(net, make_batch, "cross_entropy", probe=(4, 8))
    # two 32-channel 64x64 fp32 activations + input are retained per sample: > 500 KB
    assert b.data_bytes_per_sample > 500_000
    n = memory.fit_micro_batch(b)
    assert n >= 1 and b.fits(n) and not b.fits(n + 1)
    # a capacity that cannot hold one sample raises like the reference
    tiny = memory.MemoryBudget(capacity_bytes=b.resident_bytes + 10, param_bytes=b.param_bytes,
                               data_bytes_per_sample=b.data_bytes_per_sample,
                               fixed_overhead_bytes=b.fixed_overhead_bytes)
    with pytest.raises(mbs.ModelDoesNotFitError):
        memory.fit_micro_batch(tiny)
    # a measured micro-batch of a few hundred samples trains without OOM
    m = min(n, 256)
    x, y = make_batch(2 * m)
    _, st = mbs.mini_batch_gradient(net, params, x, y, mbs.plan_split(2 * m, m), "exact_weighted",
                                    "cross_entropy")
    assert st.n_micro == 2 and st.grad_norm > 0
