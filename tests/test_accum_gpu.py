"""K1 (fused normalise + accumulate + grad norm) vs the fp64 oracle accumulator (engine.py:100-131)."""
import numpy as np
import pytest
import torch

import paper_2110_12484_b200 as mbs
from oracle import mbs_oracle as O
from tests.gpu_util import Bag, rel_l2, to64

pytestmark = pytest.mark.gpu

SHAPES = [(64, 3, 7, 7), (64,), (1,), (3,), (8193,), (257, 129), (5, 5, 3, 3), (100000,), (2048, 1000), (7,)]


def _setup(cuda, shapes=SHAPES, channels_last=False):
    bag = Bag(shapes, cuda, channels_last_4d=channels_last)
    params = mbs.ParameterSet(bag)
    return bag, params


@pytest.mark.parametrize("mode", ["paper_faithful", "exact_weighted", "off"])
@pytest.mark.parametrize("n_b,n_mu", [(10, 4), (16, 8), (7, 7), (256, 48)])
def test_accumulate_matches_oracle(cuda, mode, n_b, n_mu):
    bag, params = _setup(cuda)
    acc = mbs.GradientAccumulator(params)
    plan = mbs.plan_split(n_b, n_mu)
    oplan = O.plan_split(n_b, n_mu)
    oacc = O.Accumulator({n: tuple(s) for n, s in zip(params.names(), params.layout.shapes)})
    acc.begin(plan.n_s_mu)
    oacc.begin(plan.n_s_mu)
    g = torch.Generator(device=cuda).manual_seed(n_b * 31 + n_mu)
    losses = []
    for k in range(plan.n_s_mu):
        f = mbs.normalization_factor(plan, k, mode)
        assert f == O.normalization_factor(oplan, k, mode)
        grads = [torch.randn(s, device=cuda, generator=g) for s in params.layout.shapes]
        loss = torch.rand((), device=cuda, generator=g)
        losses.append(float(loss))
        acc.add_tensors(grads, f, loss=loss, loss_weight=plan.sizes[k], last=(k == plan.n_s_mu - 1))
        oacc.add({n: f * to64(t) for n, t in zip(params.names(), grads)})
    stats = acc.finalize(plan.n_b)
    sums = acc.sums
    for n in params.names():
        assert rel_l2(to64(sums[n]), oacc.sums[n]) <= 1e-6, n
    flat_ref = np.concatenate([oacc.sums[n].ravel() for n in params.names()])
    assert rel_l2(to64(torch.cat([sums[n].reshape(-1) for n in params.names()])), flat_ref) <= 1e-6
    norm2 = float(stats[0])
    assert np.sqrt(norm2) == pytest.approx(O.l2_norm(oacc.sums), rel=1e-6)
    assert float(stats[1]) == pytest.approx(O.mini_loss(oplan.sizes, losses, n_b), rel=1e-12)
    assert float(stats[3]) == plan.n_s_mu
    assert acc.micro_batches_seen == plan.n_s_mu


def test_unit_factor_is_bit_exact(cuda):
    bag, params = _setup(cuda)
    acc = mbs.GradientAccumulator(params)
    acc.begin(3)
    gs = [[torch.randn(s, device=cuda) for s in params.layout.shapes] for _ in range(3)]
    for grads in gs:
        acc.add(dict(zip(params.names(), grads)))
    for i, n in enumerate(params.names()):
        want = (gs[0][i] + gs[1][i]) + gs[2][i]   # sequential plan order, fp32
        assert torch.equal(acc.sums[n], want), n


def test_unaligned_and_strided_gradients(cuda):
    bag, params = _setup(cuda, channels_last=True)
    acc = mbs.GradientAccumulator(params)
    acc.begin(2)
    grads1, grads2 = [], []
    for s, st in zip(params.layout.shapes, params.layout.strides):
        base = torch.randn(int(np.prod(s)) + 1, device=cuda)
        grads1.append(base[1:].as_strided(s, st))            # 4-byte aligned only -> scalar path
        grads2.append(torch.randn(s, device=cuda))           # NCHW contiguous vs channels_last param
    acc.add_tensors(grads1, 0.5)
    acc.add_tensors(grads2, 2.0)
    for i, n in enumerate(params.names()):
        want = to64(grads1[i]) * 0.5 + to64(grads2[i]) * 2.0
        assert rel_l2(to64(acc.sums[n]), want) <= 1e-6, n


def test_bucketed_equals_single_call(cuda):
    bag, params = _setup(cuda)
    n = len(params.names())
    a1, a2 = mbs.GradientAccumulator(params), mbs.GradientAccumulator(params)
    a1.begin(2)
    a2.begin(2)
    for k in range(2):
        grads = [torch.randn(s, device=cuda) for s in params.layout.shapes]
        a1.add_tensors(grads, 0.25, last=k == 1)
        # buckets issued in reverse (backward) order
        for lo, hi in [(7, n), (3, 7), (0, 3)]:
            a2.add_tensors(grads[lo:hi], 0.25, seg_begin=lo, last=k == 1)
    assert a1.micro_batches_seen == a2.micro_batches_seen == 2
    assert torch.equal(a1.flat, a2.flat)
    s1, s2 = a1.finalize(8), a2.finalize(8)
    # fused per-tile partials vs the post-hoc norm pass: same value, different summation grouping
    assert float(s1[0]) == pytest.approx(float(s2[0]), rel=1e-12)
    # run to run the same path is bit-reproducible (fixed-order reduction, no atomics)
    a3 = mbs.GradientAccumulator(params)
    a3.begin(2)
    a3.add_tensors(grads, 0.25)
    a3.add_tensors(grads, 0.25, last=True)
    a4 = mbs.GradientAccumulator(params)
    a4.begin(2)
    a4.add_tensors(grads, 0.25)
    a4.add_tensors(grads, 0.25, last=True)
    assert float(a3.finalize(8)[0]) == float(a4.finalize(8)[0])


def test_overflow_and_key_errors(cuda):
    bag, params = _setup(cuda)
    acc = mbs.GradientAccumulator(params)
    acc.begin(2)
    grads = {n: torch.randn(s, device=cuda) for n, s in zip(params.names(), params.layout.shapes)}
    acc.add(grads)
    acc.add(grads)
    with pytest.raises(mbs.AccumulatorOverflowError):      # engine.py:118-121
        acc.add(grads)
    acc.begin(2)
    bad = dict(grads)
    bad.pop(params.names()[0])
    with pytest.raises(mbs.AccumulatorOverflowError):      # engine.py:122-125 (key mismatch)
        acc.add(bad)
    bad = dict(grads)
    bad[params.names()[1]] = torch.randn(65, device=cuda)
    with pytest.raises(mbs.GradientKeyMismatchError):
        acc.add(bad)


def test_begin_zeroes_and_gradient_set_aliases(cuda):
    bag, params = _setup(cuda)
    acc = mbs.GradientAccumulator(params)
    acc.begin(1)
    grads = {n: torch.randn(s, device=cuda) for n, s in zip(params.names(), params.layout.shapes)}
    acc.add(grads)
    total = acc.as_gradient_set()
    assert torch.equal(total[params.names()[0]], grads[params.names()[0]])
    acc.begin(1)
    for n in params.names():          # as_gradient_set aliases the live sums
        assert float(acc.sums[n].abs().sum()) == 0.0
        assert float(total[n].abs().sum()) == 0.0


def test_nonfinite_is_flagged(cuda):
    bag, params = _setup(cuda)
    acc = mbs.GradientAccumulator(params)
    acc.begin(1)
    grads = [torch.randn(s, device=cuda) for s in params.layout.shapes]
    grads[4][17] = float("nan")
    acc.add_tensors(grads, 1.0, last=True)
    st = acc.finalize(4)
    assert float(st[2]) == 1.0


def test_size1_dim_strides_are_not_copied(cuda):
    """1x1 conv weights in channels_last: autograd's grad strides differ only on size-1 dims."""
    conv = torch.nn.Conv2d(64, 256, 1).to(cuda).to(memory_format=torch.channels_last)
    params = mbs.ParameterSet(conv)
    acc = mbs.GradientAccumulator(params)
    w = params.names()[0]
    g = torch.randn(256, 64, 1, 1, device=cuda)               # strides (64, 1, 1, 1)
    assert g.stride() != params.layout.strides[0]
    assert acc._same_memory_order(g, 0)
    assert acc._conform(g, 0) is g
    acc.begin(1)
    acc.add({w: g, params.names()[1]: torch.ones(256, device=cuda)})
    assert torch.equal(acc.sums[w], g)
    assert not acc._same_memory_order(torch.randn(256, 64, 1, 1, device=cuda).transpose(0, 1).reshape(
        256, 64, 1, 1)[:, :, :, :].as_strided((256, 64, 1, 1), (1, 256, 1, 1)), 0)


def test_gradient_set_norm_is_never_stale(cuda):
    """The device norm is attached to as_gradient_set() only when finalize() reduced it for the current
    sums; a later reference-style begin/add (engine.py:110-131) gets a freshly computed l2_norm."""
    bag, params = _setup(cuda)
    acc = mbs.GradientAccumulator(params)
    acc.begin(1)
    g1 = [torch.randn(s, device=cuda) for s in params.layout.shapes]
    acc.add_tensors(g1, 1.0, loss=torch.ones((), device=cuda), loss_weight=1.0, last=True)
    acc.finalize(1)
    gs = acc.as_gradient_set()
    assert gs.norm2 is not None
    want1 = float(torch.sqrt(sum((t.double() ** 2).sum() for t in g1)))
    assert gs.l2_norm() == pytest.approx(want1, rel=1e-6)
    acc.begin(1)
    g2 = {n: 3.0 * torch.randn(s, device=cuda) for n, s in zip(params.names(), params.layout.shapes)}
    acc.add(g2)
    gs2 = acc.as_gradient_set()
    assert gs2.norm2 is None
    want2 = float(torch.sqrt(sum((t.double() ** 2).sum() for t in g2.values())))
    assert gs2.l2_norm() == pytest.approx(want2, rel=1e-6)
