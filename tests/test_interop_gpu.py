"""ReferenceAccumulator: the reference's ``accumulator=`` seam (engine.py:186,201-220) served by K1 in HBM."""
from dataclasses import dataclass, field

import numpy as np
import pytest
import torch

import paper_2110_12484_b200 as mbs
from oracle import mbs_oracle as O
from oracle.hybrid import TorchGradFn
from paper_2110_12484_b200.interop import ReferenceAccumulator
from tests.golden_io import fhex, load_json, load_npz
from tests.gpu_util import rel_l2

pytestmark = pytest.mark.gpu


@dataclass
class GradientSet:                 # the reference's container shape (tensor.py:99-124): arrays + items()
    arrays: dict = field(default_factory=dict)

    def items(self):
        return self.arrays.items()

    def keys(self):
        return self.arrays.keys()


@dataclass
class _T:                          # the reference's Tensor as ParameterSet.items() yields it
    data: np.ndarray
    grad_required: bool = True

    @property
    def shape(self):
        return self.data.shape


def test_reference_call_sequence_against_the_reference_fixture(cuda):
    meta = load_json("accum_optim.json")
    a = load_npz("accum_optim.npz")
    names = list(meta["shapes"])
    params = {n: _T(a[f"p0/{n}"]) for n in names}
    acc = ReferenceAccumulator(params)
    for _ in range(2):                                          # begin() resets between mini-batches
        acc.begin(meta["n_micro"])                              # engine.py:202
        for k in range(meta["n_micro"]):
            mbs.accumulate(acc, GradientSet({n: a[f"g{k}/{n}"] for n in names}))   # engine.py:216
        assert acc.micro_batches_seen == meta["n_micro"]
        total = acc.as_gradient_set()                           # engine.py:220
        assert isinstance(total, GradientSet)
        got = np.concatenate([total.arrays[n].ravel() for n in names])
        want = np.concatenate([a[f"total/{n}"].ravel() for n in names])
        assert rel_l2(got, want) <= 1e-6
        assert np.sqrt(np.dot(got, got)) == pytest.approx(fhex(meta["norm"]), rel=1e-6)
    with pytest.raises(mbs.AccumulatorOverflowError):           # past `expected` (engine.py:118-121)
        acc.add(GradientSet({n: a[f"g0/{n}"] for n in names}))
    acc.begin(3)
    with pytest.raises(mbs.AccumulatorOverflowError):           # key-set mismatch (engine.py:122-125)
        acc.add(GradientSet({n: a[f"g0/{n}"] for n in names[:-1]}))
    with pytest.raises(mbs.GradientKeyMismatchError):
        acc.add(GradientSet({n: np.zeros(3) if n == names[0] else a[f"g0/{n}"] for n in names}))


def test_plugs_into_a_reference_structured_loop(cuda):
    """The oracle's mini_batch_gradient (the reference's loop, engine.py:179-230, over a float64 torch-CPU
    model) with the accumulator swapped for ReferenceAccumulator: same gradient, same statistics."""
    torch.manual_seed(0)
    net = torch.nn.Sequential(torch.nn.Conv2d(3, 6, 3, padding=1), torch.nn.ReLU(), torch.nn.Flatten(),
                              torch.nn.Linear(6 * 8 * 8, 5))
    gf = TorchGradFn(net, "cross_entropy")
    shapes = {n: v.shape for n, v in gf.params().items()}
    g = torch.Generator().manual_seed(3)
    x = torch.randn(10, 3, 8, 8, generator=g).double().numpy()
    y = torch.randint(0, 5, (10,), generator=g).numpy()
    plan = O.plan_split(10, 4)
    want, st_want = O.mini_batch_gradient(gf, shapes, x, y, plan, "exact_weighted")
    acc = ReferenceAccumulator(gf.params())
    got, st_got = O.mini_batch_gradient(gf, shapes, x, y, plan, "exact_weighted", acc)
    flat = lambda d: np.concatenate([d[n].ravel() for n in shapes])   # noqa: E731
    assert rel_l2(flat(got), flat(want)) <= 1e-6
    assert st_got["grad_norm"] == pytest.approx(st_want["grad_norm"], rel=1e-6)
    assert acc.device_sums.is_cuda and acc.device_sums.dtype == torch.float32
