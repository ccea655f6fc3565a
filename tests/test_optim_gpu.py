"""K3 (fused SGD-momentum / Adam flat step) vs the reference's own optimizer outputs (golden)."""
import numpy as np
import pytest
import torch

import paper_2110_12484_b200 as mbs
from tests.golden_io import load_json, load_npz
from tests.gpu_util import rel_l2, to64

pytestmark = pytest.mark.gpu


class _M(torch.nn.Module):
    def __init__(self, arrays, device):
        super().__init__()
        self.names = list(arrays)
        for i, (n, v) in enumerate(arrays.items()):
            setattr(self, f"t{i}", torch.nn.Parameter(torch.from_numpy(v).float().to(device)))


STATES = {"sgd": lambda: mbs.sgd_state(0.1, 0.9, 5e-4),
          "sgd_nomom": lambda: mbs.OptimizerState(kind="sgd", lr=0.05),
          "adam": lambda: mbs.adam_state(0.01, 5e-4),
          "adam_nowd": lambda: mbs.adam_state(0.003, 0.0, 0.8, 0.99, 1e-6)}


@pytest.mark.parametrize("kind", list(STATES))
def test_optimizer_matches_reference(cuda, kind):
    meta = load_json("accum_optim.json")
    a = load_npz("accum_optim.npz")
    names = list(meta["shapes"])
    mod = _M({n: a[f"p0/{n}"] for n in names}, cuda)
    params = mbs.ParameterSet(mod)
    tn = params.names()
    st = STATES[kind]()
    for step in range(3):
        grads = mbs.GradientSet({tn[i]: torch.from_numpy(a[f"g{step}/{n}"]).float().to(cuda)
                                 for i, n in enumerate(names)})
        mbs.apply_update(params, grads, st)
        for i, n in enumerate(names):
            want = a[f"{kind}/step{step}/{n}"]
            got = to64(params[tn[i]])
            assert rel_l2(got, want) <= 2e-6, (kind, step, n)
    assert st.step_count == meta[f"{kind}_step_count"]
    if kind.startswith("sgd"):
        assert set(st.velocity) == set(tn)


def test_guard_skips_nonfinite_step(cuda):
    mod = _M({"w": np.ones((8, 8), np.float32)}, cuda)
    params = mbs.ParameterSet(mod)
    g = mbs.GradientSet({params.names()[0]: torch.full((8, 8), 0.5, device=cuda)},
                        norm2=torch.tensor(float("inf"), dtype=torch.float64, device=cuda))
    st = mbs.sgd_state(0.1, 0.0, 0.0)
    mbs.apply_update(params, g, st)
    assert torch.equal(params[params.names()[0]].data, torch.ones(8, 8, device=cuda))
    g.norm2 = torch.tensor(1.0, dtype=torch.float64, device=cuda)
    mbs.apply_update(params, g, st)
    assert torch.allclose(params[params.names()[0]].data, torch.full((8, 8), 0.95, device=cuda))


def test_key_mismatch(cuda):
    mod = _M({"w": np.ones((4,), np.float32), "b": np.ones((2,), np.float32)}, cuda)
    params = mbs.ParameterSet(mod)
    with pytest.raises(mbs.GradientKeyMismatchError):
        mbs.apply_update(params, mbs.GradientSet({params.names()[0]: torch.ones(4, device=cuda)}),
                         mbs.sgd_state())
    with pytest.raises(mbs.GradientKeyMismatchError):
        mbs.apply_update(params, mbs.GradientSet({params.names()[0]: torch.ones(5, device=cuda),
                                                  params.names()[1]: torch.ones(2, device=cuda)}), mbs.sgd_state())
