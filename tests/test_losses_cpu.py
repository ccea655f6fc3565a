"""losses.py semantics of the torch loss / metric functions vs the reference (fixtures), on CPU float64.

The losses are torch ops (they run wherever the model output lives); the MBS
contract they carry is the MEAN reduction (losses.py:1-8). Values must match
the reference's NumPy implementation to float64 rounding; the gradients are
checked end-to-end by the GPU parity tests.
"""
import numpy as np
import pytest
import torch

import paper_2110_12484_b200 as mbs
from paper_2110_12484_b200 import losses as L
from tests.golden_io import fhex, load_json, load_npz


@pytest.mark.parametrize("i", range(6))
def test_losses_and_metrics_match_reference(i):
    meta = load_json("losses.json")["losses"][i]
    a = load_npz("losses.npz")
    t = {k.split("/")[1]: torch.from_numpy(v) for k, v in a.items() if k.startswith(f"l{i}/")}
    z, m = t["z"], t["t"]
    p = torch.sigmoid(z)
    assert float(L.compute_loss("mse", t["d"], t["td"])) == pytest.approx(fhex(meta["mse"]), rel=1e-12)
    assert float(L.compute_loss("cross_entropy", t["logits"], t["cls"])) == pytest.approx(
        fhex(meta["cross_entropy"]), rel=1e-12)
    assert float(L.compute_loss("bce", z, m, from_logits=True)) == pytest.approx(fhex(meta["bce_logits"]), rel=1e-12)
    assert float(L.compute_loss("bce", p, m, from_logits=False)) == pytest.approx(fhex(meta["bce_probs"]), rel=1e-10)
    assert float(L.compute_loss("bce_dice", z, m, from_logits=True)) == pytest.approx(
        fhex(meta["bce_dice_logits"]), rel=1e-12)
    assert float(L.compute_loss("bce_dice", p, m, from_logits=False)) == pytest.approx(
        fhex(meta["bce_dice_probs"]), rel=1e-10)
    assert mbs.accuracy(t["logits"], t["cls"]) == meta["accuracy"]
    for thr in (0.3, 0.5):
        for per in (False, True):
            assert mbs.dice_coefficient(p, m, thr, per) == pytest.approx(meta[f"dice_{thr}_{per}"], rel=1e-12)
            assert mbs.iou(p, m, thr, per) == pytest.approx(meta[f"iou_{thr}_{per}"], rel=1e-12)


def test_metric_edge_cases():
    e = load_json("losses.json")["empty"]
    z0 = torch.zeros(2, 1, 3, 3, dtype=torch.float64)
    assert mbs.dice_coefficient(z0, z0) == e[0] == 1.0
    assert mbs.iou(z0, z0, per_image=True) == e[1] == 1.0
    with pytest.raises(ValueError):
        mbs.iou(z0, z0, threshold=1.0)
    half = torch.full((4, 8), 0.5, dtype=torch.float64)
    tgt = (torch.arange(32).reshape(4, 8) % 2).double()
    assert float(L.compute_loss("bce", half, tgt, from_logits=False)) == pytest.approx(np.log(2.0), abs=1e-12)


def test_loss_errors():
    with pytest.raises(ValueError):
        L.compute_loss("hinge", torch.zeros(2, 2), torch.zeros(2, 2))
    with pytest.raises(ValueError):
        L.compute_loss("mse", torch.zeros(2, 2), torch.zeros(2, 3))
    with pytest.raises(ValueError):
        L.compute_loss("cross_entropy", torch.zeros(2, 3, 1), torch.zeros(2, dtype=torch.long))
