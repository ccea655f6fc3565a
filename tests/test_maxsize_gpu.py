"""Maximum size: the WHOLE C4 mini-batch (300,032 ResNet-50@224 samples, 45.2 GB host-resident uint8, more than
HBM as the reference's fp32) and the whole N1 mini-batch (80,000 U-Net@384 images + masks, 47.2 GB; masks staged
to fp32 by K2) streamed through the real path — shuffled epoch order, native gather pool, pinned
ring, H2D copy stream, K2 staging to bf16 NHWC — and checked bit-exact for EVERY micro-batch (C4: 2,344; N1: 1,667 with a
ragged tail of 32).

The host rows are 509 random template rows tiled, each stamped with its own row index in its first 8 bytes, so
every staged sample is predictable on the device (its template row with the stamp overwritten): each micro-batch
is compared in full, bit for bit, against ``x[rows].to(bf16)`` built from the template, and the stamps prove the
order (the epoch permutation, engine.py:300-311, the micro slices, engine.py:149-151). The permutation itself is
checked against the oracle's restatement at this size.
"""
import numpy as np
import pytest
import torch

import paper_2110_12484_b200 as mbs
from oracle import mbs_oracle as O
from paper_2110_12484_b200.streamer import Staging
from paper_2110_12484_b200.workloads import WORKLOADS

pytestmark = pytest.mark.gpu

T = 509                       # template rows


def _stamp(idx: torch.Tensor) -> torch.Tensor:
    """(n, 8) uint8: little-endian bytes of each row index."""
    return torch.stack([(idx >> (8 * b)) & 0xFF for b in range(8)], dim=1).to(torch.uint8)


def _tiled(tmpl: torch.Tensor, n: int) -> torch.Tensor:
    """n rows: the template rows tiled, each stamped with its row index in its first 8 bytes."""
    t = tmpl.shape[0]
    out = torch.empty((n,) + tuple(tmpl.shape[1:]), dtype=torch.uint8)
    for i in range(0, n, t):
        k = min(t, n - i)
        out[i:i + k].copy_(tmpl[:k])
    out.view(n, -1)[:, :8] = _stamp(torch.arange(n, dtype=torch.int64))
    return out


def _rows_of(staged: torch.Tensor) -> torch.Tensor:
    """Decode the stamps of a staged micro-batch (channel 0, image row 0, columns 0..7 of each sample)."""
    stamps = staged[:, 0, 0, :8].to(torch.int64)
    return sum(stamps[:, b] << (8 * b) for b in range(8))


@pytest.mark.parametrize("cfg", ["c4", "n1"])
def test_full_minibatch_streams_bit_exact(cuda, cfg):
    w = WORKLOADS[cfg]
    n, n_mu = w.mini, w.micro
    shape = tuple(w.sample_shape)
    g = torch.Generator().manual_seed(3)
    tmpl = torch.randint(0, 256, (T,) + shape, generator=g, dtype=torch.uint8)
    x = _tiled(tmpl, n)
    if w.target == "mask":
        tmpl_y = (torch.rand((T, 1) + shape[1:], generator=g) < 0.5).to(torch.uint8)
        y = _tiled(tmpl_y, n)             # stamped masks: bytes beyond {0, 1}, still staged exactly to fp32
        st = Staging(torch.bfloat16, channels_last=True, target_dtype=torch.float32)
    else:
        tmpl_y = None
        y = torch.randint(0, w.n_classes, (n,), generator=g, dtype=torch.int64)
        st = Staging(torch.bfloat16, channels_last=True)

    seed, epoch = 4, 7
    order = mbs.epoch_order(n, seed, epoch)
    assert np.array_equal(order, O.epoch_order(n, seed, epoch))      # the partition's permutation, full size
    plan = mbs.plan_split(n, n_mu)
    assert plan.sizes == O.plan_split(n, n_mu).sizes
    jobs = [(order[lo:hi], 0, hi - lo) for lo, hi in plan.index_ranges]

    tmpl_dev = tmpl.to(cuda).to(torch.bfloat16).contiguous(memory_format=torch.channels_last)
    ty_dev = tmpl_y.to(cuda).float() if tmpl_y is not None else None
    y_dev = y.to(cuda) if tmpl_y is None else None
    streamer = mbs.make_streamer(x, y, n_mu, n_slots=3)
    bad, seen = [], 0
    try:
        for k, (xk, yk) in enumerate(streamer.stream(x, y, jobs, st, prefetch=True)):
            rows = torch.from_numpy(jobs[k][0].astype(np.int64)).to(cuda)
            want = tmpl_dev[rows % T].clone()
            want[:, 0, 0, :8] = _stamp(rows).to(torch.bfloat16)
            ok = torch.equal(xk.view(torch.int16), want.view(torch.int16)) and torch.equal(_rows_of(xk), rows)
            if ty_dev is not None:
                wy = ty_dev[rows % T].clone()
                wy[:, 0, 0, :8] = _stamp(rows).float()
                ok = ok and yk.dtype == torch.float32 and torch.equal(yk, wy) and torch.equal(_rows_of(yk), rows)
            else:
                ok = ok and torch.equal(yk, y_dev[rows])
            if not ok:
                bad.append(k)
            seen += xk.shape[0]
    finally:
        streamer.close()
    assert seen == n
    assert not bad, f"{len(bad)} of {plan.n_s_mu} micro-batches differ (first: {bad[:5]})"
