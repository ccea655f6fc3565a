"""K2 staging and the pinned H2D streamer: bit-exact with the reference's index split.

The reference's micro-batch k of mini-batch m is
ascontiguousarray(x[order[m*M:(m+1)*M]][lo:hi]) (engine.py:310-311, 149-151);
staged bytes must equal torch's x[rows].to(dtype[, channels_last]).
"""
import numpy as np
import pytest
import torch

import paper_2110_12484_b200 as mbs
from oracle import mbs_oracle as O
from paper_2110_12484_b200.streamer import Staging, gather_rows, stage_rows

pytestmark = pytest.mark.gpu


def _src(dtype, shape, device, seed=0):
    g = torch.Generator().manual_seed(seed)
    if dtype == torch.uint8:
        t = torch.randint(0, 256, shape, generator=g, dtype=torch.uint8)
    else:
        t = (torch.randn(shape, generator=g, dtype=torch.float64) * 300).to(dtype)
        t.view(-1)[:5] = torch.tensor([0.0, -0.0, 1e-40, 65504.5, 3.3895e38], dtype=torch.float64).to(dtype)
    return t.to(device)


def _bits(t):
    """Bit pattern in memory order (so NHWC vs NCHW and -0.0 vs 0.0 are both caught)."""
    it = {4: torch.int32, 2: torch.int16}[t.element_size()]
    flat = t.permute(0, 2, 3, 1).reshape(-1) if (t.dim() == 4 and t.is_contiguous(
        memory_format=torch.channels_last) and not t.is_contiguous()) else t.reshape(-1)
    return flat.contiguous().view(it)


@pytest.mark.parametrize("src_dtype", [torch.uint8, torch.float32, torch.float64])
@pytest.mark.parametrize("dst_dtype", [torch.float32, torch.bfloat16, torch.float16])
@pytest.mark.parametrize("shape", [(40, 3, 32, 32), (33, 3, 17, 13), (20, 1, 8, 8), (25, 4, 16, 16), (21, 5, 6, 6),
                                   (30, 12)])
@pytest.mark.parametrize("cl", [False, True])
def test_stage_bit_exact(cuda, src_dtype, dst_dtype, shape, cl):
    x = _src(src_dtype, shape, cuda)
    rows = torch.from_numpy(O.epoch_order(shape[0], 3, 1)[:shape[0] // 2 + 1].astype(np.int64)).to(cuda)
    st = Staging(dtype=dst_dtype, channels_last=cl)
    got = stage_rows(x, src_dtype, tuple(shape[1:]), rows, 0, len(rows), st, cuda)
    want = x[rows].to(dst_dtype)
    if cl and len(shape) == 4:
        want = want.contiguous(memory_format=torch.channels_last)
        assert got.is_contiguous(memory_format=torch.channels_last)
    assert torch.equal(_bits(got), _bits(want))
    # contiguous range variant (row0)
    got2 = stage_rows(x, src_dtype, tuple(shape[1:]), None, 3, 7, st, cuda)
    want2 = x[3:10].to(dst_dtype)
    if cl and len(shape) == 4:
        want2 = want2.contiguous(memory_format=torch.channels_last)
    assert torch.equal(_bits(got2), _bits(want2))


@pytest.mark.parametrize("path", ["0", "1", "2", "3", "3:2048", "4", "4:flat128", "5", "5:ws16"])
@pytest.mark.parametrize("dst_dtype", [torch.float32, torch.bfloat16, torch.float16])
@pytest.mark.parametrize("shape", [(9, 3, 80, 80), (5, 3, 224, 224), (7, 4, 64, 64), (6, 2, 48, 48),
                                   (300, 3, 16, 16)])
def test_stage_u8_nhwc_every_path(cuda, monkeypatch, path, dst_dtype, shape):
    """Every K2 NHWC implementation (MBS_K2_PATH: per-row, grid-stride, smem tile, bulk-async TMA ring per row,
    bulk-async over the flattened pixel space with tiles crossing rows, its warp-specialised form with 8 or 16
    pixels per lane) is
    bit-exact, including ragged last tiles (80x80 = 4096 + 2304 px, 224x224 = 12 x 4096 + 1024 px) and
    more tiles than resident CTAs."""
    monkeypatch.setenv("MBS_K2_PATH", path.split(":")[0])
    monkeypatch.setenv("MBS_K2_TILE", path.split(":")[-1])
    monkeypatch.setenv("MBS_K2_FLAT", "128" if path.endswith("flat128") else "0")
    monkeypatch.setenv("MBS_K2_WS_PX", "16" if path.endswith("ws16") else "8")
    x = _src(torch.uint8, shape, cuda)
    rows = torch.from_numpy(O.epoch_order(shape[0], 5, 2).astype(np.int64)).to(cuda)
    st = Staging(dtype=dst_dtype, channels_last=True)
    got = stage_rows(x, torch.uint8, tuple(shape[1:]), rows, 0, len(rows), st, cuda)
    want = x[rows].to(dst_dtype).contiguous(memory_format=torch.channels_last)
    assert torch.equal(_bits(got), _bits(want))
    got2 = stage_rows(x, torch.uint8, tuple(shape[1:]), None, 1, shape[0] - 2, st, cuda)
    want2 = x[1:shape[0] - 1].to(dst_dtype).contiguous(memory_format=torch.channels_last)
    assert torch.equal(_bits(got2), _bits(want2))


def test_stage_bf16_rounding_matches_torch(cuda):
    # ties-to-even and NaN handling of f32 -> bf16
    vals = torch.tensor([1.00390625, 1.01171875, -2.5e-39, float("nan"), float("inf"), -float("inf"), 3.0e38,
                         1.0 + 2 ** -8, 1.0 + 3 * 2 ** -9], dtype=torch.float32)
    x = vals.repeat(4 * 16).reshape(4, 1, 1, -1).to(cuda)
    got = stage_rows(x, torch.float32, tuple(x.shape[1:]), None, 0, 4, Staging(torch.bfloat16), cuda)
    assert torch.equal(got.view(torch.int16), x.to(torch.bfloat16).view(torch.int16))


@pytest.mark.parametrize("dtype,shape", [(torch.int64, ()), (torch.float32, (1, 9, 9)), (torch.uint8, (3,)),
                                         (torch.float64, (5,))])
def test_gather_rows_bit_exact(cuda, dtype, shape):
    n = 57
    y = (torch.randint(0, 1000, (n,) + shape) if dtype != torch.float32 else torch.rand((n,) + shape)).to(dtype)
    y = y.to(cuda)
    rows = torch.randperm(n, device=cuda)[:23]
    got = gather_rows(y, dtype, shape, rows, 0, 23, cuda)
    assert torch.equal(got, y[rows])


@pytest.mark.parametrize("prefetch", [False, True])
@pytest.mark.parametrize("pinned", [False, True])
@pytest.mark.parametrize("slots", [2, 3])
def test_streamer_partition_bit_exact(cuda, prefetch, pinned, slots):
    n, M, mu = 37, 16, 5
    x = torch.randint(0, 256, (n, 3, 12, 10), dtype=torch.uint8)
    y = torch.randint(0, 10, (n,), dtype=torch.int64)
    if pinned:
        x, y = x.pin_memory(), y.pin_memory()
    order = O.epoch_order(n, 0, 2)
    jobs, want = [], []
    for start in range(0, n, M):
        idx = order[start:start + M]
        plan = O.plan_split(len(idx), mu)
        for k in range(plan.n_s_mu):
            rows = O.micro_batch_rows(order, start, plan, k)
            jobs.append((rows, 0, len(rows)))
            want.append((O.stage_micro(x.numpy(), rows), O.stage_micro(y.numpy(), rows)))
    streamer = mbs.make_streamer(x, y, mu, n_slots=slots)
    got = [(a.cpu().numpy(), b.cpu().numpy()) for a, b in
           streamer.stream(x, y, jobs, Staging(torch.float32), prefetch=prefetch)]
    assert len(got) == len(want)
    for (gx, gy), (wx, wy) in zip(got, want):
        assert np.array_equal(gx, wx.astype(np.float32))
        assert np.array_equal(gy, wy)
    t = streamer.timings()
    assert len(t) == len(jobs) and all(c >= 0 for _, c, _, _ in t)
    streamer.close()


def test_streamer_contiguous_pinned_zero_copy(cuda):
    n = 64
    x = torch.randn(n, 3, 8, 8).pin_memory()
    y = torch.rand(n, 1, 8, 8).pin_memory()
    plan = mbs.plan_split(n, 24)
    jobs = [(None, lo, hi - lo) for lo, hi in plan.index_ranges]
    streamer = mbs.make_streamer(x, y, 24)
    outs = list(streamer.stream(x, y, jobs, Staging(torch.bfloat16, channels_last=True), prefetch=True))
    for (lo, hi), (xk, yk) in zip(plan.index_ranges, outs):
        assert torch.equal(xk.float(), x[lo:hi].to(torch.bfloat16).float().to(cuda))
        assert torch.equal(yk, y[lo:hi].to(cuda))
    gathers = [g for g, _, _, _ in streamer.timings()]
    assert all(g == 0.0 for g in gathers)     # pinned + contiguous: DMA straight from the dataset
    streamer.close()
