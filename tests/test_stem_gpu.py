"""K7 stem conv (im2col + cuBLAS GEMM) vs torch's conv2d, and whole native-ops models vs float64."""
import copy

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from paper_2110_12484_b200 import stem as K7
from tests.gpu_util import rel_l2

pytestmark = pytest.mark.gpu

CASES = [((4, 3, 32, 32), 64, 7, 2, 3, False), ((2, 3, 20, 18), 16, 3, 1, 1, True), ((2, 1, 9, 9), 8, 3, 2, 0, True),
         ((3, 4, 15, 15), 32, 5, 1, 2, False)]


@pytest.mark.parametrize("case", CASES)
def test_k7_fp32_matches_conv2d(cuda, case):
    shape, o, k, s, p, bias = case
    g = torch.Generator(device=cuda).manual_seed(k + o)
    conv = torch.nn.Conv2d(shape[1], o, k, s, p, bias=bias).to(cuda)
    ref = copy.deepcopy(conv).double()
    K7.swap_stem(conv)
    assert isinstance(conv, K7.StemConv2d)
    x = torch.randn(shape, device=cuda, generator=g).contiguous(memory_format=torch.channels_last)
    y = conv(x)
    yr = ref(x.double())
    assert y.is_contiguous(memory_format=torch.channels_last)
    dy = torch.randn_like(yr)
    y.backward(dy.float())
    yr.backward(dy)
    assert rel_l2(y.detach().double().cpu().numpy(), yr.detach().cpu().numpy()) <= 1e-6
    assert rel_l2(conv.weight.grad.double().cpu().numpy(), ref.weight.grad.cpu().numpy()) <= 1e-6
    if bias:
        assert rel_l2(conv.bias.grad.double().cpu().numpy(), ref.bias.grad.cpu().numpy()) <= 1e-6


def test_k7_bf16_autocast_no_worse_than_cudnn(cuda):
    conv = torch.nn.Conv2d(3, 64, 7, 2, 3, bias=False).to(cuda)
    ref = copy.deepcopy(conv).double()
    tch = copy.deepcopy(conv)
    K7.swap_stem(conv)
    x = torch.randn(8, 3, 64, 64, device=cuda).to(torch.bfloat16).contiguous(memory_format=torch.channels_last)
    yr = ref(x.double())
    dy = torch.randn_like(yr)
    yr.backward(dy)
    errs = {}
    for name, m in (("ours", conv), ("cudnn", tch)):
        with torch.autocast("cuda", dtype=torch.bfloat16):
            y = m(x)
        assert y.dtype == torch.bfloat16
        y.backward(dy.to(y.dtype))
        errs[name] = (rel_l2(y.detach().double().cpu().numpy(), yr.detach().cpu().numpy()),
                      rel_l2(m.weight.grad.double().cpu().numpy(), ref.weight.grad.cpu().numpy()))
    assert errs["ours"][0] <= 1.5 * errs["cudnn"][0] + 1e-3, errs
    assert errs["ours"][1] <= 1.5 * errs["cudnn"][1] + 1e-3, errs


def test_k7_input_grad_when_requested(cuda):
    conv = torch.nn.Conv2d(3, 8, 3, 1, 1, bias=True).to(cuda)
    ref = copy.deepcopy(conv)
    K7.swap_stem(conv)
    x = torch.randn(2, 3, 10, 10, device=cuda).contiguous(memory_format=torch.channels_last).requires_grad_(True)
    xr = x.detach().clone().requires_grad_(True)
    conv(x).sum().backward()
    ref(xr).sum().backward()
    assert torch.allclose(x.grad, xr.grad, rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("cfg", ["c1", "c3"])
def test_native_ops_model_no_worse_than_torch_fp32(cuda, cfg):
    """build_model(ops='native') (K5 + K6 + K7 + fused U-Net skips) vs the stock model, both vs float64."""
    from paper_2110_12484_b200.workloads import WORKLOADS, build_model
    w = WORKLOADS[cfg]
    torch.manual_seed(0)
    base = build_model(w, ops="torch").to(cuda).to(memory_format=torch.channels_last).train()
    nat = build_model(w, ops="torch")
    nat.load_state_dict(base.state_dict())
    from paper_2110_12484_b200 import bn, pool
    bn.fuse_batchnorm(nat)
    pool.swap_maxpool(nat)
    K7.swap_stem(nat)
    K7.swap_pointwise(nat)
    if hasattr(nat, "native_skips"):
        nat.native_skips = True
    nat = nat.to(cuda).to(memory_format=torch.channels_last).train()
    ref = copy.deepcopy(base).double()
    hw = 32
    x = torch.randn(6, 3, hw, hw, device=cuda).contiguous(memory_format=torch.channels_last)
    nchw = copy.deepcopy(base).to(memory_format=torch.contiguous_format)
    res = {}
    for key, m, xin in (("torch", base, x), ("torch_nchw", nchw, x.contiguous()), ("ours", nat, x),
                        ("f64", ref, x.double())):
        out = m(xin)
        (out ** 2).mean().backward()
        res[key] = (out.detach().double().cpu().numpy(),
                    np.concatenate([p.grad.double().cpu().numpy().ravel() for p in m.parameters()]))
    # the fp32 floor is the largest error of two independent torch implementations (cuDNN channels-last and
    # NCHW kernels): BatchNorm over 6 samples makes the gradient chaotic at ReLU ties, so one run's error is luck
    for i, what in enumerate(("out", "grad")):
        ours = rel_l2(res["ours"][i], res["f64"][i])
        theirs = max(rel_l2(res[k][i], res["f64"][i]) for k in ("torch", "torch_nchw"))
        assert ours <= max(1e-5, 1.5 * theirs), (cfg, what, ours, theirs)


def test_pointwise_gemm_conv_matches(cuda):
    conv = torch.nn.Conv2d(16, 1, 1).to(cuda)
    ref = copy.deepcopy(conv).double()
    K7.swap_pointwise(conv)
    assert isinstance(conv, K7.PointwiseConv2d)
    x = torch.randn(2, 16, 9, 7, device=cuda).contiguous(memory_format=torch.channels_last).requires_grad_(True)
    xr = x.detach().double().requires_grad_(True)
    y, yr = conv(x), ref(xr)
    y.sum().backward()
    yr.sum().backward()
    assert rel_l2(y.detach().double().cpu().numpy(), yr.detach().cpu().numpy()) <= 1e-6
    assert rel_l2(x.grad.double().cpu().numpy(), xr.grad.cpu().numpy()) <= 1e-6
    assert rel_l2(conv.weight.grad.double().cpu().numpy(), ref.weight.grad.cpu().numpy()) <= 1e-6
    assert rel_l2(conv.bias.grad.double().cpu().numpy(), ref.bias.grad.cpu().numpy()) <= 1e-6


@pytest.mark.parametrize("case", [((3, 3, 224, 224), 7, 2, 3), ((2, 3, 37, 29), 7, 2, 3), ((2, 3, 48, 40), 3, 1, 1),
                                  ((2, 3, 17, 11), 3, 1, 1), ((2, 3, 16, 16), 3, 2, 0), ((2, 3, 15, 15), 5, 1, 2)])
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_k7_im2col_bit_identical_to_unfold(cuda, case, dtype):
    """K7's patch matrix is pure data movement: every variant (the staged-row kernels for 7x7x3 / 3x3x3
    bf16, the tile kernel otherwise; widths whose rows are / are not 16-byte multiples) must equal
    torch's unfold reordered to (kh, kw, c), zero padding columns included."""
    from paper_2110_12484_b200 import _native
    shape, k, s, p = case
    n, c, h, w = shape
    x = torch.randn(shape, device=cuda).to(dtype).contiguous(memory_format=torch.channels_last)
    ho, wo = (h + 2 * p - k) // s + 1, (w + 2 * p - k) // s + 1
    kk = k * k * c
    kp = (kk + 7) // 8 * 8
    cols = torch.full((n * ho * wo, kp), float("nan"), device=cuda, dtype=dtype)
    code = _native.BF16 if dtype == torch.bfloat16 else _native.F32
    _native.check(_native.lib().mbs_im2col(x.data_ptr(), cols.data_ptr(), code, n, h, w, c, k, s, p, kp,
                                           torch.cuda.current_stream().cuda_stream), "mbs_im2col")
    u = F.unfold(x.float(), k, padding=p, stride=s)                  # [n, c*k*k (c, kh, kw), L]
    ref = u.view(n, c, k, k, ho * wo).permute(0, 4, 2, 3, 1).reshape(n * ho * wo, kk).to(dtype)
    assert torch.equal(cols[:, :kk], ref)
    assert torch.equal(cols[:, kk:], torch.zeros_like(cols[:, kk:]))
