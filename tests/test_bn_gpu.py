"""K5 micro-batch BatchNorm (+ fused ReLU / residual) vs a float64 torch reference of the same op.

Contract: fp32 activations — outputs, dx, dresidual, dweight, dbias, saved
statistics and running statistics within rel-L2 1e-5 of float64 (the op's own
fp32 rounding; measured ~1e-7); bf16 activations — no worse than torch's own
bf16 channels-last BatchNorm against the same float64 reference (x 1.5 + a
bf16 ulp of slack). Runs are bit-reproducible (fixed-order reductions). The
module rewrite keeps every parameter / buffer / state-dict key and order.
"""
import copy

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from paper_2110_12484_b200 import bn as K5
from tests.gpu_util import rel_l2

pytestmark = pytest.mark.gpu


def _ref64(x, res, w, b, relu, dy, rm=None, rv=None, momentum=0.1, eps=1e-5):
    """float64 reference: y = relu(bn(x) + res); grads via autograd; running stats torch-style."""
    x64 = x.detach().double().requires_grad_(True)
    r64 = None if res is None else res.detach().double().requires_grad_(True)
    w64 = w.detach().double().requires_grad_(True)
    b64 = b.detach().double().requires_grad_(True)
    rm64 = None if rm is None else rm.double().clone()
    rv64 = None if rv is None else rv.double().clone()
    y = F.batch_norm(x64, rm64, rv64, w64, b64, True, momentum, eps)
    if r64 is not None:
        y = y + r64
    if relu:
        y = F.relu(y)
    y.backward(dy.double())
    dims = [0] + list(range(2, x.dim()))
    mean = x64.detach().mean(dims)
    var = x64.detach().var(dims, unbiased=False)
    return dict(y=y.detach(), dx=x64.grad, dres=None if r64 is None else r64.grad, dw=w64.grad, db=b64.grad,
                mean=mean, invstd=1.0 / torch.sqrt(var + eps), rm=rm64, rv=rv64)


def _data(cuda, shape, dtype, seed, offset=3.0):
    g = torch.Generator(device=cuda).manual_seed(seed)
    C = shape[1]
    x = (torch.randn(shape, device=cuda, generator=g) * 2.0 + offset).to(dtype)
    res = torch.randn(shape, device=cuda, generator=g).to(dtype)
    dy = torch.randn(shape, device=cuda, generator=g).to(dtype)
    w = torch.randn(C, device=cuda, generator=g) * 0.5 + 1.0
    b = torch.randn(C, device=cuda, generator=g) * 0.1
    if x.dim() == 4:
        x, res, dy = (t.contiguous(memory_format=torch.channels_last) for t in (x, res, dy))
    return x, res, dy, w, b


def _run(x, res, dy, w, b, relu, rm=None, rv=None):
    xx = x.detach().clone().requires_grad_(True)
    rr = None if res is None else res.detach().clone().requires_grad_(True)
    ww = w.detach().clone().requires_grad_(True)
    bb = b.detach().clone().requires_grad_(True)
    y = K5.micro_batch_norm(xx, ww, bb, rm, rv, relu=relu, residual=rr)
    y.backward(dy)
    return dict(y=y.detach(), dx=xx.grad, dres=None if rr is None else rr.grad, dw=ww.grad, db=bb.grad)


SHAPES = [(8, 64, 14, 14), (4, 256, 7, 9), (2, 2048, 3, 3), (16, 24, 5, 5), (3, 3, 11, 7), (2, 520, 2, 3),
          (37, 40), (5, 2056, 1, 1)]


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("mode", ["plain", "relu", "relu_res"])
def test_k5_fp32_vs_float64(cuda, shape, mode):
    relu, use_res = mode != "plain", mode == "relu_res"
    x, res, dy, w, b = _data(cuda, shape, torch.float32, seed=sum(shape) + len(mode))
    res = res if use_res else None
    C = shape[1]
    rm0 = torch.randn(C, device=cuda) * 0.1
    rv0 = torch.rand(C, device=cuda) + 0.5
    rm, rv = rm0.clone(), rv0.clone()
    got = _run(x, res, dy, w, b, relu, rm, rv)
    want = _ref64(x, res, w, b, relu, dy, rm0, rv0)
    for k in ("y", "dx", "dw", "db") + (("dres",) if use_res else ()):
        err = rel_l2(got[k].double().cpu().numpy(), want[k].cpu().numpy())
        assert err <= 1e-5, (k, err)
    assert rel_l2(rm.double().cpu().numpy(), want["rm"].cpu().numpy()) <= 1e-6
    assert rel_l2(rv.double().cpu().numpy(), want["rv"].cpu().numpy()) <= 1e-6


@pytest.mark.parametrize("shape", [(32, 64, 28, 28), (16, 256, 14, 14), (32, 2048, 7, 7), (8, 128, 9, 13)])
@pytest.mark.parametrize("mode", ["plain", "relu", "relu_res"])
def test_k5_bf16_no_worse_than_torch(cuda, shape, mode):
    relu, use_res = mode != "plain", mode == "relu_res"
    x, res, dy, w, b = _data(cuda, shape, torch.bfloat16, seed=7)
    res = res if use_res else None
    got = _run(x, res, dy, w, b, relu)
    want = _ref64(x, res, w, b, relu, dy)
    # torch's own bf16 path of the same op
    xt = x.detach().clone().requires_grad_(True)
    rt = None if res is None else res.detach().clone().requires_grad_(True)
    wt = w.detach().clone().requires_grad_(True)
    bt = b.detach().clone().requires_grad_(True)
    yt = F.batch_norm(xt, None, None, wt, bt, True, 0.1, 1e-5)
    if rt is not None:
        yt = yt + rt
    if relu:
        yt = F.relu(yt)
    yt.backward(dy)
    tgot = dict(y=yt.detach(), dx=xt.grad, dres=None if rt is None else rt.grad, dw=wt.grad, db=bt.grad)
    for k in ("y", "dx", "dw", "db") + (("dres",) if use_res else ()):
        ours = rel_l2(got[k].double().cpu().numpy(), want[k].cpu().numpy())
        theirs = rel_l2(tgot[k].double().cpu().numpy(), want[k].cpu().numpy())
        assert ours <= 1.5 * theirs + 4e-3, (k, ours, theirs)


def test_k5_deterministic(cuda):
    x, res, dy, w, b = _data(cuda, (16, 256, 14, 14), torch.bfloat16, seed=3)
    a = _run(x, res, dy, w, b, True)
    c = _run(x, res, dy, w, b, True)
    for k in a:
        assert torch.equal(a[k], c[k]), k


def test_k5_unaligned_inputs_take_the_scalar_path(cuda):
    # a storage offset of one float breaks 16-byte alignment: the V=1 kernels must give the same answer
    x, _, dy, w, b = _data(cuda, (4, 64, 6, 6), torch.float32, seed=5)
    base = torch.empty(x.numel() + 1, device=cuda)
    base[1:].view(4, 6, 6, 64).copy_(x.permute(0, 2, 3, 1))
    base.requires_grad_(True)
    xu = base[1:].view(4, 6, 6, 64).permute(0, 3, 1, 2)          # channels-last strides, misaligned
    assert xu.data_ptr() % 16 != 0 and xu.is_contiguous(memory_format=torch.channels_last)
    y = K5.micro_batch_norm(xu, w, b, relu=True)
    y.backward(dy)
    dx = base.grad[1:].view(4, 6, 6, 64).permute(0, 3, 1, 2)
    want = _ref64(x, None, w, b, True, dy)
    assert rel_l2(dx.double().cpu().numpy(), want["dx"].cpu().numpy()) <= 1e-5
    assert rel_l2(y.detach().double().cpu().numpy(), want["y"].cpu().numpy()) <= 1e-5


def test_k5_nchw_input_is_converted(cuda):
    x, res, dy, w, b = _data(cuda, (4, 32, 5, 5), torch.float32, seed=6)
    got = _run(x.contiguous(), res.contiguous(), dy.contiguous(), w, b, True)
    want = _ref64(x, res, w, b, True, dy)
    for k in ("y", "dx", "dres", "dw", "db"):
        assert rel_l2(got[k].double().cpu().numpy(), want[k].cpu().numpy()) <= 1e-5, k


def test_k5_one_value_per_channel_follows_the_reference(cuda):
    """One value per channel (a 1-sample micro-batch on a 1x1 map): torch raises, the reference does not
    (SPEC.md:92). K5: y = beta (+ReLU), dx = 0, dbeta = sum dy, dgamma = 0, running_var -> biased 0."""
    m = K5.MicroBatchNorm2d(8).to(cuda).train()
    with torch.no_grad():
        m.weight.uniform_(0.5, 1.5)
        m.bias.uniform_(-1.0, 1.0)
    x = torch.randn(1, 8, 1, 1, device=cuda, requires_grad=True)
    y = m(x)
    assert torch.allclose(y.detach().reshape(8), m.bias.detach(), rtol=0, atol=1e-5)
    dy = torch.randn_like(y)
    y.backward(dy)
    assert float(x.grad.abs().max()) <= 1e-4 * float(dy.abs().max())      # 0 up to fp32 cancellation
    assert torch.allclose(m.bias.grad, dy.reshape(8), rtol=1e-6, atol=0)
    assert float(m.weight.grad.abs().max()) <= 1e-6
    assert torch.allclose(m.running_mean, 0.1 * x.detach().reshape(8))
    assert torch.allclose(m.running_var, torch.full((8,), 0.9, device=cuda))
    with pytest.raises(ValueError):
        F.batch_norm(torch.randn(1, 8, 1, 1, device=cuda), None, None, training=True)


def _models():
    import torchvision
    from paper_2110_12484_b200.workloads import UNet
    torch.manual_seed(0)
    return [("resnet18", torchvision.models.resnet18(num_classes=10), (6, 3, 32, 32)),
            ("resnet50", torchvision.models.resnet50(num_classes=12), (4, 3, 64, 64)),
            ("unet", UNet(3, 1), (2, 3, 32, 32))]


@pytest.mark.parametrize("idx", [0, 1, 2])
def test_fused_model_no_worse_than_torch_model_fp32(cuda, idx):
    """Whole models (fp32, TF32 off): fused-K5 vs torch BatchNorm, both against a float64 copy.

    Small micro-batches make BN models ill-conditioned in fp32 (~1e-3 floor), so the
    contract is relative to torch's own fp32 error on the same model and input.
    """
    name, net, shape = _models()[idx]
    net = net.to(cuda).to(memory_format=torch.channels_last).train()
    fused = K5.fuse_batchnorm(copy.deepcopy(net))
    ref = copy.deepcopy(net).double()
    assert list(fused.state_dict()) == list(net.state_dict())
    assert [n for n, _ in fused.named_parameters()] == [n for n, _ in net.named_parameters()]
    g = torch.Generator(device=cuda).manual_seed(1)
    x = torch.randn(shape, device=cuda, generator=g).contiguous(memory_format=torch.channels_last)
    res = {}
    for key, m, xin in (("torch", net, x), ("ours", fused, x), ("f64", ref, x.double())):
        out = m(xin)
        (out ** 2).mean().backward()
        res[key] = dict(out=out.detach().double().cpu().numpy(),
                        grad=np.concatenate([p.grad.double().cpu().numpy().ravel() for p in m.parameters()]),
                        bufs=np.concatenate([v.double().cpu().numpy().ravel() for k, v in m.state_dict().items()
                                             if "running" in k]))
    for k in ("out", "grad", "bufs"):
        ours = rel_l2(res["ours"][k], res["f64"][k])
        theirs = rel_l2(res["torch"][k], res["f64"][k])
        assert ours <= max(1e-5, 1.5 * theirs), (name, k, ours, theirs)
    nbt = [v for k, v in fused.state_dict().items() if k.endswith("num_batches_tracked")]
    assert all(int(v) == 1 for v in nbt)
    # eval mode: running statistics, same as torch
    net.eval()
    fused.eval()
    with torch.no_grad():
        assert rel_l2(fused(x).double().cpu().numpy(), net(x).double().cpu().numpy()) <= 1e-4


@pytest.mark.parametrize("shape", [(32, 64, 28, 28), (16, 2048, 7, 7), (8, 24, 9, 13)])
@pytest.mark.parametrize("mode", ["plain", "relu", "relu_res"])
def test_k5_cooperative_path_matches_three_kernel_path(cuda, shape, mode, monkeypatch):
    """Small layers run as ONE cooperative kernel per direction; it must agree with the
    three-kernel (reduce / finalize / apply) path to fp32 reduction-order noise."""
    relu, use_res = mode != "plain", mode == "relu_res"
    x, res, dy, w, b = _data(cuda, shape, torch.bfloat16, seed=21)
    res = res if use_res else None
    monkeypatch.setenv("MBS_K5_FUSED_MB", "64")      # every case here takes the cooperative path when enabled
    monkeypatch.setenv("MBS_K5_FUSED", "1")
    a = _run(x, res, dy, w, b, relu)
    monkeypatch.setenv("MBS_K5_FUSED", "0")
    c = _run(x, res, dy, w, b, relu)
    for k in a:
        if a[k] is None:
            continue
        assert rel_l2(a[k].double().cpu().numpy(), c[k].double().cpu().numpy()) <= 4e-3, k   # bf16 outputs
    monkeypatch.setenv("MBS_K5_FUSED", "1")
    xf, rf, dyf, wf, bf = _data(cuda, shape, torch.float32, seed=22)
    rf = rf if use_res else None
    a = _run(xf, rf, dyf, wf, bf, relu)
    monkeypatch.setenv("MBS_K5_FUSED", "0")
    c = _run(xf, rf, dyf, wf, bf, relu)
    for k in a:
        if a[k] is None:
            continue
        assert rel_l2(a[k].double().cpu().numpy(), c[k].double().cpu().numpy()) <= 1e-6, k


def _run_dual(x, res, g1, g2, w, b, relu):
    xx = x.detach().clone().requires_grad_(True)
    rr = None if res is None else res.detach().clone().requires_grad_(True)
    ww = w.detach().clone().requires_grad_(True)
    bb = b.detach().clone().requires_grad_(True)
    y1, y2 = K5.micro_batch_norm(xx, ww, bb, relu=relu, residual=rr, dual=True)
    outs, grads = zip(*[(y, g) for y, g in ((y1, g1), (y2, g2)) if g is not None])
    torch.autograd.backward(list(outs), list(grads))
    return dict(y=y1.detach(), dx=xx.grad, dres=None if rr is None else rr.grad, dw=ww.grad, db=bb.grad)


@pytest.mark.parametrize("shape", [(8, 64, 14, 14), (4, 256, 7, 9), (2, 2048, 3, 3), (3, 24, 5, 5), (4, 3, 5, 5)])
@pytest.mark.parametrize("mode", ["relu_res", "relu", "plain"])
def test_k5_dual_output_fp32_bit_identical_to_summed_gradient(cuda, shape, mode):
    """Dual output (two consumers of one activation): K5 sums the two gradients in fp32 inside its
    backward reduce (mbs_bn_backward dy2) — in fp32 that is exactly torch's add, so every output is
    bit-identical to feeding dy1 + dy2 (C=3: unaligned vectors, Python-side add)."""
    relu, use_res = mode != "plain", mode == "relu_res"
    x, res, g1, w, b = _data(cuda, shape, torch.float32, seed=31)
    g2 = torch.randn_like(g1)
    res = res if use_res else None
    a = _run_dual(x, res, g1, g2, w, b, relu)
    c = _run(x, res, g1 + g2, w, b, relu)
    for k in a:
        if a[k] is not None:
            assert torch.equal(a[k], c[k]), k
    a = _run_dual(x, res, None, g2, w, b, relu)            # one handle unused: its gradient is None
    c = _run(x, res, g2, w, b, relu)
    for k in a:
        if a[k] is not None:
            assert torch.equal(a[k], c[k]), k


@pytest.mark.parametrize("shape", [(32, 256, 28, 28), (8, 2048, 7, 7)])
def test_k5_dual_output_bf16_no_worse_than_rounded_add(cuda, shape):
    """bf16: the in-kernel fp32 sum skips the bf16 rounding of autograd's add — as accurate or better
    against float64."""
    x, res, g1, w, b = _data(cuda, shape, torch.bfloat16, seed=32)
    g2 = torch.randn_like(g1)
    a = _run_dual(x, res, g1, g2, w, b, True)
    c = _run(x, res, g1 + g2, w, b, True)
    ref = _ref64(x, res, w, b, True, g1.double() + g2.double())
    for k in ("dx", "dres", "dw", "db"):
        ours = rel_l2(a[k].double().cpu().numpy(), ref[k].double().cpu().numpy())
        add = rel_l2(c[k].double().cpu().numpy(), ref[k].double().cpu().numpy())
        assert ours <= max(1e-5, 1.05 * add), (k, ours, add)


@pytest.mark.parametrize("shape", [(32, 256, 28, 28), (8, 2048, 7, 7)])
def test_k5_dual_output_bf16_bit_identical_to_rounded_add(cuda, shape, monkeypatch):
    """bf16: K5 rounds dy1 + dy2 to bf16 (torch's bf16 add) before the statistics and the stored
    d_residual, so the dual path equals feeding the autograd-added gradient bit for bit (three-kernel
    path on both sides: MBS_K5_FUSED=0)."""
    monkeypatch.setenv("MBS_K5_FUSED", "0")
    x, res, g1, w, b = _data(cuda, shape, torch.bfloat16, seed=33)
    g2 = torch.randn_like(g1)
    a = _run_dual(x, res, g1, g2, w, b, True)
    c = _run(x, res, g1 + g2, w, b, True)
    for k in a:
        if a[k] is not None:
            assert torch.equal(a[k], c[k]), k


@pytest.mark.parametrize("arch", ["resnet18", "resnet50"])
def test_fused_resnet_dual_handles_match_autograd_adds(cuda, arch, monkeypatch):
    """FusedResNet (block outputs handed on as two handles) vs the same fused model with autograd's
    adds (MBS_K5_DUAL=0): fp32, deterministic cuDNN — identical outputs, gradients and buffers."""
    import torchvision
    monkeypatch.setattr(torch.backends.cudnn, "deterministic", True)
    monkeypatch.setattr(torch.backends.cudnn, "benchmark", False)
    torch.manual_seed(0)
    net = getattr(torchvision.models, arch)(num_classes=10).to(cuda).to(memory_format=torch.channels_last).train()
    from paper_2110_12484_b200 import pool as K6
    monkeypatch.setenv("MBS_K5_DUAL", "1")
    dual = K6.swap_maxpool(K5.fuse_batchnorm(copy.deepcopy(net)))     # K6 stem pool: dual output too
    monkeypatch.setenv("MBS_K5_DUAL", "0")
    plain = K6.swap_maxpool(K5.fuse_batchnorm(copy.deepcopy(net)))
    assert type(dual) is K5.FusedResNet and type(plain) is not K5.FusedResNet
    assert list(dual.state_dict()) == list(net.state_dict())
    x = torch.randn(6, 3, 64, 64, device=cuda).contiguous(memory_format=torch.channels_last)
    outs = []
    for m in (dual, plain):
        out = m(x)
        (out ** 2).mean().backward()
        outs.append((out.detach(), [p.grad for p in m.parameters()], [v for v in m.state_dict().values()]))
    assert torch.equal(outs[0][0], outs[1][0])
    for a, c in zip(outs[0][1], outs[1][1]):
        assert torch.equal(a, c)
    for a, c in zip(outs[0][2], outs[1][2]):
        assert torch.equal(a, c)


def test_k5_dy2_contract_errors(cuda):
    """mbs_bn_backward's dy2 is only accepted on the fused residual + ReLU path (include/mbs.h);
    anything else is a loud MBS error, never a silent drop of the second gradient."""
    from paper_2110_12484_b200 import _native
    x, res, dy, w, b = _data(cuda, (4, 64, 6, 6), torch.bfloat16, seed=41)
    rows, C = 4 * 36, 64
    mean = torch.zeros(C, device=cuda)
    inv = torch.ones(C, device=cuda)
    dx = torch.empty_like(x)
    ws = K5._workspace(rows, C, _native.BF16, cuda)
    st = torch.cuda.current_stream().cuda_stream
    lib = _native.lib()
    # relu without residual + dy2: rejected
    rc = lib.mbs_bn_backward(x.data_ptr(), None, dy.data_ptr(), dy.data_ptr(), dx.data_ptr(), None, _native.BF16, rows,
                             C, w.data_ptr(), b.data_ptr(), mean.data_ptr(), inv.data_ptr(), 1, None, None,
                             ws.data_ptr(), st)
    assert rc != 0
    # misaligned dy2 on the residual path: rejected (scalar path cannot take it)
    dres = torch.empty_like(x)
    flat = torch.empty(x.numel() + 1, device=cuda, dtype=x.dtype)
    rc = lib.mbs_bn_backward(x.data_ptr(), res.data_ptr(), dy.data_ptr(), flat[1:].data_ptr(), dx.data_ptr(),
                             dres.data_ptr(), _native.BF16, rows, C, w.data_ptr(), b.data_ptr(), mean.data_ptr(),
                             inv.data_ptr(), 1, None, None, ws.data_ptr(), st)
    assert rc != 0
    torch.cuda.synchronize()
