"""K6 channels-last max-pool: forward AND backward bit-identical to torch's F.max_pool2d.

Covers the model shapes (ResNet stem 3x3/s2/p1, U-Net 2x2/s2), odd sizes, ties (post-ReLU zeros:
the first maximum in scan order takes the gradient), NaN propagation, bf16 and fp32, the
vectorised (C % 8) and scalar (odd C / misaligned) kernels.
"""
import pytest
import torch
import torch.nn.functional as F

from paper_2110_12484_b200 import pool as K6

pytestmark = pytest.mark.gpu

CASES = [((4, 64, 112, 112), 3, 2, 1), ((3, 64, 48, 48), 2, 2, 0), ((2, 24, 17, 13), 3, 2, 1),
         ((2, 8, 9, 9), 3, 1, 1), ((2, 5, 11, 7), 2, 2, 0), ((1, 16, 7, 7), 3, 3, 0), ((2, 32, 10, 10), 5, 2, 2),
         ((2, 16, 15, 14), 3, 2, 0), ((2, 8, 8, 9), 3, 2, 1), ((2, 40, 3, 3), 3, 2, 1)]


def _pair(x, k, s, p, dy):
    xa = x.detach().clone().requires_grad_(True)
    ya = F.max_pool2d(xa, k, s, p)
    ya.backward(dy)
    xb = x.detach().clone().requires_grad_(True)
    yb = K6.max_pool2d(xb, k, s, p)
    yb.backward(dy)
    return ya, xa.grad, yb, xb.grad


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("case", CASES)
def test_k6_bit_identical_to_torch(cuda, dtype, case):
    shape, k, s, p = case
    g = torch.Generator(device=cuda).manual_seed(sum(shape) + k)
    x = torch.randn(shape, device=cuda, generator=g)
    x = torch.relu(x - 0.3).to(dtype)                      # many exact zeros: ties
    x = x.contiguous(memory_format=torch.channels_last)
    n, c, h, w = shape
    ho, wo = (h + 2 * p - k) // s + 1, (w + 2 * p - k) // s + 1
    dy = torch.randn((n, c, ho, wo), device=cuda, generator=g).to(dtype).contiguous(memory_format=torch.channels_last)
    ya, ga, yb, gb = _pair(x, k, s, p, dy)
    assert yb.is_contiguous(memory_format=torch.channels_last)
    assert torch.equal(ya, yb)
    assert torch.equal(ga, gb)


def test_k6_nan_propagates_like_torch(cuda):
    x = torch.randn(2, 8, 8, 8, device=cuda).contiguous(memory_format=torch.channels_last)
    x[0, 3, 2, 5] = float("nan")
    x[1, 0, 7, 7] = float("nan")
    dy = torch.randn(2, 8, 4, 4, device=cuda).contiguous(memory_format=torch.channels_last)
    ya, ga, yb, gb = _pair(x, 3, 2, 1, dy)
    assert torch.equal(torch.isnan(ya), torch.isnan(yb))
    assert torch.equal(torch.nan_to_num(ya), torch.nan_to_num(yb))
    assert torch.equal(ga, gb)


def test_k6_nchw_input_and_misaligned(cuda):
    x = torch.randn(2, 16, 12, 12, device=cuda)                 # NCHW-contiguous: converted
    dy = torch.randn(2, 16, 6, 6, device=cuda)
    ya, ga, yb, gb = _pair(x, 2, 2, 0, dy)
    assert torch.equal(ya, yb) and torch.equal(ga, gb)
    base = torch.randn(2 * 12 * 12 * 16 + 1, device=cuda)
    xm = base[1:].view(2, 12, 12, 16).permute(0, 3, 1, 2)     # channels-last strides, 4-byte offset
    ya, ga, yb, gb = _pair(xm, 3, 2, 1, torch.randn(2, 16, 6, 6, device=cuda))
    assert torch.equal(ya, yb) and torch.equal(ga, gb)


def test_swapped_models_match_torch(cuda):
    import copy
    import torchvision
    from paper_2110_12484_b200.workloads import UNet
    for net, shape in ((torchvision.models.resnet18(num_classes=4), (2, 3, 64, 64)), (UNet(3, 1), (2, 3, 32, 32))):
        net = net.to(cuda).to(memory_format=torch.channels_last).eval()
        sw = K6.swap_maxpool(copy.deepcopy(net))
        assert any(isinstance(m, K6.MicroMaxPool2d) for m in sw.modules())
        x = torch.randn(shape, device=cuda).contiguous(memory_format=torch.channels_last)
        with torch.no_grad():
            assert torch.equal(net(x), sw(x))


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_pool_and_stash_join_equal_cat(cuda, dtype):
    """pool_and_stash + join_skip == (max_pool2d(s), cat([s, up])), gradients included (fp32: bit-exact)."""
    g = torch.Generator(device=cuda).manual_seed(11)
    s = torch.randn(2, 16, 12, 8, device=cuda, generator=g).to(dtype).contiguous(memory_format=torch.channels_last)
    up = torch.randn(2, 16, 12, 8, device=cuda, generator=g).to(dtype).contiguous(memory_format=torch.channels_last)
    w_p = torch.randn(2, 16, 6, 4, device=cuda, generator=g).to(dtype)
    w_c = torch.randn(2, 32, 12, 8, device=cuda, generator=g).to(dtype)

    def run(native):
        sa = s.detach().clone().requires_grad_(True)
        ua = up.detach().clone().requires_grad_(True)
        if native:
            p, buf = K6.pool_and_stash(sa, 2, 16)
            c = K6.join_skip(buf, ua)
        else:
            p, c = F.max_pool2d(sa, 2), torch.cat([sa, ua], 1)
        ((p.float() * w_p.float()).sum() + (c.float() * w_c.float()).sum()).backward()
        return p.detach(), c.detach(), sa.grad, ua.grad

    a, b = run(False), run(True)
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1]) and torch.equal(a[3], b[3])
    if dtype == torch.float32:
        assert torch.equal(a[2], b[2])
    else:   # ours sums the two skip gradients in fp32 and rounds once (torch rounds twice)
        assert (a[2].float() - b[2].float()).abs().max() <= 2 ** -7 * a[2].float().abs().max()


def test_unet_native_skips_match_plain(cuda):
    import copy
    from paper_2110_12484_b200.workloads import UNet
    torch.manual_seed(0)
    net = UNet(3, 1).to(cuda).to(memory_format=torch.channels_last).train()
    nat = copy.deepcopy(net)
    nat.native_skips = True
    x = torch.randn(2, 3, 32, 32, device=cuda).contiguous(memory_format=torch.channels_last)
    outs = []
    for m in (net, nat):
        out = m(x)
        (out ** 2).mean().backward()
        outs.append((out.detach(), [p.grad.clone() for p in m.parameters()]))
    assert torch.allclose(outs[0][0], outs[1][0], rtol=1e-5, atol=1e-6)
    for ga, gb in zip(outs[0][1], outs[1][1]):
        assert torch.allclose(ga, gb, rtol=1e-4, atol=1e-6)


@pytest.mark.parametrize("case", [((4, 64, 112, 112), 3, 2, 1), ((2, 24, 17, 13), 3, 2, 1), ((3, 64, 48, 48), 2, 2, 0),
                                  ((2, 8, 9, 9), 3, 1, 1), ((2, 5, 11, 7), 2, 2, 0)])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_k6_dual_output_bit_identical_to_summed_gradient(cuda, case, dtype):
    """Dual output (the pooled activation feeds two consumers): K6 adds the two gradients per window and
    rounds the sum to the activation dtype before the gather — exactly torch's (dy1 + dy2) then gather,
    so dx is bit-identical in fp32 and bf16; one unused handle (gradient None) is the single-output
    backward."""
    shape, k, s, p = case
    x = torch.randn(shape, device=cuda).to(dtype).contiguous(memory_format=torch.channels_last)
    xa = x.clone().requires_grad_(True)
    y1, y2 = K6.max_pool2d(xa, k, s, p, dual=True)
    g1, g2 = torch.randn_like(y1), torch.randn_like(y1)
    torch.autograd.backward([y1, y2], [g1, g2])
    xb = x.clone().requires_grad_(True)
    F.max_pool2d(xb, k, s, p).backward(g1 + g2)
    assert torch.equal(xa.grad, xb.grad)
    xc = x.clone().requires_grad_(True)
    _, y2 = K6.max_pool2d(xc, k, s, p, dual=True)
    y2.backward(g2)
    xd = x.clone().requires_grad_(True)
    F.max_pool2d(xd, k, s, p).backward(g2)
    assert torch.equal(xc.grad, xd.grad)
