"""Property tests (hypothesis, derandomized) of the model-side kernels over random geometries:
K6 max-pool bit-identical to torch (forward and backward, bf16 and fp32), K5 micro-batch BatchNorm
(+ReLU/+residual) within fp32 rounding of a float64 reference, K7 stem conv vs float64 conv2d."""
import pytest
import torch
import torch.nn.functional as F
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

from paper_2110_12484_b200 import bn as K5
from paper_2110_12484_b200 import pool as K6
from paper_2110_12484_b200 import stem as K7
from tests.gpu_util import rel_l2

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")
SETTINGS = settings(max_examples=25, deadline=None, derandomize=True,
                    suppress_health_check=[HealthCheck.too_slow, HealthCheck.function_scoped_fixture])


@SETTINGS
@given(n=st.integers(1, 3), c=st.sampled_from([1, 3, 8, 16, 24, 64]), h=st.integers(2, 19), w=st.integers(2, 19),
       k=st.integers(1, 4), s=st.integers(1, 3), p=st.integers(0, 2),
       bf16=st.booleans(), relu=st.booleans(), seed=st.integers(0, 10_000))
def test_k6_random_geometry_bit_identical(n, c, h, w, k, s, p, bf16, relu, seed):
    if 2 * p > k or h + 2 * p < k or w + 2 * p < k:
        return
    g = torch.Generator(device=DEV).manual_seed(seed)
    x = torch.randn(n, c, h, w, device=DEV, generator=g)
    if relu:
        x = torch.relu(x)                                   # exact ties
    x = x.to(torch.bfloat16 if bf16 else torch.float32).contiguous(memory_format=torch.channels_last)
    ya_in = x.detach().clone().requires_grad_(True)
    yb_in = x.detach().clone().requires_grad_(True)
    ya = F.max_pool2d(ya_in, k, s, p)
    yb = K6.max_pool2d(yb_in, k, s, p)
    assert torch.equal(ya, yb)
    dy = torch.randn(ya.shape, device=DEV, generator=g).to(x.dtype)
    ya.backward(dy)
    yb.backward(dy)
    assert torch.equal(ya_in.grad, yb_in.grad)


@SETTINGS
@given(n=st.integers(2, 5), c=st.sampled_from([4, 8, 12, 64, 136]), h=st.integers(1, 9), w=st.integers(1, 9),
       relu=st.booleans(), res=st.booleans(), offset=st.floats(-4, 4), seed=st.integers(0, 10_000))
def test_k5_random_geometry_fp32(n, c, h, w, relu, res, offset, seed):
    """Against float64; the bound is max(2e-5, 2 x torch's own fp32 error) — with a handful of values
    per channel (n*h*w small) BatchNorm's input gradient is an ill-conditioned cancellation."""
    res = res and relu
    g = torch.Generator(device=DEV).manual_seed(seed)
    x = (torch.randn(n, c, h, w, device=DEV, generator=g) * 1.5 + offset).contiguous(memory_format=torch.channels_last)
    r = torch.randn(n, c, h, w, device=DEV, generator=g).contiguous(memory_format=torch.channels_last) if res else None
    wt = torch.randn(c, device=DEV, generator=g)
    bs = torch.randn(c, device=DEV, generator=g)
    dy = torch.randn(n, c, h, w, device=DEV, generator=g).contiguous(memory_format=torch.channels_last)
    xs = x.detach().clone().requires_grad_(True)
    ws, bb = wt.detach().clone().requires_grad_(True), bs.detach().clone().requires_grad_(True)
    rs = None if r is None else r.detach().clone().requires_grad_(True)
    y = K5.micro_batch_norm(xs, ws, bb, relu=relu, residual=rs)
    y.backward(dy)
    x64 = x.double().requires_grad_(True)
    w64, b64 = wt.double().requires_grad_(True), bs.double().requires_grad_(True)
    r64 = None if r is None else r.double().requires_grad_(True)
    y64 = F.batch_norm(x64, None, None, w64, b64, True, 0.1, 1e-5)
    if r64 is not None:
        y64 = y64 + r64
    if relu:
        y64 = F.relu(y64)
    y64.backward(dy.double())
    xt = x.detach().clone().requires_grad_(True)
    wt32, bt32 = wt.detach().clone().requires_grad_(True), bs.detach().clone().requires_grad_(True)
    rt = None if r is None else r.detach().clone().requires_grad_(True)
    yt = F.batch_norm(xt, None, None, wt32, bt32, True, 0.1, 1e-5)
    if rt is not None:
        yt = yt + rt
    if relu:
        yt = F.relu(yt)
    yt.backward(dy)
    trip = ((y, yt, y64), (xs.grad, xt.grad, x64.grad), (ws.grad, wt32.grad, w64.grad), (bb.grad, bt32.grad, b64.grad))
    if res:
        trip += ((rs.grad, rt.grad, r64.grad),)
    for a, t, b in trip:
        bd = b.detach().cpu().numpy()
        if abs(bd).max() == 0:
            continue
        ours = rel_l2(a.detach().double().cpu().numpy(), bd)
        theirs = rel_l2(t.detach().double().cpu().numpy(), bd)
        assert ours <= max(2e-5, 2 * theirs), (ours, theirs)


@SETTINGS
@given(n=st.integers(1, 3), cin=st.integers(1, 4), o=st.sampled_from([8, 16, 64]), hw=st.integers(5, 21),
       k=st.sampled_from([1, 3, 5, 7]), s=st.integers(1, 2), bias=st.booleans(), seed=st.integers(0, 10_000))
def test_k7_random_geometry_fp32(n, cin, o, hw, k, s, bias, seed):
    p = k // 2
    torch.manual_seed(seed)
    conv = torch.nn.Conv2d(cin, o, k, s, p, bias=bias).to(DEV)
    ref = torch.nn.Conv2d(cin, o, k, s, p, bias=bias).to(DEV).double()
    ref.load_state_dict({kk: v.double() for kk, v in conv.state_dict().items()})
    K7.swap_stem(conv)
    x = torch.randn(n, cin, hw, hw, device=DEV).contiguous(memory_format=torch.channels_last)
    y, yr = conv(x), ref(x.double())
    dy = torch.randn_like(yr)
    y.backward(dy.float())
    yr.backward(dy)
    assert rel_l2(y.detach().double().cpu().numpy(), yr.detach().cpu().numpy()) <= 1e-6
    assert rel_l2(conv.weight.grad.double().cpu().numpy(), ref.weight.grad.cpu().numpy()) <= 1e-6
