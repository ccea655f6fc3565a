"""Paper-style parity: training WITH MBS reaches the accuracy / IoU of
training WITHOUT it on the same data, epochs and hyper-parameters.

The paper reports ResNet-50 87.16 % vs 87.04 % and U-Net IoU 95.48 vs 95.45 at mini-batch 16. Here: synthetic
but learnable tasks (there is no dataset network access), the benchmarked stack (native model ops, bf16
shadow weights + autocast, uint8 inputs staged by K2, CUDA graphs), ``train_epoch`` with ``metric_fn``;
micro-batch 8 (resp. 4) streamed vs the whole mini-batch at once (``micro_batch_size=None``, the
reference's no-MBS baseline, engine.py:313). Held-out accuracy / IoU in eval mode (BatchNorm running
statistics, which MBS accumulates per micro-batch exactly like the reference, nn.py:329-332).
"""
import copy

import pytest
import torch

import paper_2110_12484_b200 as mbs
from paper_2110_12484_b200 import graphs
from paper_2110_12484_b200.streamer import Staging
from paper_2110_12484_b200.workloads import WORKLOADS, UNet, build_model, make_native

pytestmark = pytest.mark.gpu


def _classes(n, seed):
    """10 classes: a class-specific 4x4 colour pattern, upsampled to 32x32, under uint8 noise."""
    g = torch.Generator().manual_seed(seed)
    proto = torch.rand((10, 3, 4, 4), generator=torch.Generator().manual_seed(123)) * 160 + 40
    y = torch.randint(0, 10, (n,), generator=g)
    img = torch.nn.functional.interpolate(proto[y], size=(32, 32), mode="nearest")
    img = img + torch.randn(img.shape, generator=g) * 110      # heavy noise: held-out accuracy well below 100 %
    return img.clamp(0, 255).to(torch.uint8), y


def _shapes(n, seed, s=64):
    """Binary masks of a random disc; the image is the mask brightened under uint8 noise."""
    g = torch.Generator().manual_seed(seed)
    yy, xx = torch.meshgrid(torch.arange(s), torch.arange(s), indexing="ij")
    c = torch.rand((n, 2), generator=g) * s * 0.6 + s * 0.2
    r = torch.rand((n,), generator=g) * s * 0.2 + s * 0.1
    m = ((yy[None] - c[:, 0, None, None]) ** 2 + (xx[None] - c[:, 1, None, None]) ** 2 < r[:, None, None] ** 2)
    img = 60 + 60 * m[:, None].float().expand(n, 3, s, s) + torch.randn((n, 3, s, s), generator=g) * 90
    return img.clamp(0, 255).to(torch.uint8), m[:, None].to(torch.uint8)


def _train(cuda, net0, x, y, loss_kind, opt, mini, micro, epochs, metric):
    graphs.clear()
    net = copy.deepcopy(net0)
    params = mbs.ParameterSet(net, shadow=torch.bfloat16)
    st = mbs.sgd_state(0.05, 0.9, 5e-4) if opt == "sgd" else mbs.adam_state(1e-3, 5e-4)
    staging = Staging(torch.bfloat16, True, target_dtype=torch.float32)
    for e in range(epochs):
        es = mbs.train_epoch(net, params, x, y, mini_batch_size=mini, micro_batch_size=micro,
                             normalization="exact_weighted", loss_kind=loss_kind, optimizer_state=st, seed=0,
                             epoch_index=e, staging=staging, autocast_dtype=torch.bfloat16, metric_fn=metric)
    graphs.clear()
    return net, es


@torch.no_grad()
def _eval(net, x, y, fn):
    net.eval()
    with torch.autocast("cuda", dtype=torch.bfloat16):      # the bf16 shadow weights, as in training
        out = net(x.float().contiguous(memory_format=torch.channels_last))
    net.train()
    return fn(out.float(), y)


def test_resnet18_accuracy_with_and_without_mbs(cuda):
    torch.manual_seed(0)
    net0 = build_model(WORKLOADS["c1"], ops="native").to(cuda).to(memory_format=torch.channels_last)
    x, y = _classes(2048, 1)
    xt, yt = _classes(512, 2)
    xt, yt = xt.to(cuda), yt.to(cuda)
    acc = {}
    for micro in (8, None):                                   # MBS (N_Smu = 8) vs no MBS
        net, es = _train(cuda, net0, x.to(cuda), y.to(cuda), "cross_entropy", "sgd", 64, micro, 3, mbs.accuracy)
        acc[micro] = (_eval(net, xt, yt, mbs.accuracy), es.mini_metrics[-1])
    print("held-out accuracy: MBS(micro 8) %.4f  no-MBS %.4f" % (acc[8][0], acc[None][0]))
    assert acc[None][0] >= 0.5, "the no-MBS baseline did not learn the task"
    assert abs(acc[8][0] - acc[None][0]) <= 0.05


def test_unet_iou_with_and_without_mbs(cuda):
    torch.manual_seed(0)
    net0 = make_native(UNet(3, 1)).to(cuda).to(memory_format=torch.channels_last)
    x, y = _shapes(384, 3)
    xt, yt = _shapes(96, 4)
    xt, yt = xt.to(cuda), yt.to(cuda)

    def iou(o, t):
        return mbs.iou(torch.sigmoid(o), t)
    res = {}
    for micro in (4, None):
        net, es = _train(cuda, net0, x.to(cuda), y.to(cuda), "bce_dice", "adam", 16, micro, 4, iou)
        res[micro] = _eval(net, xt, yt, iou)
    print("held-out IoU: MBS(micro 4) %.4f  no-MBS %.4f" % (res[4], res[None]))
    assert res[None] >= 0.5, "the no-MBS baseline did not learn the task"
    assert abs(res[4] - res[None]) <= 0.05
