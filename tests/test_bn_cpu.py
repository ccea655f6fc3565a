"""K5 module rewrite on a CPU host: structure, names and the no-fallback rule (no kernel calls)."""
import copy

import pytest
import torch
import torchvision

from paper_2110_12484_b200 import bn as K5
from paper_2110_12484_b200.workloads import UNet


@pytest.mark.parametrize("make", [lambda: torchvision.models.resnet18(num_classes=10),
                                  lambda: torchvision.models.resnet50(num_classes=102), lambda: UNet(3, 1)])
def test_fuse_keeps_parameters_buffers_and_order(make):
    torch.manual_seed(0)
    net = make()
    ref = copy.deepcopy(net)
    params = [id(p) for p in net.parameters()]
    K5.fuse_batchnorm(net)
    assert [id(p) for p in net.parameters()] == params            # same Parameter objects: ParameterSet-safe
    assert list(net.state_dict()) == list(ref.state_dict())
    n_bn = sum(isinstance(m, torch.nn.BatchNorm2d) for m in ref.modules())
    mbn = [m for m in net.modules() if isinstance(m, K5.MicroBatchNorm2d)]
    assert len(mbn) == n_bn
    assert not any(type(m) is torch.nn.BatchNorm2d for m in net.modules())
    assert not any(isinstance(m, torch.nn.ReLU) for m in net.modules()) or isinstance(net, torchvision.models.ResNet)
    # eval-mode inference is torch's running-statistics normalisation: identical outputs on CPU
    net.eval()
    ref.eval()
    x = torch.randn(2, 3, 32, 32)
    with torch.no_grad():
        torch.testing.assert_close(net(x), ref(x), rtol=1e-5, atol=1e-6)


def test_fused_relu_counts_resnet50():
    net = K5.fuse_batchnorm(torchvision.models.resnet50())
    mbn = [m for m in net.modules() if isinstance(m, K5.MicroBatchNorm2d)]
    # stem + 16 blocks x 3 fused with relu; 4 downsample BNs plain
    assert sum(m.fuse_relu for m in mbn) == 1 + 16 * 3
    assert sum(not m.fuse_relu for m in mbn) == 4


def test_training_on_cpu_fails_loudly():
    net = K5.fuse_batchnorm(torchvision.models.resnet18(num_classes=10)).train()
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        net(torch.randn(2, 3, 32, 32))


def test_residual_requires_fused_relu():
    m = K5.MicroBatchNorm2d(4)
    with pytest.raises(ValueError):
        K5.micro_batch_norm(torch.randn(2, 4), m.weight, m.bias, residual=torch.randn(2, 4))


def test_swap_maxpool_supported_configs():
    from paper_2110_12484_b200 import pool as K6
    m = torch.nn.Sequential(torch.nn.MaxPool2d(3, 2, 1), torch.nn.MaxPool2d(2), torch.nn.MaxPool2d(3, 2, 1, ceil_mode=True),
                            torch.nn.MaxPool2d(3, 2, 1, dilation=2), torch.nn.MaxPool2d((3, 2)))
    K6.swap_maxpool(m)
    kinds = [type(x).__name__ for x in m]
    assert kinds == ["MicroMaxPool2d", "MicroMaxPool2d", "MaxPool2d", "MaxPool2d", "MaxPool2d"]
    x = torch.randn(2, 4, 9, 9)
    with pytest.raises(RuntimeError, match="no CPU fallback"):                       # training: K6 only
        m[0](x)
    m.eval()
    torch.testing.assert_close(m[0](x), torch.nn.functional.max_pool2d(x, 3, 2, 1))   # CPU eval: torch path


def test_stem_training_on_cpu_fails_loudly():
    from paper_2110_12484_b200 import stem as K7
    m = K7.swap_stem(torch.nn.Sequential(torch.nn.Conv2d(3, 8, 7, 2, 3)))
    assert type(m[0]).__name__ == "StemConv2d"
    x = torch.randn(2, 3, 16, 16)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        m(x)
    m.eval()
    ref = torch.nn.functional.conv2d(x, m[0].weight, m[0].bias, 2, 3)
    torch.testing.assert_close(m(x), ref)


def test_build_model_native_ops():
    from paper_2110_12484_b200.workloads import WORKLOADS, build_model
    from paper_2110_12484_b200 import pool as K6
    a = build_model(WORKLOADS["c2"], ops="native")
    b = build_model(WORKLOADS["c2"], ops="torch")
    assert list(a.state_dict()) == list(b.state_dict())
    assert isinstance(a.maxpool, K6.MicroMaxPool2d)
    with pytest.raises(ValueError):
        build_model(WORKLOADS["c2"], ops="k5")
