"""Benchmark workloads named by BASELINE.json ``configs`` (synthetic data, random init).

C1 ResNet-18 (10 classes) on CIFAR-shaped 3x32x32, mini 64 / micro 8.
C2 ResNet-50 (102 classes, Flower-102 shape) 3x224x224, mini 1024 / micro 128.
C3 U-Net (classic 64..1024, transpose-conv up path, 3 -> 1 channel) 3x384x384
   with binary masks, mini 256 / micro 48 (ragged tail of 16).
C5 U-Net 768x768, micro-batch auto-sized to free HBM (memory.fit_micro_batch).

These are the model definitions only; the MBS hot path never depends on them.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
from torch import nn


class _DoubleConv(nn.Module):
    def __init__(self, cin, cout):
        super().__init__()
        self.net = nn.Sequential(nn.Conv2d(cin, cout, 3, padding=1, bias=False), nn.BatchNorm2d(cout),
                                 nn.ReLU(inplace=True), nn.Conv2d(cout, cout, 3, padding=1, bias=False),
                                 nn.BatchNorm2d(cout), nn.ReLU(inplace=True))

    def forward(self, x):
        return self.net(x)


class _Up(nn.Module):
    def __init__(self, cin, cout):
        super().__init__()
        self.up = nn.ConvTranspose2d(cin, cin // 2, kernel_size=2, stride=2)
        self.conv = _DoubleConv(cin, cout)

    def forward(self, x, skip):
        return self.conv(torch.cat([skip, self.up(x)], dim=1))


class UNet(nn.Module):
    """Classic U-Net (Ronneberger et al.), 64->1024 channels, transpose-conv up path."""

    def __init__(self, in_channels: int = 3, out_channels: int = 1):
        super().__init__()
        self.inc = _DoubleConv(in_channels, 64)
        self.downs = nn.ModuleList([_DoubleConv(c, 2 * c) for c in (64, 128, 256, 512)])
        self.ups = nn.ModuleList([_Up(2 * c, c) for c in (512, 256, 128, 64)])
        self.pool = nn.MaxPool2d(2)
        self.outc = nn.Conv2d(64, out_channels, kernel_size=1)

    native_skips = False   # set by build_model(ops="native"): skips written into the concat buffers by K6

    def forward(self, x):
        if self.native_skips and x.is_cuda and x.shape[-2] % 16 == 0 and x.shape[-1] % 16 == 0:
            return self._forward_native(x)
        skips = [self.inc(x)]
        for d in self.downs:
            skips.append(d(self.pool(skips[-1])))
        x = skips.pop()
        for u in self.ups:
            x = u(x, skips.pop())
        return self.outc(x)

    def _forward_native(self, x):
        """Same math; each skip is copied into its decoder concat buffer by the pooling kernel, the
        upsampled half is joined in place, and the two gradients of a skip are summed inside the
        pooling backward (pool.pool_and_stash / join_skip) — no torch.cat pass, no separate add."""
        from .pool import join_skip, pool_and_stash
        h = self.inc(x)
        bufs = []
        for d in self.downs:
            pooled, buf = pool_and_stash(h, 2, h.shape[1])
            bufs.append(buf)
            h = d(pooled)
        for u in self.ups:
            up = torch.nn.functional.conv_transpose2d(h, u.up.weight, None, u.up.stride, u.up.padding)
            h = u.conv(join_skip(bufs.pop(), up, u.up.bias))   # bias added while joining
        return self.outc(h)


@dataclass(frozen=True)
class Workload:
    name: str
    model: str
    sample_shape: tuple
    target: str            # "classes" | "mask"
    n_classes: int
    mini: int
    micro: int
    loss_kind: str
    optimizer: str         # "sgd" | "adam"
    normalization: str = "exact_weighted"


WORKLOADS = {
    "c1": Workload("resnet18-cifar-64/8", "resnet18", (3, 32, 32), "classes", 10, 64, 8, "cross_entropy", "sgd"),
    "c2": Workload("resnet50-224-flower102-1024/128", "resnet50", (3, 224, 224), "classes", 102, 1024, 128,
                   "cross_entropy", "sgd"),
    "c3": Workload("unet-384-carvana-256/48", "unet", (3, 384, 384), "mask", 1, 256, 48, "bce_dice", "adam"),
    "c5": Workload("unet-768-autosized", "unet", (3, 768, 768), "mask", 1, 64, 0, "bce_dice", "adam"),
    # N1 (north_star Target): U-Net@384 with a mini-batch whose data exceeds HBM: 80,000 samples = 47.2 GB as
    # uint8 image + mask, 188.7 GB as the reference's float32 arrays; micro 48 -> 1,666 x 48 + a tail of 32
    "n1": Workload("unet-384-host-resident-80000/48", "unet", (3, 384, 384), "mask", 1, 80_000, 48, "bce_dice",
                   "adam"),
    # C4: one mini-batch per GPU of 300,032 = 2,344 x 128 samples: 45.2 GB host-resident as uint8
    # (180.6 GB as the reference's float32/float64 arrays would hold it: larger than the 180 GB HBM)
    "c4": Workload("resnet50-224-host-resident-300032/128", "resnet50", (3, 224, 224), "classes", 102, 300_032,
                   128, "cross_entropy", "sgd"),
}


def build_model(w: Workload, ops: str = "torch") -> nn.Module:
    """The workload's model. ``ops="native"`` runs its BatchNorm(+ReLU/+skip add) on K5 (bn.py), its
    max-pools on K6 (pool.py), its 3-channel stem conv as K7 im2col + cuBLAS GEMM and a 1x1 head
    conv with < 8 outputs as one GEMM (stem.py);
    ``"torch"`` is the stock module. Parameters are identical either way."""
    if w.model in ("resnet18", "resnet50"):
        import torchvision
        m = getattr(torchvision.models, w.model)(num_classes=w.n_classes)
    elif w.model == "unet":
        m = UNet(w.sample_shape[0], 1)
    else:
        raise ValueError(w.model)
    if ops == "native":
        make_native(m)
    elif ops != "torch":
        raise ValueError(f"ops must be 'native' or 'torch', got {ops!r}")
    return m


def make_native(m: nn.Module) -> nn.Module:
    """Route a stock model's BatchNorm(+ReLU/+skip add), max-pools, 3-channel stem conv and narrow 1x1
    head onto K5/K6/K7 in place (class swaps only: parameter names, order and values are unchanged,
    so the stock module and its native twin share one oracle)."""
    from .bn import fuse_batchnorm
    from .pool import swap_maxpool
    from .stem import swap_pointwise, swap_stem
    fuse_batchnorm(m)
    swap_maxpool(m)
    swap_stem(m)
    swap_pointwise(m)
    if isinstance(m, UNet):
        m.native_skips = True
    return m


def gflop_per_sample(w: Workload, device) -> float:
    """Algorithmic fwd+bwd GFLOP per sample of the workload's model (torch FlopCounterMode over the
    convolutions / matmuls of a 2-sample fp32 step; ResNet-50@224 24.29, U-Net@384 649.75)."""
    from torch.utils.flop_counter import FlopCounterMode
    m = build_model(w).to(device).to(memory_format=torch.channels_last).train()
    x = torch.randn((2,) + w.sample_shape, device=device).contiguous(memory_format=torch.channels_last)
    with FlopCounterMode(display=False) as fc:
        m(x).float().sum().backward()
    total = fc.get_total_flops()
    del m, x
    return total / 2 / 1e9


def synthetic_data(w: Workload, n: int, seed: int = 0, device="cpu", pinned: bool = False):
    """uint8 images and int64 labels / uint8 {0,1} masks (the datasets' natural storage; K2 stages
    both to the model's dtypes on device, ``Staging.target_dtype`` for masks).

    Large host datasets (> 4 GB) are allocated page-locked in place and filled by tiling 509
    random samples (memcpy speed) instead of per-byte RNG.
    """
    g = torch.Generator().manual_seed(seed)
    row = int(torch.tensor(w.sample_shape).prod())
    mask_shape = (1,) + tuple(w.sample_shape[1:])
    if str(device) == "cpu" and n * row > 4 * 2 ** 30:
        x = torch.empty((n,) + w.sample_shape, dtype=torch.uint8, pin_memory=pinned)
        base = torch.randint(0, 256, (509,) + w.sample_shape, generator=g, dtype=torch.uint8)
        for i in range(0, n, base.shape[0]):
            k = min(base.shape[0], n - i)
            x[i:i + k].copy_(base[:k])
        if w.target == "classes":
            y = torch.randint(0, w.n_classes, (n,), generator=g, dtype=torch.int64)
            return x, (y.pin_memory() if pinned else y)
        y = torch.empty((n,) + mask_shape, dtype=torch.uint8, pin_memory=pinned)
        mb = (torch.rand((509,) + mask_shape, generator=g) < 0.5).to(torch.uint8)
        for i in range(0, n, mb.shape[0]):
            k = min(mb.shape[0], n - i)
            y[i:i + k].copy_(mb[:k])
        return x, y
    x = torch.randint(0, 256, (n,) + w.sample_shape, generator=g, dtype=torch.uint8)
    if w.target == "classes":
        y = torch.randint(0, w.n_classes, (n,), generator=g, dtype=torch.int64)
    else:
        y = (torch.rand((n,) + mask_shape, generator=g) < 0.5).to(torch.uint8)
    if pinned:
        return x.pin_memory(), y.pin_memory()
    return x.to(device), y.to(device)
