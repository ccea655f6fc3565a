"""Micro-batch BatchNorm on sm_100a (K5, ``csrc/mbs_bn.cu``), fused with its ReLU / residual add.

Every micro-batch forward of the benchmark models normalises with statistics of
that MICRO-batch (reference ``nn.py:275-282`` BatchNorm2d.forward: the reason MBS
keeps micro-batch membership) and updates the running statistics once per
micro-batch (``nn.py:329-332``; torch's convention: unbiased ``running_var``,
``momentum`` 0.1, ``num_batches_tracked``). Measured on B200 (``profiles/``):
torch's bf16 channels-last BatchNorm kernels were 58 % of a ResNet-50 micro-batch
step at ~1 TB/s; this module replaces them with HBM-streaming kernels and folds
the following ReLU (and, in residual blocks, the skip add) into the same passes.
The convolutions stay on cuDNN.

``fuse_batchnorm(model)`` rewrites a model IN PLACE without touching its
parameters, buffers or their names/order (so ``ParameterSet`` layouts, state
dicts and the oracle's parameter mapping are unchanged):

* every ``nn.BatchNorm2d`` becomes a :class:`MicroBatchNorm2d` (same object,
  class swapped);
* ``nn.Sequential`` runs ``[BatchNorm2d, ReLU]`` fuse (the ReLU becomes ``Identity``);
* torchvision ResNet stems and ``BasicBlock`` / ``Bottleneck`` blocks fuse
  ``bn -> relu`` and ``bn3 (+ identity) -> relu``.

Training mode on CUDA always runs the native kernels (no torch fallback; a
missing ``libmbs_native.so`` raises). Eval mode with running statistics is
plain inference normalisation (torch ops), outside the MBS training path.
"""

from __future__ import annotations

import ctypes
import os

import torch
import torch.nn.functional as F
from torch import nn

from . import _native
from .prof import TIMER

_DTYPES = {torch.bfloat16: _native.BF16, torch.float32: _native.F32}
_WS_CACHE: dict = {}


def _ptr(t):
    return None if t is None else t.data_ptr()


def _workspace(rows: int, C: int, code: int, device) -> torch.Tensor:
    key = (rows, C, code)
    nbytes = _WS_CACHE.get(key)
    if nbytes is None:
        out = ctypes.c_int64()
        _native.check(_native.lib().mbs_bn_workspace_bytes(rows, C, code, ctypes.byref(out)), "mbs_bn_workspace_bytes")
        nbytes = _WS_CACHE[key] = out.value
    return torch.empty(nbytes, dtype=torch.uint8, device=device)


def _n_kernels(C: int, tensors, nbytes: int) -> int:
    """Kernels one K5 call launches (mirrors mbs_bn.cu): 1 on the cooperative path for layers
    <= MBS_K5_FUSED_MB (default 0: off) with 16-byte channel vectors, else 3. Used for launch counts."""
    v = 16 // tensors[0].element_size()
    if os.environ.get("MBS_K5_FUSED", "1") == "0" or C % v or C // v > 256:
        return 3
    if any(t is not None and t.data_ptr() % 16 for t in tensors):
        return 3
    limit = int(os.environ.get("MBS_K5_FUSED_MB", "0")) << 20
    return 1 if nbytes <= limit else 3


def _dual_ok(C: int, tensors, relu_res: bool) -> bool:
    """Whether mbs_bn_backward takes a second output gradient (mirrors its dy2 contract in include/mbs.h):
    the fused residual path with 16-byte channel vectors, <= 256 of them, every pointer 16-byte aligned."""
    v = 16 // tensors[0].element_size()
    return (relu_res and C % v == 0 and C // v <= 256
            and all(t is None or t.data_ptr() % 16 == 0 for t in tensors))


def _channels_last(t: torch.Tensor) -> torch.Tensor:
    if t.dim() == 4:
        return t.contiguous(memory_format=torch.channels_last)
    return t.contiguous()


def _geometry(x: torch.Tensor):
    if x.dim() == 4:
        n, c, h, w = x.shape
        return n * h * w, c
    if x.dim() == 2:
        return x.shape[0], x.shape[1]
    raise ValueError(f"micro-batch BatchNorm expects (N, C) or (N, C, H, W), got {tuple(x.shape)}")


class _MicroBatchNormFn(torch.autograd.Function):
    """y = relu?(bn(x) [+ residual]) with micro-batch statistics; one running-stat update."""

    @staticmethod
    def forward(ctx, x, residual, weight, bias, running_mean, running_var, momentum, eps, relu, dual=False,
                num_batches_tracked=None):
        code = _DTYPES.get(x.dtype)
        if code is None:
            raise ValueError(f"micro-batch BatchNorm supports bfloat16 / float32 activations, got {x.dtype}")
        x = _channels_last(x)
        if residual is not None:
            residual = _channels_last(residual.to(x.dtype))
            if residual.shape != x.shape:
                raise ValueError(f"residual shape {tuple(residual.shape)} != {tuple(x.shape)}")
        rows, C = _geometry(x)
        # rows == 1 (one value per channel, e.g. a 1-sample tail micro-batch on a 1x1 map) is legal, as in the
        # reference (eps-guarded): x_hat = 0, y = beta, dx = 0, and the running variance takes the
        # biased (= reference, nn.py:329-332) variance 0. torch's BatchNorm raises here instead.
        y = torch.empty_like(x)
        mean = torch.empty(C, dtype=torch.float32, device=x.device)
        invstd = torch.empty_like(mean)
        ws = _workspace(rows, C, code, x.device)
        stream = torch.cuda.current_stream(x.device)
        st = stream.cuda_stream
        ev = TIMER.start_k5(_n_kernels(C, (x, residual, y), x.numel() * x.element_size()), stream)
        _native.check(_native.lib().mbs_bn_forward(
            _ptr(x), _ptr(residual), _ptr(y), code, rows, C, _ptr(weight), _ptr(bias), _ptr(running_mean),
            _ptr(running_var), _ptr(num_batches_tracked), float(momentum), float(eps), int(relu), _ptr(mean),
            _ptr(invstd), _ptr(ws), st),
            "mbs_bn_forward")
        # algorithmic bytes: stats read x; apply read x (+ residual), write y
        TIMER.stop("k5_bn_forward", ev, x.numel() * x.element_size() * (3 + (residual is not None)), stream)
        ctx.save_for_backward(x, residual, weight, bias, mean, invstd)
        ctx.relu = bool(int(relu) & 1)          # relu is the C-ABI flag word (bit 1: biased running variance)
        ctx.code = code
        ctx.has_res = residual is not None
        if dual:
            # two handles on the same activation: the consumers' gradients reach backward separately
            # and are summed inside K5's reduce instead of by an autograd add pass
            ctx.set_materialize_grads(False)
            return y, y.view_as(y)
        return y

    @staticmethod
    def backward(ctx, dy, dy2=None):
        x, residual, weight, bias, mean, invstd = ctx.saved_tensors
        if dy is None:
            dy, dy2 = dy2, None
        dy = _channels_last(dy.to(x.dtype))
        rows, C = _geometry(x)
        if dy2 is not None:
            dy2 = _channels_last(dy2.to(x.dtype))
            if not _dual_ok(C, (x, residual, dy, dy2), ctx.relu and ctx.has_res):
                dy, dy2 = dy + dy2, None
        dx = torch.empty_like(x)
        dres = torch.empty_like(x) if ctx.has_res else None
        dw = torch.empty_like(weight) if weight is not None and ctx.needs_input_grad[2] else None
        db = torch.empty_like(bias) if bias is not None and ctx.needs_input_grad[3] else None
        ws = _workspace(rows, C, ctx.code, x.device)
        stream = torch.cuda.current_stream(x.device)
        st = stream.cuda_stream
        ev = TIMER.start_k5(3 if dy2 is not None else
                            _n_kernels(C, (x, residual, dy, dx, dres), x.numel() * x.element_size() * (2 + ctx.has_res)),
                            stream)
        _native.check(_native.lib().mbs_bn_backward(
            _ptr(x), _ptr(residual), _ptr(dy), _ptr(dy2), _ptr(dx), _ptr(dres), ctx.code, rows, C, _ptr(weight),
            _ptr(bias), _ptr(mean), _ptr(invstd), int(ctx.relu), _ptr(dw), _ptr(db), _ptr(ws), st), "mbs_bn_backward")
        # algorithmic bytes (two-pass minimum): reduce read x, dy (+ dy2) (+ residual, + write d_residual = g);
        # elemt read x and dy (or g), write dx
        TIMER.stop("k5_bn_backward", ev,
                   x.numel() * x.element_size() * (5 + 2 * ctx.has_res + (dy2 is not None)), stream)
        return dx, dres, dw, db, None, None, None, None, None, None, None


def micro_batch_norm(x, weight, bias, running_mean=None, running_var=None, *, momentum=0.1, eps=1e-5,
                     relu=False, residual=None, dual=False, biased_running_var=False):
    """Functional form: ``relu?(batch_norm(x, training=True) [+ residual])`` on the native kernels
    (``dual``: the output as two autograd handles, see ``MicroBatchNorm2d.forward``;
    ``biased_running_var``: the running variance takes the biased micro-batch variance, the reference's
    convention, nn.py:329-332, instead of torch's unbiased one)."""
    if residual is not None and not relu:
        raise ValueError("a residual is only fused together with the ReLU")
    flags = (1 if relu else 0) | (2 if biased_running_var else 0)
    return _MicroBatchNormFn.apply(x, residual, weight, bias, running_mean, running_var, momentum, eps, flags, dual)


class MicroBatchNorm2d(nn.BatchNorm2d):
    """``nn.BatchNorm2d`` whose training forward is K5, optionally fused with ReLU / a residual add.

    ``forward(x, residual=None)`` = ``relu(bn(x) + residual)`` when ``fuse_relu``
    (``bn(x)`` [+ relu] otherwise). Parameters, buffers and state-dict keys are
    those of ``nn.BatchNorm2d``.
    """

    fuse_relu: bool = False

    def __init__(self, *args, fuse_relu: bool = False, **kw):
        super().__init__(*args, **kw)
        self.fuse_relu = fuse_relu

    def extra_repr(self):
        return super().extra_repr() + f", fuse_relu={self.fuse_relu}"

    def forward(self, x, residual=None, dual: bool = False):
        """``dual``: return the output twice (``(y, y)``, two autograd handles) for an activation with two
        consumers, so their gradients are summed inside the backward kernel."""
        batch_stats = self.training or not self.track_running_stats
        if not batch_stats:                       # inference normalisation with running statistics
            y = F.batch_norm(x, self.running_mean, self.running_var, self.weight, self.bias, False, 0.0, self.eps)
            if residual is not None:
                y = y + residual
            y = F.relu(y) if self.fuse_relu else y
            return (y, y) if dual else y
        if not x.is_cuda:
            raise RuntimeError("MicroBatchNorm2d: training-mode normalisation runs on the sm_100a kernels "
                               "(libmbs_native.so) and needs a CUDA tensor; there is no CPU fallback")
        momentum = 0.0 if self.momentum is None else self.momentum
        track = self.training and self.track_running_stats
        nbt = None
        if track:
            if self.momentum is None:              # cumulative moving average (torch semantics): needs the count
                self.num_batches_tracked.add_(1)
                momentum = 1.0 / float(self.num_batches_tracked)
            elif self.num_batches_tracked.dtype == torch.int64 and self.num_batches_tracked.is_cuda:
                nbt = self.num_batches_tracked     # += 1 inside K5's statistics finalize (no counter kernel)
            else:
                self.num_batches_tracked.add_(1)
        if residual is not None and not self.fuse_relu:
            raise ValueError("MicroBatchNorm2d: a residual needs fuse_relu=True")
        return _MicroBatchNormFn.apply(x, residual, self.weight, self.bias,
                                       self.running_mean if track else None,
                                       self.running_var if track else None,
                                       momentum, self.eps, self.fuse_relu, dual, nbt)


def _as_micro_bn(bn: nn.BatchNorm2d, relu: bool) -> MicroBatchNorm2d:
    bn.__class__ = MicroBatchNorm2d
    bn.fuse_relu = relu
    return bn


def _bottleneck_pair(self, xm, xr, dual):
    """Block on (main, skip) handles of the same input; returns the output (twice when ``dual``)."""
    identity = xr if self.downsample is None else self.downsample(xr)
    out = self.bn1(self.conv1(xm))
    out = self.bn2(self.conv2(out))
    return self.bn3(self.conv3(out), identity, dual=dual)


def _basic_pair(self, xm, xr, dual):
    identity = xr if self.downsample is None else self.downsample(xr)
    out = self.bn1(self.conv1(xm))
    return self.bn2(self.conv2(out), identity, dual=dual)


def _bottleneck_forward(self, x):
    return _bottleneck_pair(self, x, x, False)


def _basic_forward(self, x):
    return _basic_pair(self, x, x, False)


class _GlobalAvgPoolFn(torch.autograd.Function):
    """adaptive_avg_pool2d(x, 1).flatten(1) whose gradient is produced channels-last directly (one
    broadcast write) — torch's returns it NCHW-contiguous and K5's backward of the last block then paid
    a strided layout copy (ncu r01_c2_v7: 42 us + 23 us per ResNet-50 micro-batch)."""

    @staticmethod
    def forward(ctx, x):
        n, c, h, w = x.shape
        ctx.shape = (n, c, h, w)
        return x.mean((2, 3))

    @staticmethod
    def backward(ctx, dy):
        n, c, h, w = ctx.shape
        g = dy / (h * w)
        return g[:, None, None, :].expand(n, h, w, c).contiguous().permute(0, 3, 1, 2)


def _global_pool(self, x):
    ap = self.avgpool
    if isinstance(ap, nn.AdaptiveAvgPool2d) and ap.output_size in (1, (1, 1)) and x.dim() == 4 \
            and x.is_contiguous(memory_format=torch.channels_last):
        return _GlobalAvgPoolFn.apply(x)
    return torch.flatten(ap(x), 1)


def _resnet_forward(self, x):
    """torchvision ResNet._forward_impl with every block output but the last handed on as two autograd
    handles (next block's conv1 and its skip / downsample): the gradient sum of the two consumers
    happens in K5's backward reduce of the producing block (mbs_bn_backward dy2), not in an autograd add."""
    x = self.relu(self.bn1(self.conv1(x)))
    blocks = [b for layer in (self.layer1, self.layer2, self.layer3, self.layer4) for b in layer]
    from .pool import MicroMaxPool2d
    if isinstance(self.maxpool, MicroMaxPool2d) and x.is_cuda:
        xm, xr = self.maxpool(x, dual=True)    # K6 sums the first block's two input gradients
    else:
        xm = xr = self.maxpool(x)
    for i, blk in enumerate(blocks):
        dual = i + 1 < len(blocks) and isinstance(blk, (FusedBottleneck, FusedBasicBlock))
        if isinstance(blk, (FusedBottleneck, FusedBasicBlock)):
            out = blk.forward_pair(xm, xr, dual)
        else:
            out = blk(xm)
        xm, xr = out if dual else (out, out)
    return self.fc(_global_pool(self, xm))


try:
    from torchvision.models import resnet as tv_resnet

    class FusedBottleneck(tv_resnet.Bottleneck):
        """torchvision Bottleneck with bn1/bn2 -> relu and bn3 + identity -> relu on K5."""
        forward = _bottleneck_forward
        forward_pair = _bottleneck_pair

    class FusedBasicBlock(tv_resnet.BasicBlock):
        """torchvision BasicBlock with bn1 -> relu and bn2 + identity -> relu on K5."""
        forward = _basic_forward
        forward_pair = _basic_pair

    class FusedResNet(tv_resnet.ResNet):
        """torchvision ResNet whose block outputs reach the next block as two handles (dual K5 output)."""
        _forward_impl = _resnet_forward
except ImportError:  # pragma: no cover - torchvision is in the image
    tv_resnet = None


def fuse_batchnorm(model: nn.Module) -> nn.Module:
    """Route a model's BatchNorm through K5 with ReLU / residual fusion (in place; returns the model)."""
    for mod in list(model.modules()):
        if tv_resnet is not None and type(mod) is tv_resnet.Bottleneck:
            _as_micro_bn(mod.bn1, True)
            _as_micro_bn(mod.bn2, True)
            _as_micro_bn(mod.bn3, True)
            mod.__class__ = FusedBottleneck
        elif tv_resnet is not None and type(mod) is tv_resnet.BasicBlock:
            _as_micro_bn(mod.bn1, True)
            _as_micro_bn(mod.bn2, True)
            mod.__class__ = FusedBasicBlock
        elif tv_resnet is not None and type(mod) is tv_resnet.ResNet:
            _as_micro_bn(mod.bn1, True)
            mod.relu = nn.Identity()           # the stem's ReLU (blocks own their own relu modules)
            if os.environ.get("MBS_K5_DUAL", "1") != "0":   # A/B: MBS_K5_DUAL=0 keeps autograd's adds
                mod.__class__ = FusedResNet
        elif isinstance(mod, nn.Sequential):
            kids = list(mod._modules.items())
            for i, (name, child) in enumerate(kids):
                if type(child) is nn.BatchNorm2d:
                    nxt = kids[i + 1][1] if i + 1 < len(kids) else None
                    relu = isinstance(nxt, nn.ReLU)
                    _as_micro_bn(child, relu)
                    if relu:
                        mod._modules[kids[i + 1][0]] = nn.Identity()
    for mod in model.modules():                # any BatchNorm2d not covered by a pattern above
        if type(mod) is nn.BatchNorm2d:
            _as_micro_bn(mod, False)
    return model
