"""The model's first convolution (3 input channels) as K7 im2col + one cuBLAS GEMM.

With C_in = 3 cuDNN has no sm_100 implicit-GEMM kernel for the stem: it runs sm80
kernels at ~37 TFLOP/s, 0.76 ms forward + 0.37 ms weight grad of the ResNet-50
micro-batch step (``profiles/r01_c2_v3_launches.md``; zero-padding to 8 input
channels is slower, ``tools/probe_stem.py``). K7 (``csrc/mbs_im2col.cu``) writes
the patch matrix ``cols[N*Ho*Wo, Kp]`` (K = kh*kw*C, ordered (kh, kw, c), padded
to a multiple of 8); the forward is ``cols @ W`` — whose [M, O] result IS the
channels-last activation — and the weight gradient ``cols^T @ dy``. Both GEMMs
are plain library GEMMs (cuBLAS). The input of a stem conv is data, so no input
gradient is needed (if one is requested it is computed by torch).

``swap_stem(model)`` swaps the class of every ``nn.Conv2d`` with at most 4 input
channels (groups 1, dilation 1, square kernel/stride/padding, zero padding) in
place; parameters and state dicts are unchanged.
"""

from __future__ import annotations

import torch
from torch import nn

from . import _native
from .prof import TIMER

_DTYPES = {torch.bfloat16: _native.BF16, torch.float32: _native.F32}


def _compute_dtype(x):
    if torch.is_autocast_enabled("cuda"):
        return torch.get_autocast_dtype("cuda")
    return x.dtype


class _StemConvFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, weight, bias, k, s, p):
        cdt = _compute_dtype(x)
        code = _DTYPES.get(cdt)
        if code is None:
            raise ValueError(f"stem conv computes in bfloat16 / float32, got {cdt}")
        x = x.to(cdt).contiguous(memory_format=torch.channels_last)
        n, c, h, w = x.shape
        o = weight.shape[0]
        ho, wo = (h + 2 * p - k) // s + 1, (w + 2 * p - k) // s + 1
        K = k * k * c
        kp = (K + 7) // 8 * 8
        m = n * ho * wo
        with torch.autocast("cuda", enabled=False):
            wm = torch.zeros((kp, o), dtype=cdt, device=x.device)
            wm[:K] = weight.to(cdt).permute(2, 3, 1, 0).reshape(K, o)
            cols = torch.empty((m, kp), dtype=cdt, device=x.device)
            stream = torch.cuda.current_stream(x.device)
            TIMER.launches += 1
            _native.check(_native.lib().mbs_im2col(x.data_ptr(), cols.data_ptr(), code, n, h, w, c, k, s, p, kp,
                                                   stream.cuda_stream), "mbs_im2col")
            y = torch.mm(cols, wm)
            if bias is not None:
                y += bias.to(cdt)
        ctx.save_for_backward(cols, weight, x if ctx.needs_input_grad[0] else None)
        ctx.geom = (n, c, h, w, o, ho, wo, k, s, p, K, bias is not None)
        return y.view(n, ho, wo, o).permute(0, 3, 1, 2)

    @staticmethod
    def backward(ctx, dy):
        cols, weight, x = ctx.saved_tensors
        n, c, h, w, o, ho, wo, k, s, p, K, has_bias = ctx.geom
        with torch.autocast("cuda", enabled=False):
            dy2 = dy.to(cols.dtype).contiguous(memory_format=torch.channels_last).permute(0, 2, 3, 1).reshape(-1, o)
            gw = gb = gx = None
            if ctx.needs_input_grad[1]:
                gm = torch.mm(cols.t(), dy2)
                gw = gm[:K].reshape(k, k, c, o).permute(3, 2, 0, 1).to(weight.dtype).contiguous()
            if has_bias and ctx.needs_input_grad[2]:
                gb = dy2.sum(0, dtype=torch.float32).to(weight.dtype)
            if ctx.needs_input_grad[0]:
                gx = torch.nn.grad.conv2d_input(x.shape, weight.to(dy2.dtype), dy.to(dy2.dtype), s, p)
        return gx, gw, gb, None, None, None


def _square(v):
    if isinstance(v, (tuple, list)):
        return v[0] if all(e == v[0] for e in v) else None
    return v


class StemConv2d(nn.Conv2d):
    """``nn.Conv2d`` whose CUDA forward is K7 im2col + cuBLAS GEMM (parameters unchanged)."""

    def forward(self, x):
        if not x.is_cuda:
            if self.training:
                raise RuntimeError("StemConv2d: training runs on the sm_100a K7 kernel (libmbs_native.so) and "
                                   "needs a CUDA tensor; there is no CPU fallback")
            return super().forward(x)          # eval-mode inference of a CPU copy: the same convolution
        return _StemConvFn.apply(x, self.weight, self.bias, self._k, self._s, self._p)


def supported(m: nn.Conv2d) -> bool:
    k, s, p, d = _square(m.kernel_size), _square(m.stride), _square(m.padding), _square(m.dilation)
    return (m.in_channels <= 4 and m.groups == 1 and d == 1 and m.padding_mode == "zeros"
            and None not in (k, s) and isinstance(p, int))


def swap_stem(model: nn.Module) -> nn.Module:
    """Route every supported low-channel ``nn.Conv2d`` (the stem) through K7 + GEMM, in place."""
    for m in model.modules():
        if type(m) is nn.Conv2d and supported(m):
            m.__class__ = StemConv2d
            m._k, m._s, m._p = int(_square(m.kernel_size)), int(_square(m.stride)), int(_square(m.padding))
    return model


class PointwiseConv2d(nn.Conv2d):
    """A 1x1 conv with few output channels (the U-Net head, 64 -> 1) as one cuBLAS GEMM over the
    channels-last activation viewed as [N*H*W, C_in] — cuDNN has no tensor-core kernel for
    C_out < 8 and runs a direct kernel (1.9 ms of the U-Net@384 step). Autograd through mm."""

    def forward(self, x):
        if not x.is_cuda or x.dim() != 4:
            return super().forward(x)
        n, c, h, w = x.shape
        x2 = x.contiguous(memory_format=torch.channels_last).permute(0, 2, 3, 1).reshape(n * h * w, c)
        wt = self.weight.reshape(self.out_channels, c).t()
        y = torch.addmm(self.bias, x2, wt) if self.bias is not None else torch.mm(x2, wt)
        return y.view(n, h, w, self.out_channels).permute(0, 3, 1, 2)


def swap_pointwise(model: nn.Module, max_out: int = 7) -> nn.Module:
    """Route 1x1 / stride-1 / unpadded convs with at most ``max_out`` output channels through one GEMM."""
    for m in model.modules():
        if (type(m) is nn.Conv2d and _square(m.kernel_size) == 1 and _square(m.stride) == 1 and
                _square(m.padding) == 0 and m.groups == 1 and _square(m.dilation) == 1 and m.out_channels <= max_out):
            m.__class__ = PointwiseConv2d
    return model
