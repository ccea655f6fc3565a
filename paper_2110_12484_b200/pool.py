"""Channels-last max-pool on sm_100a (K6, ``csrc/mbs_pool.cu``) for the model's MaxPool2d.

torch's NHWC max-pool keeps an int64 index per output element; on B200 it was
8.5 % of the ResNet-50 micro-batch step (``profiles/r01_c2_v3_launches.md``) and
~10 % of the U-Net@384 step. K6 keeps a one-byte window-relative argmax and a
gather backward; forward and backward are bit-identical to ``F.max_pool2d``
(first maximum wins, NaN propagates, ascending-order fp32 gradient sums).

``swap_maxpool(model)`` turns every supported ``nn.MaxPool2d`` (square kernel,
stride and padding, dilation 1, floor mode, no returned indices) into a
:class:`MicroMaxPool2d` in place; parameters and state dicts are untouched
(max-pool has none). CUDA bf16/fp32 activations always run K6 (a missing
``libmbs_native.so`` raises); CPU tensors use torch (eval / oracle runs).
"""

from __future__ import annotations

import torch
from torch import nn

from . import _native
from .prof import TIMER

_DTYPES = {torch.bfloat16: _native.BF16, torch.float32: _native.F32}


def _square(v):
    if isinstance(v, (tuple, list)):
        return v[0] if len(v) == 2 and v[0] == v[1] else None
    return v


class _MaxPoolFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, k, s, p, dual=False):
        code = _DTYPES.get(x.dtype)
        if code is None:
            raise ValueError(f"K6 max-pool supports bfloat16 / float32, got {x.dtype}")
        x = x.contiguous(memory_format=torch.channels_last)
        n, c, h, w = x.shape
        ho, wo = (h + 2 * p - k) // s + 1, (w + 2 * p - k) // s + 1
        y = torch.empty((n, c, ho, wo), dtype=x.dtype, device=x.device, memory_format=torch.channels_last)
        idx = torch.empty((n, ho, wo, c), dtype=torch.uint8, device=x.device)
        stream = torch.cuda.current_stream(x.device)
        TIMER.launches += 1
        _native.check(_native.lib().mbs_maxpool_forward(x.data_ptr(), y.data_ptr(), idx.data_ptr(), code, n, h, w, c,
                                                        k, s, p, None, 0, 0, stream.cuda_stream), "mbs_maxpool_forward")
        ctx.save_for_backward(idx)
        ctx.geom = (n, c, h, w, k, s, p, code)
        if dual:   # two autograd handles: the consumers' gradients are summed inside the backward gather
            ctx.set_materialize_grads(False)
            return y, y.view_as(y)
        return y

    @staticmethod
    def backward(ctx, dy, dy2=None):
        (idx,) = ctx.saved_tensors
        n, c, h, w, k, s, p, code = ctx.geom
        if dy is None:
            dy, dy2 = dy2, None
        dt = {_native.BF16: torch.bfloat16, _native.F32: torch.float32}[code]
        dy = dy.to(dt).contiguous(memory_format=torch.channels_last)
        if dy2 is not None:
            dy2 = dy2.to(dt).contiguous(memory_format=torch.channels_last)
        dx = torch.empty((n, c, h, w), dtype=dy.dtype, device=dy.device, memory_format=torch.channels_last)
        stream = torch.cuda.current_stream(dy.device)
        TIMER.launches += 1
        _native.check(_native.lib().mbs_maxpool_backward(dy.data_ptr(), None if dy2 is None else dy2.data_ptr(),
                                                         idx.data_ptr(), dx.data_ptr(), code, n, h, w,
                                                         c, k, s, p, None, 0, 0, stream.cuda_stream),
                      "mbs_maxpool_backward")
        return dx, None, None, None, None


class _PoolStashFn(torch.autograd.Function):
    """(maxpool_k(s), buf): buf is a channels-last concat buffer with s in channels [0, C_s) and
    ``c_extra`` channels left for the decoder's upsampled tensor (written later by ``join_skip``).

    Backward fuses the skip-connection gradient: ds = maxpool_bwd(d_pooled) + d_buf[:, :C_s]."""

    @staticmethod
    def forward(ctx, s, k, c_extra):
        code = _DTYPES.get(s.dtype)
        if code is None:
            raise ValueError(f"K6 max-pool supports bfloat16 / float32, got {s.dtype}")
        s = s.contiguous(memory_format=torch.channels_last)
        n, c, h, w = s.shape
        y = torch.empty((n, c, h // k, w // k), dtype=s.dtype, device=s.device, memory_format=torch.channels_last)
        idx = torch.empty((n, h // k, w // k, c), dtype=torch.uint8, device=s.device)
        buf = torch.empty((n, c + c_extra, h, w), dtype=s.dtype, device=s.device, memory_format=torch.channels_last)
        stream = torch.cuda.current_stream(s.device)
        TIMER.launches += 1
        _native.check(_native.lib().mbs_maxpool_forward(s.data_ptr(), y.data_ptr(), idx.data_ptr(), code, n, h, w, c,
                                                        k, k, 0, buf.data_ptr(), c + c_extra, 0, stream.cuda_stream),
                      "mbs_maxpool_forward(stash)")
        ctx.save_for_backward(idx)
        ctx.geom = (n, c, h, w, k, code, c + c_extra)
        return y, buf

    @staticmethod
    def backward(ctx, dy, dbuf):
        (idx,) = ctx.saved_tensors
        n, c, h, w, k, code, ctot = ctx.geom
        dt = {_native.BF16: torch.bfloat16, _native.F32: torch.float32}[code]
        if dy is None:
            dy = torch.zeros((n, c, h // k, w // k), dtype=dt, device=idx.device, memory_format=torch.channels_last)
        dy = dy.to(dt).contiguous(memory_format=torch.channels_last)
        if dbuf is not None:
            dbuf = dbuf.to(dt).contiguous(memory_format=torch.channels_last)
        dx = torch.empty((n, c, h, w), dtype=dt, device=dy.device, memory_format=torch.channels_last)
        stream = torch.cuda.current_stream(dy.device)
        TIMER.launches += 1
        _native.check(_native.lib().mbs_maxpool_backward(
            dy.data_ptr(), None, idx.data_ptr(), dx.data_ptr(), code, n, h, w, c, k, k, 0,
            None if dbuf is None else dbuf.data_ptr(), ctot, 0, stream.cuda_stream), "mbs_maxpool_backward(addend)")
        return dx, None, None


_COLSUM_CTAS = 2 * 148


def _copy_channels(src, s_c, s_c0, dst, d_c, d_c0, m, c, bias, colsum=None):
    stream = torch.cuda.current_stream(src.device)
    TIMER.launches += 1
    _native.check(_native.lib().mbs_copy_channels(src.data_ptr(), s_c, s_c0, dst.data_ptr(), d_c, d_c0, m, c,
                                                  None if bias is None else bias.data_ptr(),
                                                  None if colsum is None else colsum.data_ptr(),
                                                  0 if colsum is None else colsum.shape[0], _DTYPES[src.dtype],
                                                  stream.cuda_stream), "mbs_copy_channels")


class _JoinFn(torch.autograd.Function):
    """buf[:, C_s:] = up (+ bias), in place (the second half of the U-Net concat); returns buf.

    ``bias`` (fp32, nullable) is the ConvTranspose bias, added while copying instead of in a
    separate broadcast pass over the upsampled tensor."""

    @staticmethod
    def forward(ctx, buf, up, bias, c_skip):
        up = up.to(buf.dtype).contiguous(memory_format=torch.channels_last)
        n, ctot, h, w = buf.shape
        cu = ctot - c_skip
        if bias is not None:
            bias = bias.detach().float().contiguous()
        _copy_channels(up, cu, 0, buf, ctot, c_skip, n * h * w, cu, bias)
        ctx.mark_dirty(buf)
        ctx.geom = (n, ctot, h, w, c_skip, bias is not None)
        return buf

    @staticmethod
    def backward(ctx, g):
        n, ctot, h, w, cs, has_bias = ctx.geom
        g = g.contiguous(memory_format=torch.channels_last)
        cu = ctot - cs
        gup = torch.empty((n, cu, h, w), dtype=g.dtype, device=g.device, memory_format=torch.channels_last)
        v = 16 // g.element_size()
        fuse = (has_bias and ctx.needs_input_grad[2] and cu % v == 0 and 256 % (cu // v) == 0
                and ctot % v == 0 and cs % v == 0 and g.data_ptr() % 16 == 0)
        parts = torch.empty((_COLSUM_CTAS, cu), dtype=torch.float32, device=g.device) if fuse else None
        _copy_channels(g, ctot, cs, gup, cu, 0, n * h * w, cu, None, parts)
        gb = None
        if has_bias and ctx.needs_input_grad[2]:   # the bias gradient: column sums taken during the copy
            gb = parts.sum(0) if fuse else gup.sum(dim=(0, 2, 3), dtype=torch.float32)
        return g, gup, gb, None


def pool_and_stash(s, kernel_size: int, c_extra: int):
    """``(max_pool2d(s, k), buf)`` with ``buf[:, :C_s] = s`` — the U-Net skip written straight into the
    decoder's concat buffer by the pooling kernel (non-overlapping k x k windows tiling s)."""
    return _PoolStashFn.apply(s, int(kernel_size), int(c_extra))


def join_skip(buf, up, bias=None):
    """Complete ``buf`` from :func:`pool_and_stash` with the upsampled tensor (plus its per-channel
    ``bias``, if given): equals ``torch.cat([s, up + bias], 1)``."""
    return _JoinFn.apply(buf, up, bias, buf.shape[1] - up.shape[1])


def max_pool2d(x, kernel_size: int, stride: int | None = None, padding: int = 0, dual: bool = False):
    """Functional K6 max-pool (square window, dilation 1, floor mode); ``dual``: the output as two
    autograd handles whose gradients are summed inside the backward kernel."""
    return _MaxPoolFn.apply(x, int(kernel_size), int(stride or kernel_size), int(padding), dual)


class MicroMaxPool2d(nn.MaxPool2d):
    """``nn.MaxPool2d`` whose CUDA forward/backward run K6 (bit-identical to torch)."""

    def forward(self, x, dual: bool = False):
        if not x.is_cuda and self.training:
            raise RuntimeError("MicroMaxPool2d: training runs on the sm_100a K6 kernels (libmbs_native.so) and "
                               "needs a CUDA tensor; there is no CPU fallback")
        if not x.is_cuda or x.dim() != 4:           # eval-mode inference of a CPU copy / unbatched input
            y = super().forward(x)
            return (y, y) if dual else y
        return _MaxPoolFn.apply(x, self._k, self._s, self._p, dual)


def supported(m: nn.MaxPool2d) -> bool:
    k, s, p, d = _square(m.kernel_size), _square(m.stride or m.kernel_size), _square(m.padding), _square(m.dilation)
    return (None not in (k, s, p, d) and d == 1 and not m.ceil_mode and not m.return_indices and k * k <= 255
            and 0 <= 2 * p <= k)


def swap_maxpool(model: nn.Module) -> nn.Module:
    """Route every supported ``nn.MaxPool2d`` of ``model`` through K6 (in place; returns the model)."""
    for m in model.modules():
        if type(m) is nn.MaxPool2d and supported(m):
            m.__class__ = MicroMaxPool2d
            m._k = int(_square(m.kernel_size))
            m._s = int(_square(m.stride or m.kernel_size))
            m._p = int(_square(m.padding))
    return model


__all__ = ["MicroMaxPool2d", "max_pool2d", "swap_maxpool", "supported", "pool_and_stash", "join_skip"]
