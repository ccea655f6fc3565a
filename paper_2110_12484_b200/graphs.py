"""CUDA-graph capture of one micro-batch forward + loss + backward.

Measured on B200 (``tools/probe_cpu_issue.py``): issuing one ResNet-50
micro-batch step eagerly costs ~11-13 ms of host time (≈700 kernel launches,
autograd, the K5/K6/K7 ctypes calls) against ~13.8 ms of GPU time at micro
128 — the micro loop is CPU-bound to within a few percent, and any host
jitter idles the GPU. The MBS micro loop is the textbook case for CUDA graphs:
every micro-batch of a plan runs the same kernels on the same shapes, the
weights do not change until the optimizer step after the last micro-batch,
and only the input bytes and the normalisation factor differ.

``MicroStepGraph`` captures model(x) → loss → backward once per distinct
(model, micro-batch shape/dtype, target shape/dtype, loss, autocast) — a plan
has at most two (full and ragged tail) — into static input/target/gradient
buffers. Per micro-batch the host copies the staged inputs into the static
buffers, replays the graph, and K1 accumulates the static gradients with the
micro-batch's factor (the factor stays OUT of the graph: ``normalize_via``
"fused"). Autocast weight casts are captured as kernels (cache disabled), so
each replay reads the current fp32 master weights; BN running statistics and
``num_batches_tracked`` update inside the graph exactly as in eager mode.
Capture warm-up iterations run on a side stream and every buffer of the model
(BN running statistics) is restored afterwards, so capturing does not change
training state.
"""

from __future__ import annotations

import ctypes

import torch

from .losses import compute_loss

_CACHE: dict = {}
MAX_GRAPHS = 8          # captured steps kept (each holds its model and a private memory pool); oldest evicted


class MicroStepGraph:
    def __init__(self, model, plist, loss_kind, x_like, y_like, autocast_dtype, loss_from_logits, dice_smoothing,
                 warmup: int = 2, headroom: float = 1.15):
        dev = x_like.device
        fmt = torch.channels_last if (x_like.dim() == 4 and x_like.is_contiguous(memory_format=torch.channels_last)
                                      and not x_like.is_contiguous()) else torch.contiguous_format
        self.x = torch.empty_like(x_like, memory_format=fmt)
        self.x.copy_(x_like)
        self.y = y_like.detach().clone()
        self.plist = plist
        self._fmt = fmt

        def step():
            ctx = (torch.autocast("cuda", dtype=autocast_dtype, cache_enabled=False)
                   if autocast_dtype is not None else torch.autocast("cuda", enabled=False))
            with ctx:
                out = model(self.x)
                loss = compute_loss(loss_kind, out, self.y, from_logits=loss_from_logits,
                                    dice_smoothing=dice_smoothing)
            loss.backward()
            return loss, out

        bufs = {k: v.detach().clone() for k, v in model.state_dict().items() if k not in dict(model.named_parameters())}
        saved_grads = [p.grad for p in plist]
        torch.cuda.synchronize(dev)
        torch.cuda.reset_peak_memory_stats(dev)
        base = torch.cuda.memory_allocated(dev)
        side = torch.cuda.Stream(dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):
            for _ in range(warmup):
                for p in plist:
                    p.grad = None
                step()
        torch.cuda.current_stream(dev).wait_stream(side)
        torch.cuda.synchronize(dev)
        with torch.no_grad():
            live = model.state_dict()
            for k, v in bufs.items():
                live[k].copy_(v)
        for p in plist:
            p.grad = None
        torch.cuda.empty_cache()           # warm-up blocks back to the driver before the private pool grows
        need = torch.cuda.max_memory_allocated(dev) - base
        free = torch.cuda.mem_get_info(dev)[0]
        if free < headroom * need + (1 << 30):
            # the private pool would not fit next to the eager allocator's blocks (e.g. a micro-batch
            # auto-sized to fill HBM): keep this shape eager
            raise MemoryError(f"graph pool needs ~{need / 2**30:.1f} GiB, {free / 2**30:.1f} GiB free")
        from .prof import TIMER
        n0 = TIMER.launches
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            loss, out = step()
            self.loss, self.out = loss.detach(), out.detach()
        self.native_launches = TIMER.launches - n0   # this repo's kernels inside the graph (K5/K6/K7/...)
        self.grads = [p.grad for p in plist]
        if any(g is None for g in self.grads):
            raise RuntimeError("a parameter received no gradient in the captured micro-batch step")
        for p, g in zip(plist, saved_grads):
            p.grad = g
        self.ptrs = (ctypes.c_void_p * len(self.grads))(*[g.data_ptr() for g in self.grads])

    def replay(self, xk, yk):
        self.x.copy_(xk)
        self.y.copy_(yk)
        self.graph.replay()
        from .prof import TIMER
        TIMER.launches += self.native_launches
        return self.loss


def graph_for(model, plist, loss_kind, xk, yk, autocast_dtype, loss_from_logits, dice_smoothing,
              headroom: float = 1.15) -> MicroStepGraph:
    """The cached capture for this micro shape; ``headroom`` x the step's activation bytes must be free
    (2.3 when an eager step of the same size must still fit next to the pool, e.g. the DP last micro)."""
    key = (id(model), tuple(xk.shape), xk.dtype, xk.is_contiguous(), tuple(yk.shape), yk.dtype, loss_kind,
           autocast_dtype, bool(loss_from_logits), float(dice_smoothing), tuple(p.data_ptr() for p in plist[:4]))
    g = _CACHE.get(key)
    if g is None:
        while len(_CACHE) >= MAX_GRAPHS:
            _CACHE.pop(next(iter(_CACHE)))
            torch.cuda.empty_cache()
        g = _CACHE[key] = MicroStepGraph(model, plist, loss_kind, xk, yk, autocast_dtype, loss_from_logits,
                                         dice_smoothing, headroom=headroom)
    return g


def clear() -> None:
    """Drop every captured graph (and its private memory pool)."""
    _CACHE.clear()
    torch.cuda.empty_cache()
