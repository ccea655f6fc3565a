"""CUDA-graph capture of one micro-batch forward + loss + backward.

Measured on B200 (``tools/probe_cpu_issue.py``): issuing one ResNet-50
micro-batch step eagerly costs ~11-13 ms of host time (≈700 kernel launches,
autograd, the K5/K6/K7 ctypes calls) against ~13.8 ms of GPU time at micro
128 — the micro loop is CPU-bound to within a few percent, and any host
jitter idles the GPU. The MBS micro loop is the textbook case for CUDA graphs:
every micro-batch of a plan runs the same kernels on the same shapes, the
weights do not change until the optimizer step after the last micro-batch,
and only the input bytes and the normalisation factor differ.

``MicroStepGraph`` captures model(x) → loss (one graph) and backward (a second
graph sharing the first one's memory pool) once per distinct (model,
micro-batch shape/dtype, target shape/dtype, loss, autocast) — a plan has at
most two (full and ragged tail) — into static input/target/gradient buffers.
Per micro-batch K2 stages the input straight into the static input buffer
(``static_buffers``: the micro-batch sources ask for it, so the staged bytes
are written once), the two graphs replay back to back (the boundary between
them is where the schedule tracer marks the end of forward), and K1
accumulates the static gradients with the micro-batch's factor (the factor
stays OUT of the graph: ``normalize_via`` "fused"). Autocast weight casts are captured as kernels (cache disabled), so
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


def _fmt(t: torch.Tensor):
    return torch.channels_last if (t.dim() == 4 and t.is_contiguous(memory_format=torch.channels_last)
                                   and not t.is_contiguous()) else torch.contiguous_format


class MicroStepGraph:
    def __init__(self, model, plist, loss_kind, x_like, y_like, autocast_dtype, loss_from_logits, dice_smoothing,
                 warmup: int = 2, headroom: float = 1.15):
        dev = x_like.device
        fmt = _fmt(x_like)
        self.x = torch.empty_like(x_like, memory_format=fmt)
        self.x.copy_(x_like)
        self.y = y_like.detach().clone()
        self.plist = plist
        self._fmt = fmt

        def forward():
            ctx = (torch.autocast("cuda", dtype=autocast_dtype, cache_enabled=False)
                   if autocast_dtype is not None else torch.autocast("cuda", enabled=False))
            with ctx:
                out = model(self.x)
                loss = compute_loss(loss_kind, out, self.y, from_logits=loss_from_logits,
                                    dice_smoothing=dice_smoothing)
            return loss, out

        def step():
            loss, out = forward()
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
        self.fwd_graph = torch.cuda.CUDAGraph()
        self.bwd_graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.fwd_graph):
            loss, out = forward()
            # K1 reads the loss slot as fp32 (mbs_accum_add's loss pointer): convert inside the graph
            self.loss, self.out = loss.detach().float(), out.detach()
        with torch.cuda.graph(self.bwd_graph, pool=self.fwd_graph.pool()):
            loss.backward()
        del loss, out
        self.native_launches = TIMER.launches - n0   # this repo's kernels inside the graphs (K5/K6/K7/...)
        self.grads = [p.grad for p in plist]
        if any(g is None for g in self.grads):
            raise RuntimeError("a parameter received no gradient in the captured micro-batch step")
        for p, g in zip(plist, saved_grads):
            p.grad = g
        self.ptrs = (ctypes.c_void_p * len(self.grads))(*[g.data_ptr() for g in self.grads])

    def replay(self, xk, yk, between=None):
        """Forward + loss graph, ``between()`` (the tracer's forward-end mark), backward graph. Inputs already
        staged into the static buffers (``static_buffers``) are not copied again."""
        if xk.data_ptr() != self.x.data_ptr():
            self.x.copy_(xk)
        if yk.data_ptr() != self.y.data_ptr():
            self.y.copy_(yk)
        self.fwd_graph.replay()
        if between is not None:
            between()
        self.bwd_graph.replay()
        from .prof import TIMER
        TIMER.launches += self.native_launches
        return self.loss


def _key(model, plist, loss_kind, x_shape, x_dtype, x_fmt, y_shape, y_dtype, autocast_dtype, loss_from_logits,
         dice_smoothing):
    return (id(model), tuple(x_shape), x_dtype, x_fmt, tuple(y_shape), y_dtype, loss_kind, autocast_dtype,
            bool(loss_from_logits), float(dice_smoothing), tuple(p.data_ptr() for p in plist[:4]))


def static_buffers(model, plist, loss_kind, x_shape, x_dtype, channels_last, y_shape, y_dtype, autocast_dtype,
                   loss_from_logits, dice_smoothing):
    """(static input, static target) of the captured step for a micro-batch of this shape, or None if none
    is captured yet: the micro-batch sources stage straight into them."""
    fmt = torch.contiguous_format
    if channels_last and len(x_shape) == 4:
        fmt = _fmt(torch.empty(x_shape, device="meta", memory_format=torch.channels_last))
    g = _CACHE.get(_key(model, plist, loss_kind, x_shape, x_dtype, fmt, y_shape, y_dtype, autocast_dtype,
                        loss_from_logits, dice_smoothing))
    return (g.x, g.y) if g is not None else None


def graph_for(model, plist, loss_kind, xk, yk, autocast_dtype, loss_from_logits, dice_smoothing,
              headroom: float = 1.15) -> MicroStepGraph:
    """The cached capture for this micro shape; ``headroom`` x the step's activation bytes must be free
    (2.3 when an eager step of the same size must still fit next to the pool, e.g. the DP last micro)."""
    key = _key(model, plist, loss_kind, xk.shape, xk.dtype, _fmt(xk), yk.shape, yk.dtype, autocast_dtype,
               loss_from_logits, dice_smoothing)
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
