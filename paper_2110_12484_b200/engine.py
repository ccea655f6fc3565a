"""Micro-batch streaming training loop on the B200 — the reference's ``engine.py`` API.

Same functions, argument meaning and exceptions as the reference
(``engine.py:37-335``): ``plan_split``, ``normalization_factor``,
``normalize_loss``, ``GradientAccumulator``, ``accumulate``,
``mini_batch_gradient``, ``train_mini_batch``, ``train_epoch``. What changes
is where the work runs:

* the model is a torch ``nn.Module`` whose forward/backward stay on
  cuDNN/cuBLAS (optionally under autocast);
* micro-batches come from HBM (K2 staging) or from host memory through the
  pinned H2D streamer (``streamer.py``);
* the per-micro normalise-and-accumulate is ONE fused sm_100a kernel over the
  flat gradient (K1, ``mbs_accum_add``): ``acc = s*g`` on the first
  micro-batch of a mini-batch (the zero of ``begin`` folded in),
  ``acc += s*g`` afterwards, with the grad-norm partials and the loss record
  fused into the last pass; the optimizer is one fused flat pass (K3);
* the loss / grad-norm statistics stay on device until read: there is no
  host synchronisation inside the micro loop.

``normalize_via``: the reference folds the factor into the backward seed
(``"seed"``, ``engine.py:214-215``) or scales the recorded loss
(``"loss_scale"``, ``engine.py:211-213``). Both remain available; the default
``"fused"`` runs backward with seed 1 and applies the factor inside K1. All
three are the same linear map (``backward`` is linear in the seed), so the
accumulated gradients agree to fp32 rounding (tests/test_engine_gpu.py).
"""

from __future__ import annotations

import ctypes
import math
import os
import weakref
from contextlib import nullcontext
from dataclasses import dataclass, field
from typing import Callable

import numpy as np
import torch

from . import _native as N
from .errors import AccumulatorOverflowError, GradientKeyMismatchError, NonFiniteError
from .losses import LossValue, compute_loss
from .optim import OptimizerState, apply_update
from .prof import TIMER
from .rng import epoch_order
from .streamer import MicroBatchStreamer, Staging, device_micro_batches
from .tensor import GradientSet, ParameterSet

NORMALIZATION_MODES = ("paper_faithful", "exact_weighted", "off")  # engine.py:34
NORMALIZE_VIA = ("fused", "seed", "loss_scale")


# ---------------------------------------------------------------------------
# Plan (engine.py:37-97)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class MicroBatchPlan:
    """Ordered split of one mini-batch into contiguous micro-batches (engine.py:37-53)."""

    n_b: int
    n_mu: int
    n_s_mu: int
    sizes: tuple
    index_ranges: tuple

    def __post_init__(self):
        if sum(self.sizes) != self.n_b:
            raise ValueError("micro-batch sizes must cover the mini-batch exactly")
        if any(s < 1 or s > self.n_mu for s in self.sizes):
            raise ValueError("every micro-batch size must lie in [1, n_mu]")
        if len(self.sizes) != self.n_s_mu or len(self.index_ranges) != self.n_s_mu:
            raise ValueError("plan length disagrees with n_s_mu")


def plan_split(n_b: int, n_mu: int) -> MicroBatchPlan:
    """Split n_b samples into micro-batches of at most n_mu (engine.py:56-78), via ``mbs_plan_split``."""
    L = N.lib()
    nm, ns = ctypes.c_int64(), ctypes.c_int64()
    N.check(L.mbs_plan_split(int(n_b), int(n_mu), ctypes.byref(nm), ctypes.byref(ns), None, 0), "plan_split")
    sizes = (ctypes.c_int64 * ns.value)()
    N.check(L.mbs_plan_split(int(n_b), int(n_mu), None, None, sizes, ns.value), "plan_split")
    sizes = tuple(int(s) for s in sizes)
    ranges, start = [], 0
    for s in sizes:
        ranges.append((start, start + s))
        start += s
    return MicroBatchPlan(n_b=int(n_b), n_mu=nm.value, n_s_mu=ns.value, sizes=sizes, index_ranges=tuple(ranges))


def normalization_factor(plan: MicroBatchPlan, k: int, mode: str) -> float:
    """Scale applied to micro-batch k's loss before backward (engine.py:81-91)."""
    if not 0 <= k < plan.n_s_mu:
        raise ValueError(f"micro-batch index {k} outside plan of {plan.n_s_mu}")
    if mode == "paper_faithful":
        return 1.0 / plan.n_s_mu
    if mode == "exact_weighted":
        return plan.sizes[k] / plan.n_b
    if mode == "off":
        return 1.0
    raise ValueError(f"unknown normalization mode {mode!r}")


def normalize_loss(loss: LossValue, plan: MicroBatchPlan, k: int, mode: str) -> LossValue:
    """engine.py:94-97."""
    factor = normalization_factor(plan, k, mode)
    return LossValue(value=loss.value * factor, n_samples=loss.n_samples)


# ---------------------------------------------------------------------------
# Gradient accumulator (engine.py:100-137) — K1
# ---------------------------------------------------------------------------

def _stream_ptr(stream=None) -> int:
    return (stream or torch.cuda.current_stream()).cuda_stream


class GradientAccumulator:
    """Running fp32 sum of micro-batch gradients in one flat HBM buffer (engine.py:100-131).

    ``sums`` / ``as_gradient_set()`` alias the live buffer (as the reference's
    do). ``begin`` is lazy: the next ``add`` assigns instead of
    accumulating, so no zero pass is ever paid on the hot path.
    """

    DEFAULT_MAX_MICRO = 1 << 16

    def __init__(self, params: ParameterSet, expected: int | None = None, *, max_micro: int | None = None):
        if not isinstance(params, ParameterSet):
            raise TypeError("GradientAccumulator needs a paper_2110_12484_b200.ParameterSet")
        self.params = params
        self.layout = params.layout
        self.max_micro = int(max_micro or self.DEFAULT_MAX_MICRO)
        self.flat = torch.zeros(self.layout.total, dtype=torch.float32, device=params.device)
        self.stats_dev = torch.zeros(4 + 2 * self.max_micro, dtype=torch.float64, device=params.device)
        offs = N.i64_array(self.layout.offsets)
        nums = N.i64_array(self.layout.numels)
        h = ctypes.c_void_p()
        N.check(N.lib().mbs_accum_create(self.flat.data_ptr(), self.layout.total, len(self.layout.names), offs, nums,
                                         self.max_micro, ctypes.byref(h)), "mbs_accum_create")
        self._h = h
        self._views = self.layout.views(self.flat)
        # the tensors autograd fills: the module's parameters (bf16 shadows in shadow-weight mode)
        self._plist = list(params.grad_params) if params.grad_params is not None else \
            [params[n] for n in self.layout.names]
        self._ptr_table = (ctypes.c_void_p * len(self._plist))()
        self._dtype_table = (ctypes.c_int * len(self._plist))(
            *[N.BF16 if p.dtype == torch.bfloat16 else N.F32 for p in self._plist])
        self._typed = any(p.dtype == torch.bfloat16 for p in self._plist)
        gsz = [2 if p.dtype == torch.bfloat16 else 4 for p in self._plist]
        # algorithmic K1 bytes per full pass: read g (2 or 4 B) + write acc (4 B) [+ read acc (4 B)]
        self._k1_bytes_assign = sum(n * (g + 4) for n, g in zip(self.layout.numels, gsz))
        self._k1_bytes_acc = self._k1_bytes_assign + 4 * self.layout.n_params
        self._pending_zero = False
        self._fresh = True
        self._norm_valid = False
        self._covered = 0
        self.expected = expected
        if expected is not None:
            self.begin(expected)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                torch.cuda.synchronize(self.flat.device)
                N.lib().mbs_accum_destroy(h)
            except Exception:
                pass

    # -- reference surface --
    @property
    def micro_batches_seen(self) -> int:
        seen = ctypes.c_int64()
        N.check(N.lib().mbs_accum_seen(self._h, ctypes.byref(seen), None), "mbs_accum_seen")
        return seen.value

    @property
    def sums(self) -> dict:
        self._materialize()
        return dict(self._views)

    def begin(self, expected: int) -> None:
        """Reset for the next mini-batch (engine.py:110-115); the zero is folded into the next add."""
        if expected is not None and expected > self.max_micro:
            raise ValueError(f"{expected} micro-batches exceed max_micro={self.max_micro}")
        N.check(N.lib().mbs_accum_begin(self._h, -1 if expected is None else int(expected)), "mbs_accum_begin")
        self.expected = expected
        self._pending_zero = True
        self._fresh = True
        self._norm_valid = False
        self._covered = 0

    def add(self, grads: GradientSet | dict) -> None:
        """sums += grads in parameter order (engine.py:117-128)."""
        arrays = grads.arrays if isinstance(grads, GradientSet) else dict(grads)
        if set(arrays) != set(self.layout.names):
            raise AccumulatorOverflowError("gradient keys do not match accumulator parameters")
        tensors = []
        for i, n in enumerate(self.layout.names):
            g = arrays[n]
            if tuple(g.shape) != self.layout.shapes[i]:
                raise GradientKeyMismatchError(f"gradient shape {tuple(g.shape)} != parameter shape "
                                               f"{self.layout.shapes[i]} for {n!r}")
            tensors.append(g)
        self.add_tensors(tensors, 1.0)

    def as_gradient_set(self) -> GradientSet:
        """engine.py:130-131 — a GradientSet ALIASING the live sums."""
        self._materialize()
        # the device norm is attached only when finalize() reduced it for exactly these sums; otherwise
        # GradientSet.l2_norm() recomputes it and the K3 guard is off (the reference has no guard)
        norm2 = self.stats_dev[0] if self._norm_valid else None
        return GradientSet(dict(self._views), flat=self.flat, layout=self.layout, norm2=norm2)

    # -- B200 surface --
    def _materialize(self):
        if self._pending_zero and self.micro_batches_seen == 0:
            N.check(N.lib().mbs_accum_zero(self._h, _stream_ptr()), "mbs_accum_zero")
        self._pending_zero = False

    def _same_memory_order(self, g: torch.Tensor, i: int) -> bool:
        """Dense tensors of one shape share their memory order iff strides agree on every dim of size > 1
        (autograd's layout contract ignores size-1 dims, e.g. 1x1 conv weights in channels_last)."""
        shape, stride = self.layout.shapes[i], self.layout.strides[i]
        if tuple(g.shape) != shape or any(a != b for a, b, n in zip(g.stride(), stride, shape) if n > 1):
            return False
        return sum((n - 1) * st for n, st in zip(shape, g.stride())) == g.numel() - 1   # dense, no overlap

    def _conform(self, g: torch.Tensor, i: int, allow_bf16: bool = True) -> torch.Tensor:
        """g in the segment's memory order and in fp32 or bf16 (K1 reads both; anything else is cast;
        ``allow_bf16=False`` for the fp32-only peer all-reduce kernel)."""
        shape, stride = self.layout.shapes[i], self.layout.strides[i]
        ok = (torch.float32, torch.bfloat16) if allow_bf16 else (torch.float32,)
        if g.dtype in ok and g.device == self.flat.device and (
                tuple(g.stride()) == stride or self._same_memory_order(g, i)):
            return g
        out = torch.empty_strided(shape, stride, dtype=torch.float32, device=self.flat.device)
        out.copy_(g)
        return out

    def _add(self, ptrs, dtypes, seg_begin, n, factor, lp, lf, loss_weight, last, stream):
        if dtypes is None:
            return N.lib().mbs_accum_add(self._h, ptrs, seg_begin, n, float(factor), lp, lf, float(loss_weight),
                                         int(bool(last)), _stream_ptr(stream))
        return N.lib().mbs_accum_add_typed(self._h, ptrs, ctypes.cast(dtypes, ctypes.c_void_p), seg_begin, n,
                                           float(factor), lp, lf, float(loss_weight), int(bool(last)),
                                           _stream_ptr(stream))

    def add_tensors(self, tensors: list, factor: float, *, loss: torch.Tensor | None = None,
                    loss_factor: float | None = None, loss_weight: float = 0.0, last: bool = False,
                    seg_begin: int = 0, stream=None) -> None:
        """K1 over segments [seg_begin, seg_begin+len(tensors)): acc (+)= factor * g."""
        n = len(tensors)
        ptrs = (ctypes.c_void_p * n)()
        dtypes = (ctypes.c_int * n)()
        keep = []
        for j, g in enumerate(tensors):
            g = self._conform(g, seg_begin + j)
            keep.append(g)
            ptrs[j] = g.data_ptr()
            dtypes[j] = N.BF16 if g.dtype == torch.bfloat16 else N.F32
        lp = None
        if loss is not None:
            loss = loss.detach()
            if loss.dtype != torch.float32:
                loss = loss.float()
            keep.append(loss)
            lp = loss.data_ptr()
        lf = float(factor if loss_factor is None else loss_factor)
        t0 = TIMER.start(stream)
        N.check(self._add(ptrs, dtypes, int(seg_begin), n, factor, lp, lf, loss_weight, last, stream), "mbs_accum_add")
        if t0 is not None:
            nb = sum((2 if t.dtype == torch.bfloat16 else 4) * t.numel() for t in keep[:n])
            elems = sum(self.layout.numels[seg_begin:seg_begin + n])
            TIMER.stop("k1_accumulate", t0, nb + (4 if self._fresh else 8) * elems, stream)
        self._norm_valid = False   # a K1 pass since the last finalize
        self._covered += n
        if self._covered >= len(self.layout.names):
            self._covered = 0
            self._fresh = False
        self._pending_zero = False

    def graph_grads_ok(self, grads: list) -> bool:
        """Whether static (graph-captured) gradients can feed K1 without a re-layout."""
        strides = self.layout.strides
        return len(grads) == len(self._plist) and all(
            g is not None and g.dtype is p.dtype and (g.stride() == strides[j] or self._same_memory_order(g, j))
            for j, (g, p) in enumerate(zip(grads, self._plist)))

    def add_pointer_table(self, ptrs, factor: float, *, loss: torch.Tensor | None = None,
                          loss_factor: float | None = None, loss_weight: float = 0.0, last: bool = False,
                          stream=None) -> None:
        """K1 over every segment from a prebuilt device-pointer table (a captured micro step's gradients)."""
        lp = None
        if loss is not None:
            if loss.dtype != torch.float32:      # K1 reads the loss slot as fp32
                loss = loss.detach().float()
            lp = loss.data_ptr()
        lf = float(factor if loss_factor is None else loss_factor)
        t0 = TIMER.start(stream)
        N.check(self._add(ptrs, self._dtype_table, 0, len(self._plist), factor, lp, lf, loss_weight, last, stream),
                "mbs_accum_add")
        if t0 is not None:
            TIMER.stop("k1_accumulate", t0, self._k1_bytes_assign if self._fresh else self._k1_bytes_acc, stream)
        self._fresh = False
        self._norm_valid = False   # a K1 pass since the last finalize
        self._covered = 0
        self._pending_zero = False

    def add_module_grads(self, factor: float, *, loss: torch.Tensor | None = None,
                         loss_factor: float | None = None, loss_weight: float = 0.0, last: bool = False,
                         stream=None) -> None:
        """K1 straight from the module's ``.grad`` tensors, which are then released.

        Hot path: the pointer table is a preallocated ctypes array; a gradient
        is only re-laid-out when its dtype/strides differ from the parameter's.
        """
        ptrs = self._ptr_table
        keep = []
        strides = self.layout.strides
        dts = self._dtype_table
        for j, p in enumerate(self._plist):
            g = p.grad
            if g is None:
                raise AccumulatorOverflowError("gradient keys do not match accumulator parameters "
                                               "(a parameter received no gradient)")
            if g.dtype is not p.dtype or (g.stride() != strides[j] and not self._same_memory_order(g, j)):
                g = self._conform(g, j)
                keep.append(g)
                dts[j] = N.BF16 if g.dtype == torch.bfloat16 else N.F32
            ptrs[j] = g.data_ptr()
        lp = None
        if loss is not None:
            loss = loss.detach()
            if loss.dtype != torch.float32:
                loss = loss.float()
            keep.append(loss)
            lp = loss.data_ptr()
        lf = float(factor if loss_factor is None else loss_factor)
        n = len(self._plist)
        t0 = TIMER.start(stream)
        N.check(self._add(ptrs, dts, 0, n, factor, lp, lf, loss_weight, last, stream), "mbs_accum_add")
        for j, p in enumerate(self._plist):        # restore the per-parameter dtype codes
            dts[j] = N.BF16 if p.dtype == torch.bfloat16 else N.F32
        if t0 is not None:
            TIMER.stop("k1_accumulate", t0, self._k1_bytes_assign if self._fresh else self._k1_bytes_acc, stream)
        self._fresh = False
        self._norm_valid = False   # a K1 pass since the last finalize
        self._covered = 0
        self._pending_zero = False
        for p in self._plist:
            p.grad = None

    def add_allreduce(self, peer, factor: float, *, from_module: bool = True, tensors: list | None = None,
                      loss: torch.Tensor | None = None, loss_factor: float | None = None, loss_weight: float = 0.0,
                      timeout_ms: float = 60_000.0, stream=None) -> None:
        """K1C: this rank's last micro-batch fused with the all-reduce over peer memory (``mbs_accum_add_allreduce``).

        With ``from_module`` the gradients are the parameters' ``.grad`` tensors (then released);
        ``from_module=False`` and ``tensors=None`` contributes only the accumulator (a rank without a
        micro-batch in this mini-batch).
        """
        ptrs, keep = None, []
        if from_module or tensors is not None:
            src = [p.grad for p in self._plist] if from_module else list(tensors)
            ptrs = self._ptr_table
            for j, g in enumerate(src):
                if g is None:
                    raise AccumulatorOverflowError("gradient keys do not match accumulator parameters "
                                                   "(a parameter received no gradient)")
                g = self._conform(g, j, allow_bf16=False)
                keep.append(g)
                ptrs[j] = g.data_ptr()
        lp = None
        if loss is not None:
            loss = loss.detach().float()
            keep.append(loss)
            lp = loss.data_ptr()
        lf = float(factor if loss_factor is None else loss_factor)
        t0 = TIMER.start(stream)
        N.check(N.lib().mbs_accum_add_allreduce(self._h, peer.handle, ptrs, float(factor), lp, lf, float(loss_weight),
                                                float(timeout_ms), _stream_ptr(stream)), "mbs_accum_add_allreduce")
        TIMER.stop("k1c_accumulate_allreduce", t0, 12 * self.layout.n_params, stream)
        self._fresh = False
        self._norm_valid = False   # a K1 pass since the last finalize
        self._covered = 0
        self._pending_zero = False
        if from_module:
            for p in self._plist:
                p.grad = None

    def finalize(self, n_b: int, *, recompute_norm: bool = False, stream=None) -> torch.Tensor:
        """Reduce the grad-norm partials and the loss record into ``stats_dev`` (device)."""
        if recompute_norm:
            t0 = TIMER.start(stream)
            N.check(N.lib().mbs_accum_norm(self._h, _stream_ptr(stream)), "mbs_accum_norm")
            TIMER.stop("k1_norm", t0, 4 * self.layout.n_params, stream)
        t0 = TIMER.start(stream)
        N.check(N.lib().mbs_accum_finalize(self._h, int(n_b), self.stats_dev.data_ptr(), _stream_ptr(stream)),
                "mbs_accum_finalize")
        TIMER.stop("k4_finalize", t0, 0, stream)
        self._norm_valid = True
        return self.stats_dev


def accumulate(acc: GradientAccumulator, grads: GradientSet) -> GradientAccumulator:
    """engine.py:134-137."""
    acc.add(grads)
    return acc


# ---------------------------------------------------------------------------
# Statistics (engine.py:166-176, 264-273) — resolved lazily, one D2H per mini-batch
# ---------------------------------------------------------------------------

class MiniBatchStats:
    """Per-mini-batch observables (engine.py:166-176), copied off the device asynchronously.

    Reading any field synchronises on that copy; a non-finite accumulated
    gradient or micro-batch loss raises ``NonFiniteError`` there.
    ``train_mini_batch`` / ``train_epoch`` resolve it before the optimizer
    step, so on a non-finite mini-batch the parameters, the optimizer moments
    and ``step_count`` are exactly where the reference leaves them (it raises
    in the forward, ``nn.py:578-579``, before any update).
    """

    def __init__(self, stats_dev: torch.Tensor, n_micro: int, max_micro: int, outputs: list, stream=None):
        self._n = int(n_micro)
        self._max = int(max_micro)
        head = torch.cat([stats_dev[:4 + self._n], stats_dev[4 + self._max:4 + self._max + self._n]])
        self._host = torch.empty(head.shape, dtype=torch.float64, pin_memory=True)
        self._host.copy_(head, non_blocking=True)
        self._event = torch.cuda.Event()
        self._event.record(stream or torch.cuda.current_stream())
        self._outputs = outputs
        self._resolved = None
        self.step_count = 0

    def resolve(self) -> dict:
        if self._resolved is None:
            self._event.synchronize()
            h = self._host.tolist()
            n = self._n
            self._resolved = dict(norm2=h[0], loss=h[1], nonfinite=h[2] != 0.0, losses_raw=h[4:4 + n],
                                  losses_normalized=h[4 + n:4 + 2 * n])
            if self._resolved["nonfinite"] or not all(math.isfinite(v) for v in self._resolved["losses_raw"]):
                raise NonFiniteError(-1, "non-finite accumulated gradient or micro-batch loss; "
                                         "the optimizer step was skipped")
        return self._resolved

    @property
    def losses_raw(self) -> list:
        return self.resolve()["losses_raw"]

    @property
    def losses_normalized(self) -> list:
        return self.resolve()["losses_normalized"]

    @property
    def loss(self) -> float:
        return self.resolve()["loss"]

    @property
    def grad_norm(self) -> float:
        return math.sqrt(self.resolve()["norm2"])

    @property
    def n_micro(self) -> int:
        return self._n

    @property
    def outputs(self) -> torch.Tensor | None:
        if not self._outputs:
            return None
        if len(self._outputs) > 1:
            self._outputs = [torch.cat(self._outputs, dim=0)]
        return self._outputs[0]


@dataclass
class EpochStats:
    """engine.py:264-273."""

    mini_losses: list
    mean_loss: float
    mini_metrics: list
    mini_sizes: list
    step_count: int
    mini_stats: list = field(default_factory=list)


# ---------------------------------------------------------------------------
# The micro loop (engine.py:179-230)
# ---------------------------------------------------------------------------

def _as_tensor(a):
    if isinstance(a, torch.Tensor):
        return a
    return torch.from_numpy(np.ascontiguousarray(a))


def _micro_source(x, y, jobs, staging, prefetch, streamer, dest=None, tracer=None):
    if x.device.type == "cuda":
        return device_micro_batches(x, y.to(x.device) if y.device != x.device else y, jobs, staging, dest=dest,
                                    tracer=tracer)
    if streamer is None:
        raise ValueError("host-resident inputs need a MicroBatchStreamer (pass streamer=...)")
    return streamer.stream(x, y, jobs, staging, prefetch=prefetch, dest=dest, tracer=tracer)


def _graph_dest(model, acc, loss_kind, autocast_dtype, loss_from_logits, dice_smoothing, normalize_via):
    """Where the sources stage a micro-batch: the static buffers of its captured micro step when one exists
    (K2 then writes the model input once), else a fresh tensor (None)."""
    if not (CUDA_GRAPHS and normalize_via == "fused" and model.training):
        return None
    from . import graphs
    plist = acc._plist

    def dest(x_shape, x_dtype, channels_last, y_shape, y_dtype):
        return graphs.static_buffers(model, plist, loss_kind, x_shape, x_dtype, channels_last, y_shape, y_dtype,
                                     autocast_dtype, loss_from_logits, dice_smoothing)
    return dest


def make_streamer(x: torch.Tensor, y: torch.Tensor, max_rows: int, *, n_slots: int = 3, n_threads=None):
    """A streamer sized for micro-batches of up to ``max_rows`` rows of x / y."""
    xr = x.element_size() * int(np.prod(x.shape[1:]))
    yr = y.element_size() * int(np.prod(y.shape[1:])) if y.dim() > 1 else y.element_size()
    return MicroBatchStreamer(xr, yr, max_rows, n_slots=n_slots, n_threads=n_threads)


def mini_batch_gradient(model: torch.nn.Module, params: ParameterSet, x, y, plan: MicroBatchPlan,
                        normalization: str = "paper_faithful", loss_kind: str = "mse", *,
                        loss_from_logits: bool = True, dice_smoothing: float = 1.0, prefetch: bool = False,
                        accumulator: GradientAccumulator | None = None, normalize_via: str = "fused",
                        forward_mode: str = "train", staging: Staging | None = None,
                        autocast_dtype: torch.dtype | None = None, streamer: MicroBatchStreamer | None = None,
                        keep_outputs: bool = True, tracer=None, _close_trace: bool = True) -> tuple:
    """Accumulated gradient of one mini-batch, micro-batch by micro-batch (engine.py:179-230).

    ``x``/``y`` are device tensors (sliced / staged in HBM) or host tensors
    (streamed through ``streamer``; one is created when omitted). ``tracer``:
    a ``streaming.ScheduleTracer`` recording the real per-micro schedule.
    Returns (GradientSet aliasing the accumulator, MiniBatchStats).
    """
    x, y = _as_tensor(x), _as_tensor(y)
    if x.shape[0] != plan.n_b:
        raise ValueError(f"batch has {x.shape[0]} samples but plan expects {plan.n_b}")
    if normalize_via not in NORMALIZE_VIA:
        raise ValueError(f"unknown normalize_via {normalize_via!r}")
    if normalization not in NORMALIZATION_MODES:
        raise ValueError(f"unknown normalization mode {normalization!r}")
    if forward_mode not in ("train", "eval"):
        raise ValueError(f"mode must be 'train' or 'eval', got {forward_mode!r}")
    acc = accumulator if accumulator is not None else GradientAccumulator(params)
    acc.begin(plan.n_s_mu)
    model.train(forward_mode == "train")
    own_streamer = None
    if x.device.type == "cpu" and streamer is None:
        streamer = own_streamer = make_streamer(x, y, plan.n_mu)
    jobs = [(None, lo, hi - lo) for lo, hi in plan.index_ranges]
    dest = _graph_dest(model, acc, loss_kind, autocast_dtype, loss_from_logits, dice_smoothing, normalize_via)
    try:
        source = _micro_source(x, y, jobs, staging, prefetch, streamer, dest, tracer)
        outputs = _run_micro_loop(model, acc, plan, source, normalization, loss_kind, loss_from_logits,
                                  dice_smoothing, normalize_via, autocast_dtype, keep_outputs, tracer)
    finally:
        if own_streamer is not None:
            own_streamer.close()
    if tracer is not None:
        tracer.update_begin()
    stats_dev = acc.finalize(plan.n_b)
    if tracer is not None and _close_trace:
        tracer.update_end()
    stats = MiniBatchStats(stats_dev, plan.n_s_mu, acc.max_micro, outputs)
    return acc.as_gradient_set(), stats


def _run_micro_loop(model, acc, plan, source, normalization, loss_kind, loss_from_logits, dice_smoothing,
                    normalize_via, autocast_dtype, keep_outputs, tracer=None):
    """The micro loop; K1 records (raw loss, factor, size_k) per micro for the stats."""
    outputs = []
    ctx = torch.autocast("cuda", dtype=autocast_dtype) if autocast_dtype is not None else nullcontext()
    with weight_cast_cache(autocast_dtype):
        return _micro_loop_body(model, acc, plan, source, normalization, loss_kind, loss_from_logits,
                                dice_smoothing, normalize_via, ctx, keep_outputs, outputs, autocast_dtype, tracer)


def weight_cast_cache(autocast_dtype):
    """Keep torch's autocast weight-cast cache alive across the micro-batches of ONE mini-batch.

    The weights are constant until the optimizer step that follows the last
    micro-batch, so each fp32 master weight needs its low-precision copy once
    per mini-batch, not once per micro-batch (ResNet-50: 54 casts and 142 MB
    of traffic per micro saved). torch clears the cache when the OUTERMOST
    autocast region exits; an outer region with autocast DISABLED keeps the
    nesting count up without changing how forward or backward run. The cache
    is dropped when this region exits, i.e. before the optimizer step.
    """
    if autocast_dtype is None:
        return nullcontext()
    return torch.autocast("cuda", dtype=autocast_dtype, enabled=False)


def _micro_loop_body(model, acc, plan, source, normalization, loss_kind, loss_from_logits, dice_smoothing,
                     normalize_via, ctx, keep_outputs, outputs, autocast_dtype=None, tracer=None):
    k = -1
    for k, (xk, yk) in enumerate(source):
        if k >= plan.n_s_mu:
            raise AccumulatorOverflowError("source yielded more micro-batches than the plan")
        factor = normalization_factor(plan, k, normalization)
        if tracer is not None:
            tracer.micro_begin(k)
        g = _graph_for(model, acc, loss_kind, xk, yk, autocast_dtype, loss_from_logits, dice_smoothing,
                       normalize_via, keep_outputs)
        if g is not None:                 # CUDA-graph replay of fwd + loss + bwd; K1 outside the graph
            loss = g.replay(xk, yk, between=tracer.forward_end if tracer is not None else None)
            acc.add_pointer_table(g.ptrs, factor, loss=loss, loss_factor=factor, loss_weight=float(plan.sizes[k]),
                                  last=(k == plan.n_s_mu - 1))
            if tracer is not None:
                tracer.micro_end()
            if keep_outputs:
                outputs.append(g.out.clone())   # the static output is overwritten by the next replay
            continue
        with ctx:
            out = model(xk)
            loss = compute_loss(loss_kind, out, yk, from_logits=loss_from_logits, dice_smoothing=dice_smoothing)
        if tracer is not None:
            tracer.forward_end()
        if normalize_via == "seed":
            loss.backward(torch.full_like(loss, factor))
            kscale = 1.0
        elif normalize_via == "loss_scale":
            (loss * factor).backward()
            kscale = 1.0
        else:
            loss.backward()
            kscale = factor
        acc.add_module_grads(kscale, loss=loss, loss_factor=factor, loss_weight=float(plan.sizes[k]),
                             last=(k == plan.n_s_mu - 1))
        if tracer is not None:
            tracer.micro_end()
        if keep_outputs:
            outputs.append(out.detach())
    if k + 1 != plan.n_s_mu:
        raise ValueError(f"source yielded {k + 1} micro-batches, plan expects {plan.n_s_mu}")
    return outputs


CUDA_GRAPHS = os.environ.get("MBS_CUDA_GRAPHS", "1") != "0"
# model -> the micro-step shapes whose capture failed (weak keys: a collected model's entry goes with it,
# and a failure for one shape, e.g. an HBM-filling ragged tail, does not disable the others)
_NO_GRAPH: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


def _graph_for(model, acc, loss_kind, xk, yk, autocast_dtype, loss_from_logits, dice_smoothing, normalize_via,
               keep_outputs, headroom: float = 1.15):
    """The captured micro step for this micro-batch shape, or None to run eagerly.

    Graphs need: CUDA inputs, training mode, the factor applied by K1 (normalize_via "fused") and
    gradients in the parameters' memory order (kept outputs are cloned from the static output). A shape whose
    capture fails runs eagerly from then on (the failure is kept per model and shape, not retried every
    micro-batch)."""
    if not (CUDA_GRAPHS and normalize_via == "fused" and model.training
            and isinstance(xk, torch.Tensor) and xk.is_cuda and isinstance(yk, torch.Tensor) and yk.is_cuda):
        return None
    shape_key = (tuple(xk.shape), xk.dtype, tuple(yk.shape), yk.dtype, loss_kind, autocast_dtype,
                 bool(loss_from_logits), float(dice_smoothing))
    failed = _NO_GRAPH.get(model)
    if failed is not None and shape_key in failed:
        return None
    from . import graphs
    try:
        g = graphs.graph_for(model, acc._plist, loss_kind, xk, yk, autocast_dtype, loss_from_logits, dice_smoothing,
                             headroom=headroom)
    except Exception as e:                 # noqa: BLE001 - capture limits: fall back to eager, loudly
        import warnings
        if not isinstance(e, MemoryError):
            warnings.warn(f"CUDA-graph capture of the micro step failed ({type(e).__name__}: {e}); running eagerly")
        _NO_GRAPH.setdefault(model, set()).add(shape_key)
        torch.cuda.empty_cache()          # nothing of a failed capture may crowd the eager path
        return None
    if not acc.graph_grads_ok(g.grads):
        _NO_GRAPH.setdefault(model, set()).add(shape_key)
        return None
    return g


def train_mini_batch(model: torch.nn.Module, params: ParameterSet, batch: tuple, plan: MicroBatchPlan,
                     normalization: str, loss_kind: str, optimizer_state: OptimizerState, *,
                     loss_from_logits: bool = True, dice_smoothing: float = 1.0, prefetch: bool = False,
                     accumulator: GradientAccumulator | None = None,
                     lr_for_step: Callable[[int], float] | None = None, tracer=None, **kw) -> tuple:
    """Stream micro-batches, then update once (engine.py:233-261)."""
    x, y = batch
    total, stats = mini_batch_gradient(model, params, x, y, plan, normalization, loss_kind,
                                       loss_from_logits=loss_from_logits, dice_smoothing=dice_smoothing,
                                       prefetch=prefetch, accumulator=accumulator, tracer=tracer,
                                       _close_trace=False, **kw)
    # The reference raises NonFiniteError in the forward, before any update (nn.py:578-579): resolve the
    # mini-batch's device statistics (one D2H, one host wait per mini-batch) BEFORE the step, so neither the
    # parameters nor step_count / the LR schedule move on a non-finite mini-batch.
    stats.resolve()
    if lr_for_step is not None:
        optimizer_state.lr = lr_for_step(optimizer_state.step_count)
    apply_update(params, total, optimizer_state)
    if tracer is not None:
        tracer.update_end()
    stats.step_count = optimizer_state.step_count
    return params, stats


def train_epoch(model: torch.nn.Module, params: ParameterSet, x, y, *, mini_batch_size: int,
                micro_batch_size: int | None, normalization: str, loss_kind: str,
                optimizer_state: OptimizerState, seed: int, epoch_index: int, shuffle: bool = True,
                loss_from_logits: bool = True, dice_smoothing: float = 1.0, prefetch: bool = False,
                lr_for_step: Callable[[int], float] | None = None,
                metric_fn: Callable | None = None, keep_mini_stats: bool = False,
                accumulator: GradientAccumulator | None = None, staging: Staging | None = None,
                autocast_dtype: torch.dtype | None = None, streamer: MicroBatchStreamer | None = None,
                normalize_via: str = "fused", tracer=None) -> EpochStats:
    """One pass over the dataset in the reference's deterministic shuffled order (engine.py:276-335).

    The whole epoch's micro-batch sequence (mini-batch m = order[m*M:(m+1)*M],
    each split by ``plan_split``; the last mini-batch may be short and gets its
    own plan) is streamed as ONE sequence, so the H2D copy of the next
    mini-batch's first micro-batch overlaps the current mini-batch's tail and
    optimizer step. ``micro_batch_size=None`` is the no-MBS baseline.
    """
    x, y = _as_tensor(x), _as_tensor(y)
    n = x.shape[0]
    if n == 0:
        raise ValueError("dataset is empty")
    if normalization not in NORMALIZATION_MODES:
        raise ValueError(f"unknown normalization mode {normalization!r}")
    order = epoch_order(n, seed, epoch_index, shuffle)
    on_device = x.device.type == "cuda"
    if on_device and y.device != x.device:
        y = y.to(x.device)
    order_dev = torch.from_numpy(order.astype(np.int64)).to(x.device) if (on_device and shuffle) else None
    minis, jobs = [], []
    for start in range(0, n, mini_batch_size):
        idx = order[start:start + mini_batch_size]
        n_mu = micro_batch_size if micro_batch_size is not None else len(idx)
        plan = plan_split(len(idx), n_mu)
        minis.append((start, idx, plan))
        for lo, hi in plan.index_ranges:
            if not shuffle:
                jobs.append((None, start + lo, hi - lo))
            elif on_device:
                jobs.append((order_dev[start + lo:start + hi], 0, hi - lo))
            else:
                jobs.append((idx[lo:hi], 0, hi - lo))
    acc = accumulator if accumulator is not None else GradientAccumulator(params)
    own_streamer = None
    if not on_device and streamer is None:
        max_rows = max(p.n_mu for _, _, p in minis)
        streamer = own_streamer = make_streamer(x, y, max_rows)
    model.train()
    dest = _graph_dest(model, acc, loss_kind, autocast_dtype, loss_from_logits, dice_smoothing, normalize_via)
    source = iter(_micro_source(x, y, jobs, staging, prefetch, streamer, dest, tracer))
    mini_sizes, all_stats, mini_metrics = [], [], []
    try:
        for start, idx, plan in minis:
            acc.begin(plan.n_s_mu)
            outputs = _run_micro_loop(model, acc, plan, _take(source, plan.n_s_mu), normalization, loss_kind,
                                      loss_from_logits, dice_smoothing, normalize_via, autocast_dtype,
                                      keep_outputs=metric_fn is not None or keep_mini_stats, tracer=tracer)
            if tracer is not None:
                tracer.update_begin()
            stats_dev = acc.finalize(plan.n_b)
            stats = MiniBatchStats(stats_dev, plan.n_s_mu, acc.max_micro, outputs)
            stats.resolve()     # NonFiniteError before the update, as the reference (nn.py:578-579)
            if lr_for_step is not None:
                optimizer_state.lr = lr_for_step(optimizer_state.step_count)
            apply_update(params, acc.as_gradient_set(), optimizer_state)
            if tracer is not None:
                tracer.update_end()
            stats.step_count = optimizer_state.step_count
            mini_sizes.append(len(idx))
            if metric_fn is not None:
                yb = y[torch.from_numpy(idx.astype(np.int64)).to(y.device)] if on_device else \
                    y[torch.from_numpy(idx.astype(np.int64))]
                mini_metrics.append(float(metric_fn(stats.outputs, yb.to(stats.outputs.device))))
            all_stats.append(stats)
            if not keep_mini_stats:
                stats._outputs = []
    finally:
        if own_streamer is not None:
            own_streamer.close()
    mini_losses = [s.loss for s in all_stats]
    mean_loss = float(np.dot(mini_losses, mini_sizes) / n)
    return EpochStats(mini_losses=mini_losses, mean_loss=mean_loss, mini_metrics=mini_metrics,
                      mini_sizes=mini_sizes, step_count=optimizer_state.step_count,
                      mini_stats=all_stats if keep_mini_stats else [])


def _take(it, n: int):
    for _ in range(n):
        try:
            yield next(it)
        except StopIteration:
            return
