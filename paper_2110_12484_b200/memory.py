"""Micro-batch auto-sizing against MEASURED free HBM — ``memory.py:24-101`` semantics.

The reference bills an analytic float64 byte model of a simulated device
(``memory.py:18-21,59-85``) and picks ``n = (capacity - resident) //
per_sample`` (``fit_micro_batch``, ``memory.py:88-101``). On the B200 the same
rule is fed with measured quantities: capacity = free HBM reported by
``cudaMemGetInfo`` (plus what this process already holds), resident = the
flat parameter / accumulator / optimizer buffers actually allocated, and
per-sample bytes = the slope of the peak allocated memory of one training
micro-step between two probe sizes (activations, workspaces, staged input).
"""

from __future__ import annotations

from contextlib import nullcontext
from dataclasses import dataclass

import torch

from .errors import ModelDoesNotFitError
from .losses import compute_loss

_OPTIMIZER_SLOTS = {"sgd": 1, "adam": 2}   # memory.py:21


@dataclass(frozen=True)
class MemoryBudget:
    """memory.py:24-49 — byte accounting against a device capacity."""

    capacity_bytes: int
    param_bytes: int
    data_bytes_per_sample: int
    fixed_overhead_bytes: int = 0

    def __post_init__(self):
        if self.capacity_bytes <= 0:
            raise ValueError("capacity_bytes must be positive")
        if self.data_bytes_per_sample <= 0:
            raise ValueError("data_bytes_per_sample must be positive")
        if min(self.param_bytes, self.fixed_overhead_bytes) < 0:
            raise ValueError("byte counts must be non-negative")

    @property
    def resident_bytes(self) -> int:
        return self.param_bytes + self.fixed_overhead_bytes

    def bytes_for(self, n_samples: int) -> int:
        return self.resident_bytes + n_samples * self.data_bytes_per_sample

    def fits(self, n_samples: int) -> bool:
        return self.bytes_for(n_samples) <= self.capacity_bytes


def optimizer_state_multiplier(optimizer_kind: str) -> int:
    """memory.py:52-56."""
    try:
        return _OPTIMIZER_SLOTS[optimizer_kind]
    except KeyError:
        raise ValueError(f"unknown optimizer kind {optimizer_kind!r}") from None


def fit_micro_batch(budget: MemoryBudget) -> int:
    """Largest micro-batch whose data space fits beside the model (memory.py:88-101)."""
    free = budget.capacity_bytes - budget.resident_bytes
    n = free // budget.data_bytes_per_sample
    if n < 1:
        raise ModelDoesNotFitError(
            f"device capacity {budget.capacity_bytes} cannot hold the model ({budget.resident_bytes} resident "
            f"bytes) plus one sample ({budget.data_bytes_per_sample} bytes/sample)")
    return int(n)


def parameter_space_bytes(n_params: int, optimizer_kind: str, bytes_per_element: int = 4) -> int:
    """Parameters + accumulated gradient + optimizer slots (memory.py:59-62, fp32 on the B200)."""
    return bytes_per_element * n_params * (2 + optimizer_state_multiplier(optimizer_kind))


def _probe_peak(model, make_batch, n: int, loss_kind: str, autocast_dtype, device) -> int:
    x, y = make_batch(n)
    torch.cuda.synchronize(device)
    torch.cuda.reset_peak_memory_stats(device)
    base = torch.cuda.memory_allocated(device)
    ctx = torch.autocast("cuda", dtype=autocast_dtype) if autocast_dtype is not None else nullcontext()
    with ctx:
        loss = compute_loss(loss_kind, model(x), y)
    loss.backward()
    for p in model.parameters():
        p.grad = None
    torch.cuda.synchronize(device)
    peak = torch.cuda.max_memory_allocated(device) - base
    del x, y, loss
    return int(peak)


def measure_budget(model: torch.nn.Module, make_batch, loss_kind: str, *, optimizer_kind: str = "sgd",
                   autocast_dtype=None, probe: tuple = (2, 4), safety: float = 0.92, device=None,
                   baseline_bytes: int = 0) -> MemoryBudget:
    """Measured ``MemoryBudget`` for training ``model`` on this GPU.

    ``make_batch(n)`` returns a device (x, y) micro-batch of n samples already
    staged the way training will stage it. Per-sample bytes = slope of the
    probe peaks; fixed overhead = the intercept (cuDNN workspaces, the
    per-micro gradient tensors). ``safety`` keeps a margin for allocator
    fragmentation. ``baseline_bytes``: device bytes allocated before the model
    was placed (other tensors of the process), excluded from what is resident.
    """
    device = torch.device(device or "cuda")
    model.train()
    n1, n2 = probe
    p1 = _probe_peak(model, make_batch, n1, loss_kind, autocast_dtype, device)
    p2 = _probe_peak(model, make_batch, n2, loss_kind, autocast_dtype, device)
    per_sample = max(1, (p2 - p1) // (n2 - n1))
    overhead = max(0, p1 - n1 * per_sample)
    free, _total = torch.cuda.mem_get_info(device)
    n_params = sum(p.numel() for p in model.parameters() if p.requires_grad)
    held = max(0, torch.cuda.memory_allocated(device) - int(baseline_bytes))
    capacity = int((free + held) * safety)
    # what is already resident (params, accumulator, optimizer state) is part of `held`
    resident = max(held, parameter_space_bytes(n_params, optimizer_kind))
    return MemoryBudget(capacity_bytes=capacity, param_bytes=resident, data_bytes_per_sample=int(per_sample),
                        fixed_overhead_bytes=int(overhead))


def bn_safe_micro_batch(n_b: int, n_mu: int) -> int:
    """Largest micro-batch size <= n_mu whose plan (engine.py:56-78) has no 1-sample micro-batch.

    The reference allows a 1-sample tail (e.g. 33/16 -> [16, 16, 1]; eps-guarded BatchNorm).
    K5 (``bn.MicroBatchNorm2d``) follows the reference there, but torch's stock BatchNorm raises when a
    channel then holds a single value (BatchNorm1d, or 1x1 spatial maps). ``auto_micro_batch`` applies
    this guard for models that still contain stock torch BatchNorm layers; the plan of a given
    (n_b, n_mu) is never altered.
    """
    if n_b < 1 or n_mu < 1:
        raise ValueError("batch sizes must be positive")
    if n_b == 1:
        return 1
    m = min(n_mu, n_b)
    while m > 1 and n_b % m == 1:
        m -= 1
    return m


def has_stock_batchnorm(model: torch.nn.Module) -> bool:
    """Whether a training-mode forward may run torch's own BatchNorm (which rejects 1-value channels)."""
    from .bn import MicroBatchNorm2d
    return any(isinstance(m, torch.nn.modules.batchnorm._BatchNorm) and not isinstance(m, MicroBatchNorm2d)
               for m in model.modules())


def auto_micro_batch(budget: MemoryBudget, n_b: int, model: torch.nn.Module | None = None) -> int:
    """The micro-batch for a mini-batch of ``n_b``: ``fit_micro_batch`` (memory.py:88-101) capped at n_b,
    then, for models with stock torch BatchNorm, the largest size <= that with no 1-sample micro-batch
    (``bn_safe_micro_batch``)."""
    n = min(fit_micro_batch(budget), int(n_b))
    if model is not None and has_stock_batchnorm(model):
        n = bn_safe_micro_batch(int(n_b), n)
    return n
