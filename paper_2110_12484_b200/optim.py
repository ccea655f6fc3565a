"""Optimizer step from the accumulated gradient — ``optim.py`` on flat HBM buffers (K3).

``sgd_step`` (``optim.py:52-65``) and ``adam_step`` (``optim.py:68-93``), both
with weight decay coupled into the gradient, run as ONE fused, vectorised
sweep over the flat parameter buffer (``mbs_sgd_step`` / ``mbs_adam_step``):
SGD reads grad, w, v and writes w, v (20 B/param); Adam reads grad, w, m, v
and writes w, m, v (28 B/param). The step counter increments exactly once per
mini-batch (``optim.py:65,93``; the deferred-update contract).

The moment buffers are created lazily as zeros on the first step, as the
reference does (``optim.py:58-61,78-83``); ``velocity`` / ``first_moment`` /
``second_moment`` expose them as name -> view dicts.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import torch

from . import _native as N
from .prof import TIMER
from .tensor import GradientSet, ParameterSet


@dataclass
class OptimizerState:
    """optim.py:17-37 (same fields; moments are flat device buffers)."""

    kind: str  # "sgd" | "adam"
    lr: float
    momentum: float = 0.0
    weight_decay: float = 0.0
    adam_beta1: float = 0.9
    adam_beta2: float = 0.999
    adam_eps: float = 1e-8
    step_count: int = 0
    _flat: dict = field(default_factory=dict, repr=False)
    _layout: object = field(default=None, repr=False)

    def __post_init__(self):
        if self.kind not in ("sgd", "adam"):
            raise ValueError(f"unknown optimizer kind {self.kind!r}")
        if self.lr <= 0:
            raise ValueError("learning rate must be positive")
        if self.momentum < 0 or self.weight_decay < 0:
            raise ValueError("momentum and weight_decay must be non-negative")

    def _buffers(self, params: ParameterSet, names: tuple) -> list:
        if self._layout is not None and self._layout != params.layout:
            raise ValueError("optimizer state was created for a different parameter layout")
        self._layout = params.layout
        out = []
        for n in names:
            if n not in self._flat:
                self._flat[n] = torch.zeros(params.layout.total, dtype=torch.float32, device=params.device)
            out.append(self._flat[n])
        return out

    def _views(self, name: str) -> dict:
        if name not in self._flat:
            return {}
        return self._layout.views(self._flat[name])

    @property
    def velocity(self) -> dict:
        return self._views("velocity")

    @property
    def first_moment(self) -> dict:
        return self._views("first_moment")

    @property
    def second_moment(self) -> dict:
        return self._views("second_moment")


def sgd_state(lr: float = 0.01, momentum: float = 0.9, weight_decay: float = 0.0005) -> OptimizerState:
    """optim.py:40-42."""
    return OptimizerState(kind="sgd", lr=lr, momentum=momentum, weight_decay=weight_decay)


def adam_state(lr: float = 0.01, weight_decay: float = 0.0005, beta1: float = 0.9, beta2: float = 0.999,
               eps: float = 1e-8) -> OptimizerState:
    """optim.py:45-49."""
    return OptimizerState(kind="adam", lr=lr, weight_decay=weight_decay, adam_beta1=beta1, adam_beta2=beta2,
                          adam_eps=eps)


def _stream_ptr(stream=None) -> int:
    return (stream or torch.cuda.current_stream()).cuda_stream


def _shadow_ptr(params: ParameterSet):
    """The bf16 shadow K3 refreshes in the same pass (shadow-weight mode), else None."""
    sh = getattr(params, "shadow", None)
    return sh.data_ptr() if sh is not None else None


def _guard_ptr(grads: GradientSet):
    return grads.norm2.data_ptr() if grads.norm2 is not None else None


def sgd_step(params: ParameterSet, grads: GradientSet, state: OptimizerState, *, stream=None) -> None:
    """g' = g + wd*w; v = momentum*v + g'; w -= lr*v (optim.py:52-65)."""
    grads.validate_against(params)
    g = grads.flat_for(params.layout)
    (v,) = state._buffers(params, ("velocity",))
    t0 = TIMER.start(stream)
    N.check(N.lib().mbs_sgd_step(params.flat.data_ptr(), g.data_ptr(), v.data_ptr(), params.layout.total,
                                 float(state.lr), float(state.momentum), float(state.weight_decay),
                                 _guard_ptr(grads), _shadow_ptr(params), _stream_ptr(stream)), "mbs_sgd_step")
    # algorithmic bytes: read g, w, v; write w, v (20 B/param) + the bf16 shadow write (2 B/param) if any
    TIMER.stop("k3_sgd", t0, (20 + 2 * (_shadow_ptr(params) is not None)) * params.layout.n_params, stream)
    state.step_count += 1


def adam_step(params: ParameterSet, grads: GradientSet, state: OptimizerState, *, stream=None) -> None:
    """Bias-corrected Adam, weight decay added to the gradient (optim.py:68-93)."""
    grads.validate_against(params)
    g = grads.flat_for(params.layout)
    m, v = state._buffers(params, ("first_moment", "second_moment"))
    t = state.step_count + 1
    t0 = TIMER.start(stream)
    N.check(N.lib().mbs_adam_step(params.flat.data_ptr(), g.data_ptr(), m.data_ptr(), v.data_ptr(),
                                  params.layout.total, float(state.lr), float(state.adam_beta1),
                                  float(state.adam_beta2), float(state.adam_eps), float(state.weight_decay), t,
                                  _guard_ptr(grads), _shadow_ptr(params), _stream_ptr(stream)), "mbs_adam_step")
    TIMER.stop("k3_adam", t0, (28 + 2 * (_shadow_ptr(params) is not None)) * params.layout.n_params, stream)
    state.step_count = t


def apply_update(params: ParameterSet, grads: GradientSet, state: OptimizerState, *, stream=None) -> None:
    """One optimizer step; exactly one step_count increment (optim.py:96-101)."""
    if state.kind == "sgd":
        sgd_step(params, grads, state, stream=stream)
    else:
        adam_step(params, grads, state, stream=stream)


def linear_lr(initial_lr: float, step: int, total_steps: int) -> float:
    """optim.py:104-110: initial * (1 - step/total), never negative."""
    if total_steps <= 0:
        raise ValueError("total_steps must be positive")
    if not 0 <= step <= total_steps:
        raise ValueError(f"step {step} outside [0, {total_steps}]")
    return max(0.0, initial_lr * (1.0 - step / total_steps))
