"""The reference's model-spec front end on the B200 stack: a reference ``ModelSpec`` (its layer stacks of
dense / conv2d / relu / batchnorm / flatten / maxpool2d descriptors) becomes a torch module whose training
forward runs on this package's kernels, with the reference's parameter names, layouts and bit-identical
initial values, so a reference user's spec, seed and parameter dictionaries carry over unchanged.

Reference: ``nn.py:33-73`` (descriptors), ``nn.py:76-93`` (``spec_parameter_count``), ``nn.py:125-127``
(``_uniform_fan_in``), ``nn.py:130-425`` (per-layer parameter names, shapes, init and semantics),
``nn.py:427-509`` (``Model`` shape composition, ``build_model``).

* Parameter names and order are the reference's: ``layer{i}.weight`` / ``layer{i}.bias`` for dense and
  conv layers, ``layer{i}.gamma`` / ``layer{i}.beta`` for batchnorm, in layer order. Dense weights keep
  the reference's (in_features, out_features) layout (``y = x @ W + b``, ``nn.py:141,153-157``).
* Initial values: uniform(-sqrt(1/fan_in), +sqrt(1/fan_in)) drawn in float64 from the named Philox
  substream ``init/<name>`` of the seed — the reference's exact draws — then rounded once to fp32;
  gamma = 1, beta = 0.
* Training-mode batchnorm is K5 with MICRO-batch statistics and the reference's biased running variance
  (``nn.py:320-327``; ``MBS_BN_BIASED_RUNNING_VAR``), fused with a directly following ReLU; max-pool is K6
  (the reference pools without padding, first maximum wins, ``nn.py:371-420``); dense / conv run on
  cuBLAS / cuDNN. Eval mode normalises with the running statistics (``nn.py:328-330``).
* Shape composition errors are the reference's ``ShapeCompositionError(layer_index, message)``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.nn.functional as F
from torch import nn

from . import bn as K5
from .errors import ShapeCompositionError
from .pool import swap_maxpool
from .rng import named_stream
from .tensor import ParameterSet


# ---------------------------------------------------------------------------
# Layer descriptors (nn.py:33-73): same names, fields and defaults
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class Dense:
    in_features: int
    out_features: int
    bias: bool = True


@dataclass(frozen=True)
class Conv2d:
    in_channels: int
    out_channels: int
    kernel: int
    stride: int = 1
    padding: int = 0


@dataclass(frozen=True)
class Relu:
    pass


@dataclass(frozen=True)
class BatchNorm:
    features: int
    epsilon: float = 1e-5
    momentum: float = 0.1


@dataclass(frozen=True)
class Flatten:
    pass


@dataclass(frozen=True)
class MaxPool2d:
    kernel: int
    stride: int | None = None  # defaults to kernel


_KINDS = {c.__name__: c for c in (Dense, Conv2d, Relu, BatchNorm, Flatten, MaxPool2d)}


def as_descriptor(entry):
    """This module's descriptor for a spec entry: one of ours, the reference's own dataclass instance (same
    class name and fields), or a plain dict with a ``"type"`` key (the golden fixtures' format)."""
    if isinstance(entry, tuple(_KINDS.values())):
        return entry
    if isinstance(entry, dict):
        kind = entry.get("type")
        fields = {k: v for k, v in entry.items() if k != "type"}
    else:
        kind = type(entry).__name__
        fields = dict(getattr(entry, "__dict__", {}))
    cls = _KINDS.get(kind)
    if cls is None:
        raise TypeError(f"unknown layer descriptor {entry!r}")
    return cls(**fields)


def spec_parameter_count(spec) -> int:
    """Total learnable scalars declared by a model spec (nn.py:76-93)."""
    total = 0
    for entry in map(as_descriptor, spec):
        if isinstance(entry, Dense):
            total += entry.in_features * entry.out_features + (entry.out_features if entry.bias else 0)
        elif isinstance(entry, Conv2d):
            total += entry.out_channels * entry.in_channels * entry.kernel * entry.kernel + entry.out_channels
        elif isinstance(entry, BatchNorm):
            total += 2 * entry.features
    return total


def _uniform_fan_in(seed: int, stream_name: str, shape: tuple, fan_in: int) -> np.ndarray:
    """nn.py:125-127 — float64 draws of the named substream."""
    bound = float(np.sqrt(1.0 / fan_in))
    return named_stream(seed, stream_name).uniform(-bound, bound, size=shape)


def _out_hw(h: int, w: int, k: int, s: int, p: int) -> tuple:
    return (h + 2 * p - k) // s + 1, (w + 2 * p - k) // s + 1


# ---------------------------------------------------------------------------
# Runtime layers (the reference's parameter names and layouts)
# ---------------------------------------------------------------------------

class _Dense(nn.Module):
    def __init__(self, d: Dense):
        super().__init__()
        self.weight = nn.Parameter(torch.empty(d.in_features, d.out_features))     # reference layout (in, out)
        self.bias = nn.Parameter(torch.empty(d.out_features)) if d.bias else None

    def forward(self, x):
        return torch.addmm(self.bias, x, self.weight) if self.bias is not None else x @ self.weight


class _Conv(nn.Module):
    def __init__(self, d: Conv2d):
        super().__init__()
        self.stride, self.padding = d.stride, d.padding
        self.weight = nn.Parameter(torch.empty(d.out_channels, d.in_channels, d.kernel, d.kernel))
        self.bias = nn.Parameter(torch.empty(d.out_channels))

    def forward(self, x):
        return F.conv2d(x, self.weight, self.bias, self.stride, self.padding)


class _BatchNorm(nn.Module):
    def __init__(self, d: BatchNorm):
        super().__init__()
        self.eps, self.momentum = float(d.epsilon), float(d.momentum)
        self.gamma = nn.Parameter(torch.ones(d.features))
        self.beta = nn.Parameter(torch.zeros(d.features))
        self.register_buffer("running_mean", torch.zeros(d.features))
        self.register_buffer("running_var", torch.ones(d.features))
        self.fuse_relu = False

    def forward(self, x):
        if not self.training:                                     # nn.py:328-330: running statistics
            y = F.batch_norm(x, self.running_mean, self.running_var, self.gamma, self.beta, False, 0.0, self.eps)
            return F.relu(y) if self.fuse_relu else y
        if not x.is_cuda:
            raise RuntimeError("refspec BatchNorm: training-mode normalisation runs on the sm_100a K5 kernels "
                               "(libmbs_native.so) and needs a CUDA tensor; there is no CPU fallback")
        return K5.micro_batch_norm(x, self.gamma, self.beta, self.running_mean, self.running_var,
                                   momentum=self.momentum, eps=self.eps, relu=self.fuse_relu,
                                   biased_running_var=True)


class _Relu(nn.Module):
    def __init__(self):
        super().__init__()
        self.fused = False                                        # applied by the preceding K5 batchnorm

    def forward(self, x):
        return x if self.fused else F.relu(x)


class _Flatten(nn.Module):
    def forward(self, x):
        return x.reshape(x.shape[0], -1)


class RefModel(nn.Module):
    """A validated reference layer stack bound to a per-sample input shape (nn.py:427-455); children are
    named ``layer{i}`` so parameter names are the reference's."""

    def __init__(self, spec, input_shape):
        super().__init__()
        self.spec = tuple(as_descriptor(e) for e in spec)
        self.input_shape = tuple(int(d) for d in input_shape)
        if any(d < 1 for d in self.input_shape):
            raise ShapeCompositionError(0, f"input shape {self.input_shape} has non-positive dims")
        shape = self.input_shape
        for i, e in enumerate(self.spec):
            try:
                mod, shape = self._layer(e, shape)
            except ValueError as exc:
                raise ShapeCompositionError(i, str(exc)) from exc
            self.add_module(f"layer{i}", mod)
        self.output_shape = shape
        layers = list(self.children())
        for a, b in zip(layers, layers[1:]):                      # batchnorm -> relu: one K5 pass
            if isinstance(a, _BatchNorm) and isinstance(b, _Relu):
                a.fuse_relu, b.fused = True, True

    @staticmethod
    def _layer(e, shape):
        if isinstance(e, Dense):
            if len(shape) != 1 or shape[0] != e.in_features:
                raise ValueError(f"dense expects per-sample shape ({e.in_features},), got {shape}")
            return _Dense(e), (e.out_features,)
        if isinstance(e, Conv2d):
            if len(shape) != 3 or shape[0] != e.in_channels:
                raise ValueError(f"conv2d expects per-sample shape ({e.in_channels}, H, W), got {shape}")
            h, w = _out_hw(shape[1], shape[2], e.kernel, e.stride, e.padding)
            if h < 1 or w < 1:
                raise ValueError(f"conv2d kernel {e.kernel} stride {e.stride} padding {e.padding} "
                                 f"does not fit input {shape}")
            return _Conv(e), (e.out_channels, h, w)
        if isinstance(e, Relu):
            return _Relu(), shape
        if isinstance(e, BatchNorm):
            if len(shape) not in (1, 3) or shape[0] != e.features:
                raise ValueError(f"batchnorm expects per-sample shape ({e.features},) or ({e.features}, H, W), "
                                 f"got {shape}")
            return _BatchNorm(e), shape
        if isinstance(e, Flatten):
            return _Flatten(), (int(np.prod(shape)),)
        if isinstance(e, MaxPool2d):
            k = e.kernel
            s = e.stride if e.stride is not None else k
            if len(shape) != 3:
                raise ValueError(f"maxpool2d expects per-sample shape (C, H, W), got {shape}")
            h, w = _out_hw(shape[1], shape[2], k, s, 0)
            if h < 1 or w < 1:
                raise ValueError(f"maxpool2d kernel {k} stride {s} does not fit input {shape}")
            return swap_maxpool(nn.MaxPool2d(k, s)), (shape[0], h, w)      # K6 when supported
        raise ValueError(f"unknown layer descriptor {e!r}")

    @property
    def has_batchnorm(self) -> bool:
        return any(isinstance(e, BatchNorm) for e in self.spec)

    def param_shapes(self) -> dict:
        """Reference names -> shapes, in the reference's insertion order (nn.py:457-461)."""
        return {n: tuple(p.shape) for n, p in self.named_parameters()}

    def reset_state(self) -> None:
        """Running statistics back to (0, 1) (nn.py:463-466)."""
        for m in self.modules():
            if isinstance(m, _BatchNorm):
                m.running_mean.zero_()
                m.running_var.fill_(1.0)

    def forward(self, x):
        for m in self.children():
            x = m(x)
        return x


def init_values(model: RefModel, seed: int) -> dict:
    """The reference's float64 initial parameter values for ``model`` (nn.py:146-150, 220-226, 311-313)."""
    out = {}
    for i, e in enumerate(model.spec):
        if isinstance(e, Dense):
            names = [f"layer{i}.weight"] + ([f"layer{i}.bias"] if e.bias else [])
            for n in names:
                shape = (e.in_features, e.out_features) if n.endswith("weight") else (e.out_features,)
                out[n] = _uniform_fan_in(seed, f"init/{n}", shape, e.in_features)
        elif isinstance(e, Conv2d):
            fan_in = e.in_channels * e.kernel * e.kernel
            out[f"layer{i}.weight"] = _uniform_fan_in(seed, f"init/layer{i}.weight",
                                                      (e.out_channels, e.in_channels, e.kernel, e.kernel), fan_in)
            out[f"layer{i}.bias"] = _uniform_fan_in(seed, f"init/layer{i}.bias", (e.out_channels,), fan_in)
        elif isinstance(e, BatchNorm):
            out[f"layer{i}.gamma"] = np.ones(e.features)
            out[f"layer{i}.beta"] = np.zeros(e.features)
    return out


def load_reference_params(model: RefModel, values: dict) -> None:
    """Copy reference-named arrays into the module: a dict of arrays, or a reference ``ParameterSet``
    itself (``tensor.py:77-78`` ``arrays()``)."""
    if callable(getattr(values, "arrays", None)):
        values = values.arrays()
    named = dict(model.named_parameters())
    if set(values) != set(named):
        raise KeyError(f"parameter names differ: {sorted(set(values) ^ set(named))}")
    with torch.no_grad():
        for n, p in named.items():
            v = np.asarray(getattr(values[n], "data", values[n]), dtype=np.float64)
            if v.shape != tuple(p.shape):
                raise ValueError(f"{n}: shape {v.shape} != {tuple(p.shape)}")
            p.copy_(torch.from_numpy(v).to(p.dtype))


def build_model(spec, input_shape, seed: int, *, device=None) -> tuple:
    """nn.py:492-509 on the B200 stack: ``(ParameterSet, RefModel)`` with the reference's names and
    bit-identical (then fp32-rounded) initial values. ``device`` defaults to the current CUDA device."""
    model = RefModel(spec, input_shape)
    load_reference_params(model, init_values(model, seed))
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    model = model.to(dev)
    return ParameterSet(model), model


def reference_arrays(params: ParameterSet) -> dict:
    """The current values as reference-named float64 host arrays (to hand back to reference code)."""
    return {n: params[n].detach().double().cpu().numpy() for n in params.names()}
