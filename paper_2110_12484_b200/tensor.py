"""Flat device parameter / gradient sets — the B200 form of ``tensor.py:53-146``.

The reference keeps one float64 NumPy array per parameter name
(``ParameterSet``, ``tensor.py:53-96``) and per-parameter gradient dicts
(``GradientSet``, ``tensor.py:99-146``). On the B200 every trainable
parameter of a torch module is re-homed into ONE flat fp32 HBM buffer
(segment i at a 128-byte aligned offset), and the module's parameters become
views into it. The accumulator, the optimizer state and the all-reduce use
the same layout, so the accumulate (K1), optimizer (K3) and NCCL passes are
single flat sweeps; names map to (offset, shape, stride) exactly once, at
setup (the shim-side ``validate_against``).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Iterator

import torch

from .errors import GradientKeyMismatchError

ALIGN = 32  # floats: every segment starts on a 128-byte boundary


def _is_dense(t: torch.Tensor) -> bool:
    return t.is_contiguous() or (t.dim() == 4 and t.is_contiguous(memory_format=torch.channels_last))


@dataclass(frozen=True)
class ParamLayout:
    """name -> (offset, shape, stride) table of a flat parameter buffer."""

    names: tuple
    shapes: tuple
    strides: tuple
    offsets: tuple
    numels: tuple
    total: int  # padded element count (multiple of ALIGN)

    @staticmethod
    def build(named: list) -> "ParamLayout":
        names, shapes, strides, offsets, numels = [], [], [], [], []
        off = 0
        for name, t in named:
            if not _is_dense(t):
                raise ValueError(f"parameter {name!r} must be contiguous or channels_last")
            names.append(name)
            shapes.append(tuple(t.shape))
            strides.append(tuple(t.stride()))
            offsets.append(off)
            numels.append(t.numel())
            off += (t.numel() + ALIGN - 1) // ALIGN * ALIGN
        total = max(off, ALIGN)
        return ParamLayout(tuple(names), tuple(shapes), tuple(strides), tuple(offsets), tuple(numels), total)

    def view(self, flat: torch.Tensor, i: int) -> torch.Tensor:
        return flat.as_strided(self.shapes[i], self.strides[i], flat.storage_offset() + self.offsets[i])

    def views(self, flat: torch.Tensor) -> dict:
        return {n: self.view(flat, i) for i, n in enumerate(self.names)}

    def index(self, name: str) -> int:
        return self.names.index(name)

    @property
    def n_params(self) -> int:
        return sum(self.numels)


class ParameterSet:
    """Ordered, uniquely named fp32 parameters backed by one flat HBM buffer.

    ``ParameterSet(module)`` moves every ``requires_grad`` parameter of the
    module into ``self.flat`` (the module keeps working unchanged: its
    parameters become views). Iteration order is the module's registration
    order — the reference's insertion order (``tensor.py:53-58``).
    """

    def __init__(self, module: torch.nn.Module | None = None, *, layout: ParamLayout | None = None,
                 flat: torch.Tensor | None = None, device=None, shadow: torch.dtype | None = None):
        """``shadow=torch.bfloat16``: bf16 shadow-weight mode for bf16-autocast training. Every matmul
        weight (``dim >= 2``: conv / linear) of the module is replaced by a bf16 Parameter viewing a
        flat bf16 shadow of the fp32 master buffer; the forward reads it directly (no per-forward
        autocast cast), its gradient stays bf16 (no fp32 conversion pass: K1 widens it), and the
        optimizer step (K3) writes the rounded bf16 copy of the updated master in the same pass.
        ``params[name]`` keeps returning the fp32 master. Call ``sync_shadow()`` after modifying
        masters outside the optimizer (``load_`` does it)."""
        self.module = module
        self.shadow = None
        self.grad_params = None
        if module is not None:
            named = [(n, p) for n, p in module.named_parameters() if p.requires_grad]
            if not named:
                raise ValueError("module has no trainable parameters")
            for n, p in named:
                if p.dtype != torch.float32:
                    raise ValueError(f"parameter {n!r} must be float32 (got {p.dtype}); keep master "
                                     "weights fp32 and use autocast for low-precision compute")
            dev = torch.device(device) if device is not None else named[0][1].device
            if dev.type != "cuda":
                raise ValueError("ParameterSet lives in HBM: move the module to a CUDA device first")
            self.layout = ParamLayout.build(named)
            self.flat = torch.zeros(self.layout.total, dtype=torch.float32, device=dev)
            self._params = {}
            with torch.no_grad():
                for i, (n, p) in enumerate(named):
                    v = self.layout.view(self.flat, i)
                    v.copy_(p.data)
                    p.data = v
                    self._params[n] = p
            self.grad_params = [p for _, p in named]
            if shadow is not None:
                if shadow != torch.bfloat16:
                    raise ValueError("shadow weights are bfloat16")
                self.shadow = torch.zeros(self.layout.total, dtype=torch.bfloat16, device=dev)
                for i, (n, p) in enumerate(named):
                    if p.dim() < 2:
                        continue
                    owner, _, attr = n.rpartition(".")
                    sub = module.get_submodule(owner) if owner else module
                    sp = torch.nn.Parameter(self.layout.view(self.shadow, i))
                    setattr(sub, attr, sp)
                    self.grad_params[i] = sp
                self.sync_shadow()
        else:
            if layout is None or flat is None:
                raise ValueError("ParameterSet needs a module, or a layout and a flat buffer")
            self.layout = layout
            self.flat = flat
            self._params = layout.views(flat)

    # -- reference ParameterSet surface (tensor.py:53-96) --
    def names(self) -> list:
        return list(self.layout.names)

    def items(self) -> Iterator:
        return iter(self._params.items())

    def arrays(self) -> dict:
        return {n: (p.data if isinstance(p, torch.nn.Parameter) else p) for n, p in self._params.items()}

    def copy(self) -> "ParameterSet":
        """Detached snapshot with the same layout (not bound to the module)."""
        return ParameterSet(layout=self.layout, flat=self.flat.detach().clone())

    def total_elements(self) -> int:
        return self.layout.n_params

    def __getitem__(self, name: str):
        return self._params[name]

    def __contains__(self, name: str) -> bool:
        return name in self._params

    def __len__(self) -> int:
        return len(self._params)

    def __iter__(self):
        return iter(self.layout.names)

    def sync_shadow(self) -> None:
        """Refresh the bf16 shadow from the fp32 masters (round-to-nearest-even, like autocast's cast)."""
        if self.shadow is not None:
            with torch.no_grad():
                self.shadow.copy_(self.flat)

    def load_(self, other: "ParameterSet | dict") -> None:
        """Copy values in (from a snapshot or a name -> tensor/array dict)."""
        with torch.no_grad():
            if isinstance(other, ParameterSet) and other.layout == self.layout:
                self.flat.copy_(other.flat)
                self.sync_shadow()
                return
            for i, n in enumerate(self.layout.names):
                src = other[n]
                src = src.data if isinstance(src, torch.nn.Parameter) else src
                self.layout.view(self.flat, i).copy_(torch.as_tensor(src))
        self.sync_shadow()

    @property
    def device(self):
        return self.flat.device


class GradientSet:
    """Per-parameter gradients keyed by name (``tensor.py:99-146``).

    When produced by the accumulator it aliases the accumulator's flat buffer
    (``as_gradient_set`` aliases the live sums, engine.py:130-131)
    and carries that buffer (``flat``/``layout``) so the optimizer runs as one
    flat pass, plus the device grad-norm guard of the last finalize.
    """

    def __init__(self, arrays: dict | None = None, *, flat: torch.Tensor | None = None,
                 layout: ParamLayout | None = None, norm2: torch.Tensor | None = None):
        self.arrays = dict(arrays or {})
        self.flat = flat
        self.layout = layout
        self.norm2 = norm2  # 0-d float64 device tensor (||g||^2), when known

    def __getitem__(self, name):
        return self.arrays[name]

    def __contains__(self, name):
        return name in self.arrays

    def __len__(self):
        return len(self.arrays)

    def keys(self):
        return self.arrays.keys()

    def items(self):
        return self.arrays.items()

    def copy(self) -> "GradientSet":
        if self.flat is not None:
            flat = self.flat.clone()
            return GradientSet(self.layout.views(flat), flat=flat, layout=self.layout)
        return GradientSet({n: g.clone() for n, g in self.arrays.items()})

    def scaled(self, factor: float) -> "GradientSet":
        return GradientSet({n: g * factor for n, g in self.arrays.items()})

    def l2_norm(self) -> float:
        """sqrt(sum_params dot(g, g)) in float64 (tensor.py:126-130)."""
        if self.norm2 is not None:
            return float(torch.sqrt(self.norm2).item())
        total = torch.zeros((), dtype=torch.float64, device=next(iter(self.arrays.values())).device)
        for g in self.arrays.values():
            gd = g.detach().reshape(-1).double()
            total += torch.dot(gd, gd)
        return float(torch.sqrt(total).item())

    def validate_against(self, params: ParameterSet) -> None:
        """Keys equal the parameter names; shapes match (tensor.py:132-146)."""
        expected = set(params.names())
        got = set(self.arrays)
        if expected != got:
            raise GradientKeyMismatchError(
                f"gradient keys do not match parameters (missing={sorted(expected - got)}, "
                f"extra={sorted(got - expected)})")
        for name, g in self.arrays.items():
            if tuple(g.shape) != tuple(params[name].shape):
                raise GradientKeyMismatchError(
                    f"gradient shape {tuple(g.shape)} != parameter shape {tuple(params[name].shape)} "
                    f"for {name!r}")

    def flat_for(self, layout: ParamLayout) -> torch.Tensor:
        """The gradient as one flat fp32 buffer in ``layout`` (zero-copy when already flat)."""
        if self.flat is not None and self.layout == layout:
            return self.flat
        dev = next(iter(self.arrays.values())).device
        flat = torch.zeros(layout.total, dtype=torch.float32, device=dev)
        for i, n in enumerate(layout.names):
            layout.view(flat, i).copy_(self.arrays[n])
        return flat
