"""The reference's own injection seam, served by K1: ``mini_batch_gradient(accumulator=...)``.

The reference's only plug-in point on the hot path is the ``accumulator=`` keyword of
``mini_batch_gradient`` (``engine.py:186``); its loop calls ``accumulator.begin(n_s_mu)``
(``engine.py:202``), ``accumulate(accumulator, grads)`` -> ``accumulator.add(grads)`` once per micro-batch
(``engine.py:216``, ``134-137``) and ``accumulator.as_gradient_set()`` (``engine.py:220``), then
``apply_update`` reads the result (``optim.py:96``). ``ReferenceAccumulator`` has exactly that surface
(plus ``sums`` / ``micro_batches_seen`` / ``expected``, ``engine.py:103-108``) over a flat fp32 HBM buffer:
each ``add`` packs the micro-batch's host gradient arrays into one pinned buffer, copies it to the device
in one transfer and runs ONE K1 launch (``mbs_accum_add``) over every segment; the per-mini-batch result
comes back as the caller's own ``GradientSet`` type with float64 arrays. So the unmodified reference
training loop runs its accumulation on the B200:

    from mbstream import engine                                    # the reference
    from paper_2110_12484_b200.interop import ReferenceAccumulator
    acc = ReferenceAccumulator(params)                             # the reference's ParameterSet
    total, stats = engine.mini_batch_gradient(model, params, x, y, plan, "exact_weighted", "mse",
                                              accumulator=acc)

Differences, by design: the sums are fp32 (the north star's "accumulates in fp32"; rel-L2 ~1e-7 vs the
reference's float64), and ``as_gradient_set()`` / ``sums`` return host COPIES of the device sums rather
than aliases of live arrays (``engine.py:130-131``) — the next ``begin`` does not zero a returned set.
Errors are the reference's: ``AccumulatorOverflowError`` past ``expected`` or on a key-set mismatch
(``engine.py:118-125``).
"""

from __future__ import annotations

import numpy as np
import torch

from .engine import GradientAccumulator
from .errors import AccumulatorOverflowError, GradientKeyMismatchError
from .tensor import ParameterSet, ParamLayout


def _named_shapes(params) -> list:
    """(name, shape) of the grad-required parameters of a reference ParameterSet (``tensor.py:53-96``),
    or of a plain name -> array mapping, in insertion order."""
    out = []
    for name, t in params.items():
        if getattr(t, "grad_required", True):
            shape = getattr(t, "shape", None)
            out.append((name, tuple(shape) if shape is not None else tuple(np.shape(t))))
    if not out:
        raise ValueError("no grad-required parameters")
    return out


class ReferenceAccumulator:
    """``engine.GradientAccumulator``'s surface (engine.py:100-131) on K1 and a flat fp32 HBM buffer."""

    def __init__(self, params, expected: int | None = None, device=None):
        if not torch.cuda.is_available():
            raise RuntimeError("ReferenceAccumulator accumulates on the GPU (libmbs_native.so); no CPU fallback")
        dev = torch.device(device or "cuda")
        named = _named_shapes(params)
        self.names = [n for n, _ in named]
        self.shapes = {n: s for n, s in named}
        self.layout = ParamLayout.build([(n, torch.empty(s, device="meta")) for n, s in named])
        self._pset = ParameterSet(layout=self.layout, flat=torch.zeros(self.layout.total, dtype=torch.float32,
                                                                         device=dev))
        self._acc = GradientAccumulator(self._pset)
        self._host = torch.zeros(self.layout.total, dtype=torch.float32, pin_memory=True)
        self._dev = torch.zeros(self.layout.total, dtype=torch.float32, device=dev)
        self._host_views = {n: self._host[o:o + int(np.prod(s, dtype=np.int64))].view(s) if s else
                            self._host[o:o + 1].view(()) for n, s, o in zip(self.names, self.layout.shapes,
                                                                            self.layout.offsets)}
        self._dev_views = [self.layout.view(self._dev, i) for i in range(len(self.names))]
        self._gset_type = None
        self.expected = None
        if expected is not None:
            self.begin(expected)

    # -- the reference surface --
    def begin(self, expected: int) -> None:
        """engine.py:110-115: zero the sums (folded into the next K1 pass), counter 0, expect N_Smu adds."""
        self._acc.begin(expected)
        self.expected = expected

    def add(self, grads) -> None:
        """engine.py:117-128: sums += grads (one H2D transfer + one K1 launch over every segment)."""
        arrays = grads.arrays if hasattr(grads, "arrays") else dict(grads.items())
        if self.expected is not None and self.micro_batches_seen >= self.expected:
            raise AccumulatorOverflowError(f"already accumulated {self.micro_batches_seen} of {self.expected} "
                                           "micro-batches")
        if set(arrays) != set(self.names):
            raise AccumulatorOverflowError("gradient keys do not match accumulator parameters")
        for n in self.names:
            g = np.asarray(arrays[n])
            if g.shape != self.shapes[n]:
                raise GradientKeyMismatchError(f"gradient shape {g.shape} != parameter shape {self.shapes[n]} "
                                               f"for {n!r}")
        torch.cuda.current_stream(self._dev.device).synchronize()   # the previous transfer has left the buffer
        for n in self.names:
            self._host_views[n].copy_(torch.from_numpy(np.asarray(arrays[n], dtype=np.float64)))
        self._dev.copy_(self._host, non_blocking=True)
        self._acc.add_tensors(self._dev_views, 1.0)
        self._gset_type = type(grads)

    def _download(self) -> dict:
        self._acc._materialize()
        flat = self._acc.flat.detach().to("cpu", torch.float64).numpy()
        return {n: flat[o:o + int(np.prod(s, dtype=np.int64))].reshape(s).copy()
                for n, s, o in zip(self.names, self.layout.shapes, self.layout.offsets)}

    def as_gradient_set(self):
        """engine.py:130-131: the sums as the caller's GradientSet type (float64 host copies)."""
        arrays = self._download()
        t = self._gset_type
        if t is None or t is dict:
            return arrays
        return t(arrays)

    @property
    def sums(self) -> dict:
        return self._download()

    @property
    def micro_batches_seen(self) -> int:
        return self._acc.micro_batches_seen

    @property
    def device_sums(self) -> torch.Tensor:
        """The live flat fp32 accumulator in HBM (for a device-side optimizer step: ``optim.apply_update``)."""
        return self._acc.flat
