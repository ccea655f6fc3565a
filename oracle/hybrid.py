"""Hybrid model oracle — TEST INFRASTRUCTURE ONLY (see mbs_oracle.py header).

The reference's own autograd (``nn.py``) expresses only dense / conv2d / relu /
batchnorm / flatten / maxpool2d stacks (``nn.py:33-73``); it cannot express
ResNet (no residual add) or U-Net (no upsample / concat). For those models the
oracle computes each micro-batch's forward/backward with torch on the CPU in
float64 and feeds the gradient into the float64 MBS arithmetic of
``mbs_oracle`` (plan, factor, accumulator, grad-norm, optimizer). The loss
pullback is the reference's NumPy pullback (``losses.py``), seeded exactly as
``backward(tape, factor)`` seeds it (``nn.py:596``).

SURVEY.md §7 measured this hybrid against the pure reference at <= 8.6e-16
max-rel where both run; ``tests/test_oracle_golden.py`` re-checks it against the
reference-generated fixtures.
"""

from __future__ import annotations

import copy

import numpy as np
import torch

from . import mbs_oracle as O


class TorchGradFn:
    """``grad_fn(xk, yk, seed) -> (loss, grads, out)`` over a float64 CPU copy of a module."""

    def __init__(self, module: torch.nn.Module, loss_kind: str, *, from_logits: bool = True,
                 dice_smoothing: float = 1.0, dtype=torch.float64):
        self.module = copy.deepcopy(module).to("cpu", dtype)
        self.module.train()
        self.loss_kind = loss_kind
        self.from_logits = from_logits
        self.dice_smoothing = dice_smoothing
        self.dtype = dtype
        self.names = [n for n, p in self.module.named_parameters() if p.requires_grad]

    def params(self) -> dict:
        """Live float64 numpy views of the module parameters (mutated by the optimizer)."""
        return {n: p.data.numpy() for n, p in self.module.named_parameters() if p.requires_grad}

    def __call__(self, xk, yk, seed):
        xt = torch.as_tensor(np.asarray(xk)).to(self.dtype)
        for p in self.module.parameters():
            p.grad = None
        out = self.module(xt)
        val, gout = O.compute_loss(self.loss_kind, out.detach().numpy(), yk,
                                   self.from_logits, self.dice_smoothing)
        out.backward(torch.from_numpy(seed * gout).to(self.dtype))
        grads = {n: p.grad.detach().numpy().astype(np.float64).copy()
                 for n, p in self.module.named_parameters() if p.requires_grad}
        return val, grads, out.detach().numpy()
