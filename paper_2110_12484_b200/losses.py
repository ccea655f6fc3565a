"""Mean-reduced losses and metrics on device — ``losses.py`` semantics in torch ops.

Losses are NOT a hot-path kernel ("losses stay torch ops"); what
matters for MBS is the contract that every loss is the MEAN over the
micro-batch (``losses.py:1-8``), which makes the normalised accumulation
exact. Each function states the reference lines whose value and gradient it
reproduces (autograd gives the same pullback as the reference's explicit
one).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.nn.functional as F

PROB_CLAMP = 1e-12  # losses.py:17
LOSS_KINDS = ("mse", "cross_entropy", "bce", "bce_dice")  # losses.py:19


@dataclass
class LossValue:
    """losses.py:24-36 — a mean-reduced scalar (kept on device as a 0-d tensor)."""

    value: torch.Tensor
    n_samples: int
    reduction: str = "mean"


def _check_same_shape(output, target, kind):
    if tuple(output.shape) != tuple(target.shape):
        raise ValueError(f"{kind}: output shape {tuple(output.shape)} != target shape {tuple(target.shape)}")


def mse(output: torch.Tensor, target: torch.Tensor) -> torch.Tensor:
    """losses.py:72-75: mean((o-t)^2); grad 2(o-t)/size."""
    _check_same_shape(output, target, "mse")
    output = output.float() if output.dtype in (torch.bfloat16, torch.float16) else output
    d = output - target.to(output.dtype)
    return (d * d).mean()


def cross_entropy(logits: torch.Tensor, classes: torch.Tensor) -> torch.Tensor:
    """losses.py:78-87: mean NLL of log-softmax; grad (softmax - onehot)/n."""
    if logits.dim() != 2 or classes.dim() != 1 or classes.shape[0] != logits.shape[0]:
        raise ValueError(f"cross_entropy expects logits (N, K) and class indices (N,), got "
                         f"{tuple(logits.shape)} and {tuple(classes.shape)}")
    return F.cross_entropy(logits.float() if logits.dtype in (torch.bfloat16, torch.float16) else logits,
                           classes.long())


def bce_logits(z: torch.Tensor, target: torch.Tensor) -> torch.Tensor:
    """losses.py:98-102: mean(max(z,0) - z t + log1p(exp(-|z|))); grad (sigmoid(z)-t)/size."""
    z = z.float() if z.dtype in (torch.bfloat16, torch.float16) else z
    return F.binary_cross_entropy_with_logits(z, target.to(z.dtype))


def bce_probs(p: torch.Tensor, target: torch.Tensor) -> torch.Tensor:
    """losses.py:90-95: clamp to [1e-12, 1-1e-12]; zero gradient outside the clamp."""
    p = p.float() if p.dtype in (torch.bfloat16, torch.float16) else p
    c = p.clamp(PROB_CLAMP, 1.0 - PROB_CLAMP)
    t = target.to(p.dtype)
    return -(t * torch.log(c) + (1.0 - t) * torch.log1p(-c)).mean()


def dice_soft(p: torch.Tensor, target: torch.Tensor, smoothing: float) -> torch.Tensor:
    """losses.py:105-114: per-sample soft dice loss, batch-mean."""
    n = p.shape[0]
    pf, gf = p.reshape(n, -1), target.reshape(n, -1).to(p.dtype)
    num = 2.0 * (pf * gf).sum(dim=1) + smoothing
    den = pf.sum(dim=1) + gf.sum(dim=1) + smoothing
    return (1.0 - num / den).mean()


def compute_loss(kind: str, output: torch.Tensor, target: torch.Tensor, *, from_logits: bool = True,
                 dice_smoothing: float = 1.0) -> torch.Tensor:
    """Training-loop dispatch (losses.py:184-207). Returns a 0-d device tensor, always computed and
    returned in fp32 (or fp64) even when the model output is bf16/fp16 (autocast): the 1e-12 clamp of
    ``bce`` and the mean reductions need it, and K1 reads the loss as fp32."""
    if kind == "mse":
        return mse(output, target)
    if kind == "cross_entropy":
        return cross_entropy(output, target)
    if kind == "bce":
        _check_same_shape(output, target, kind)
        return bce_logits(output, target) if from_logits else bce_probs(output, target)
    if kind == "bce_dice":
        _check_same_shape(output, target, kind)
        z = output.float() if output.dtype in (torch.bfloat16, torch.float16) else output
        if from_logits:
            return bce_logits(z, target) + dice_soft(torch.sigmoid(z), target, dice_smoothing)
        return bce_probs(z, target) + dice_soft(z, target, dice_smoothing)
    raise ValueError(f"unknown loss kind {kind!r}")


# ---------------------------------------------------------------------------
# Metrics (losses.py:214-263)
# ---------------------------------------------------------------------------

def _set_ratio(a: torch.Tensor, b: torch.Tensor, kind: str) -> torch.Tensor:
    inter = (a & b).sum(dim=-1).double()
    if kind == "dice":
        total = (a.sum(dim=-1) + b.sum(dim=-1)).double()
        return torch.where(total == 0, torch.ones_like(total), 2.0 * inter / total.clamp_min(1))
    union = (a | b).sum(dim=-1).double()
    return torch.where(union == 0, torch.ones_like(union), inter / union.clamp_min(1))


def _mask_metric(prediction, ground_truth, threshold, kind, per_image) -> float:
    if not 0.0 < threshold < 1.0:
        raise ValueError(f"threshold must lie in (0, 1), got {threshold}")
    a = ground_truth > 0.5
    b = prediction > threshold
    if per_image:
        n = a.shape[0]
        return float(_set_ratio(a.reshape(n, -1), b.reshape(n, -1), kind).mean().item())
    return float(_set_ratio(a.reshape(1, -1), b.reshape(1, -1), kind)[0].item())


def dice_coefficient(prediction, ground_truth, threshold: float = 0.5, per_image: bool = False) -> float:
    """losses.py:246-254 — 2|A.B|/(|A|+|B|) on thresholded masks; 1.0 when both are empty."""
    return _mask_metric(prediction, ground_truth, threshold, "dice", per_image)


def iou(prediction, ground_truth, threshold: float = 0.5, per_image: bool = False) -> float:
    """losses.py:257-259 — |A.B|/|A+B| on thresholded masks; 1.0 when both are empty."""
    return _mask_metric(prediction, ground_truth, threshold, "iou", per_image)


def accuracy(output: torch.Tensor, target: torch.Tensor) -> float:
    """losses.py:262-272 — argmax accuracy (ties toward the lowest class index)."""
    if output.dim() != 2 or output.shape[1] < int(target.max().item()) + 1:
        raise ValueError(f"output shape {tuple(output.shape)} cannot score the target classes")
    return float((output.argmax(dim=1) == target.to(output.device)).double().mean().item())
