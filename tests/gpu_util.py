"""Helpers for the GPU parity tests."""
import numpy as np
import torch
from torch import nn


class Bag(nn.Module):
    """A module holding free parameters of given shapes (names p0, p1, ...)."""

    def __init__(self, shapes, device, seed=0, channels_last_4d=False):
        super().__init__()
        g = torch.Generator().manual_seed(seed)
        for i, s in enumerate(shapes):
            t = torch.randn(*s, generator=g).to(device)
            if channels_last_4d and len(s) == 4:
                t = t.contiguous(memory_format=torch.channels_last)
            setattr(self, f"p{i}", nn.Parameter(t))


def rel_l2(a, b):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    d = np.linalg.norm(a - b)
    n = np.linalg.norm(b)
    return d / n if n > 0 else d


def to64(t):
    return t.detach().double().cpu().numpy()
