"""One forward+backward of K5 on representative ResNet-50 / U-Net BatchNorm layers (for ncu capture).

ncu --set full -k regex:k_bn python tools/k5_ncu.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2110_12484_b200 import bn as K5  # noqa: E402

SHAPES = [((128, 256, 56, 56), True), ((128, 64, 56, 56), False), ((128, 1024, 14, 14), True),
          ((128, 2048, 7, 7), True)]


def main():
    dev = torch.device("cuda")
    flush = torch.empty(512 * 2 ** 20, dtype=torch.uint8, device=dev)
    for shape, res in SHAPES:
        x = torch.randn(shape, device=dev, dtype=torch.bfloat16).contiguous(memory_format=torch.channels_last)
        r = torch.randn_like(x).requires_grad_(True) if res else None
        dy = torch.randn_like(x)
        w = torch.ones(shape[1], device=dev, requires_grad=True)
        b = torch.zeros(shape[1], device=dev, requires_grad=True)
        xx = x.requires_grad_(True)
        flush.zero_()
        y = K5.micro_batch_norm(xx, w, b, relu=True, residual=r)
        flush.zero_()
        y.backward(dy)
        torch.cuda.synchronize()


if __name__ == "__main__":
    main()
