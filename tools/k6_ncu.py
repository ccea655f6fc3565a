"""One call each of K6 max-pool fwd/bwd (+stash/addend), the channel-slice copy and K7 im2col at model shapes (for ncu).

ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:"k_maxpool|k_copy|k_im2col" python tools/k6_ncu.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2110_12484_b200 import pool as K6  # noqa: E402
from paper_2110_12484_b200 import stem as K7  # noqa: E402


def main():
    dev = torch.device("cuda")
    bf = torch.bfloat16
    cl = torch.channels_last
    # ResNet stem max-pool 3x3/s2/p1
    x = torch.randn(128, 64, 112, 112, device=dev, dtype=bf).contiguous(memory_format=cl).requires_grad_(True)
    y = K6.max_pool2d(x, 3, 2, 1)
    y.backward(torch.randn_like(y))
    # U-Net level-0 pool + stash + join (48 x 64 x 384 x 384)
    s = torch.randn(48, 64, 384, 384, device=dev, dtype=bf).contiguous(memory_format=cl).requires_grad_(True)
    p, buf = K6.pool_and_stash(s, 2, 64)
    up = torch.randn(48, 64, 384, 384, device=dev, dtype=bf).contiguous(memory_format=cl).requires_grad_(True)
    bias = torch.zeros(64, device=dev, requires_grad=True)
    j = K6.join_skip(buf, up, bias)
    (p.float().sum() + j.float().sum()).backward()
    # ResNet stem conv im2col
    conv = K7.swap_stem(torch.nn.Conv2d(3, 64, 7, 2, 3, bias=False).to(dev))
    xi = torch.randn(128, 3, 224, 224, device=dev, dtype=bf).contiguous(memory_format=cl)
    with torch.autocast("cuda", dtype=bf):
        conv(xi).float().sum().backward()
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
