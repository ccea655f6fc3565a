"""Probe (GPU box): host issue cost of one micro-batch fwd+bwd of the native-ops models (batch 2, where
the GPU is idle-bound) vs the GPU time at the benchmark micro-batch — is the micro loop CPU-bound?"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2110_12484_b200.workloads import WORKLOADS, build_model  # noqa: E402
from paper_2110_12484_b200.losses import compute_loss  # noqa: E402


def run(cfg, batch, ops, iters=20):
    w = WORKLOADS[cfg]
    dev = torch.device("cuda")
    m = build_model(w, ops=ops).to(dev).to(memory_format=torch.channels_last).train()
    x = torch.randn((batch,) + w.sample_shape, device=dev).to(torch.bfloat16).contiguous(memory_format=torch.channels_last)
    y = (torch.randint(0, w.n_classes, (batch,), device=dev) if w.target == "classes"
         else (torch.rand((batch, 1) + w.sample_shape[1:], device=dev) < 0.5).float())

    def one():
        with torch.autocast("cuda", dtype=torch.bfloat16):
            loss = compute_loss(w.loss_kind, m(x), y)
        loss.backward()
    for _ in range(3):
        one()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(iters):
        one()
    e1.record()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{cfg} {ops} batch {batch}: host issue {1e3 * (t1 - t0) / iters:.2f} ms/step, "
          f"GPU {e0.elapsed_time(e1) / iters:.2f} ms/step, wall {1e3 * (t2 - t0) / iters:.2f} ms/step", flush=True)


if __name__ == "__main__":
    for cfg, big in (("c2", 128), ("c3", 48)):
        for ops in ("native", "torch"):
            run(cfg, 2, ops)
            run(cfg, big, ops)
