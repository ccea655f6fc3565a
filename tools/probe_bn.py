"""Probe: how much of a ResNet-50 micro-batch step is BatchNorm, per dtype / layout (GPU box only).

Prints per-variant ms per fwd+bwd step at batch 128 and the BN kernels' share from torch.profiler.
"""
import sys
import time

import torch
import torchvision


def step_ms(model, x, y, dtype, iters=10):
    crit = torch.nn.CrossEntropyLoss()

    def one():
        with torch.autocast("cuda", dtype=dtype, enabled=dtype is not None):
            loss = crit(model(x), y)
        loss.backward()
    for _ in range(3):
        one()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        one()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters, one


def bn_share(one):
    from torch.profiler import profile, ProfilerActivity
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        one()
        torch.cuda.synchronize()
    tot = 0.0
    bn = 0.0
    names = {}
    for e in prof.key_averages():
        t = e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
        if e.device_type.name != "CUDA":
            continue
        tot += t
        if "batch_norm" in e.key.lower() or "bn_" in e.key.lower() or "batchnorm" in e.key.lower():
            bn += t
            names[e.key[:90]] = t
    return bn / max(tot, 1), tot / 1000, names


def main():
    dev = torch.device("cuda")
    torch.backends.cudnn.benchmark = True
    n = 128
    for layout in ("cl", "nchw"):
        for dtype in (torch.bfloat16, torch.float16):
            model = torchvision.models.resnet50(num_classes=102).to(dev)
            x = torch.randn(n, 3, 224, 224, device=dev)
            if layout == "cl":
                model = model.to(memory_format=torch.channels_last)
                x = x.to(memory_format=torch.channels_last)
            y = torch.randint(0, 102, (n,), device=dev)
            ms, one = step_ms(model, x, y, dtype)
            share, tot, names = bn_share(one)
            print(f"{layout} {dtype}: {ms:.2f} ms/step ({n / ms * 1000:.0f} samples/s) BN share {share:.3f} "
                  f"of {tot:.1f} ms kernel time", flush=True)
            for k, v in sorted(names.items(), key=lambda kv: -kv[1])[:4]:
                print(f"    {v / 1000:8.2f} ms  {k}")
    # isolated BN layer bandwidth: layer1-like 128x256x56x56 bf16 channels_last
    for shape in ((128, 256, 56, 56), (128, 64, 112, 112), (128, 1024, 14, 14)):
        x = torch.randn(shape, device=dev, dtype=torch.bfloat16).to(memory_format=torch.channels_last)
        x.requires_grad_(True)
        bn = torch.nn.BatchNorm2d(shape[1]).to(dev)
        g = torch.randn_like(x)
        for _ in range(3):
            bn(x).backward(g)
        torch.cuda.synchronize()
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        for _ in range(20):
            out = bn(x)
        e1.record()
        for _ in range(20):
            out = bn(x)
            out.backward(g)
        e2.record()
        torch.cuda.synchronize()
        f = e0.elapsed_time(e1) / 20
        fb = e1.elapsed_time(e2) / 20
        nb = x.numel() * 2
        print(f"BN {shape} bf16 CL: fwd {f * 1000:.1f} us ({3 * nb / f / 1e6:.0f} GB/s algorithmic, 3 passes), "
              f"fwd+bwd {fb * 1000:.1f} us ({8 * nb / fb / 1e6:.0f} GB/s, 8 passes)", flush=True)


if __name__ == "__main__":
    main()
