"""K5 performance probe (GPU box): model micro-batch step time with torch BN vs fused K5, and
isolated K5 layer bandwidth (algorithmic bytes / CUDA-event time, L2 flushed before each rep)."""
import sys
import os

import torch
import torchvision

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2110_12484_b200 import bn as K5  # noqa: E402
from paper_2110_12484_b200 import pool as K6  # noqa: E402
from paper_2110_12484_b200 import stem as K7  # noqa: E402
from paper_2110_12484_b200.workloads import UNet  # noqa: E402


def step_ms(model, x, y, loss_fn, iters=10):
    def one():
        with torch.autocast("cuda", dtype=torch.bfloat16):
            loss = loss_fn(model(x), y)
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


def top_kernels(one, k=12):
    from torch.profiler import profile, ProfilerActivity
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        one()
        torch.cuda.synchronize()
    rows = []
    tot = 0.0
    for e in prof.key_averages():
        if e.device_type.name != "CUDA":
            continue
        t = e.device_time_total
        tot += t
        rows.append((t, e.count, e.key[:100]))
    rows.sort(reverse=True)
    print(f"    kernel time {tot / 1000:.2f} ms")
    for t, c, n in rows[:k]:
        print(f"    {t / 1000:7.2f} ms {100 * t / tot:5.1f}% x{c:<4d} {n}")


def models():
    dev = torch.device("cuda")
    ce = torch.nn.CrossEntropyLoss()
    bce = torch.nn.BCEWithLogitsLoss()
    for name, make, shape, tgt, lf in (
            ("resnet50 b128@224", lambda: torchvision.models.resnet50(num_classes=102), (128, 3, 224, 224),
             lambda n: torch.randint(0, 102, (n,), device=dev), ce),
            ("unet b48@384", lambda: UNet(3, 1), (48, 3, 384, 384),
             lambda n: (torch.rand(n, 1, 384, 384, device=dev) < 0.5).float(), bce)):
        for fused in (False, True):
            torch.manual_seed(0)
            m = make().to(dev).to(memory_format=torch.channels_last).train()
            if fused:
                K5.fuse_batchnorm(m)
                K6.swap_maxpool(m)
                K7.swap_stem(m)
                K7.swap_pointwise(m)
                if hasattr(m, "native_skips"):
                    m.native_skips = True
            x = torch.randn(shape, device=dev).to(memory_format=torch.channels_last)
            y = tgt(shape[0])
            ms, one = step_ms(m, x, y, lf)
            print(f"{name} {'native ops' if fused else 'torch ops'}: {ms:.2f} ms/step "
                  f"({shape[0] / ms * 1000:.0f} samples/s)", flush=True)
            top_kernels(one)
            del m, x, y
            torch.cuda.empty_cache()


def layers():
    dev = torch.device("cuda")
    flush = torch.empty(512 * 2 ** 20, dtype=torch.uint8, device=dev)
    for shape in ((128, 64, 112, 112), (128, 256, 56, 56), (128, 64, 56, 56), (128, 512, 28, 28),
                  (128, 1024, 14, 14), (128, 2048, 7, 7), (48, 64, 384, 384)):
        C = shape[1]
        x = torch.randn(shape, device=dev, dtype=torch.bfloat16).contiguous(memory_format=torch.channels_last)
        r = torch.randn_like(x)
        dy = torch.randn_like(x)
        w = torch.ones(C, device=dev, requires_grad=True)
        b = torch.zeros(C, device=dev, requires_grad=True)
        nb = x.numel() * 2
        for relu, res in ((False, None), (True, None), (True, r)):
            xx = x.detach().requires_grad_(True)
            rr = None if res is None else res.detach().requires_grad_(True)
            fw, bw = [], []
            for rep in range(12):
                flush.zero_()
                e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
                e[0].record()
                y = K5.micro_batch_norm(xx, w, b, relu=relu, residual=rr)
                e[1].record()
                flush.zero_()
                e2 = torch.cuda.Event(enable_timing=True)
                e2.record()
                y.backward(dy)
                e[2].record()
                torch.cuda.synchronize()
                if rep >= 2:
                    fw.append(e[0].elapsed_time(e[1]))
                    bw.append(e2.elapsed_time(e[2]))
            fw.sort()
            bw.sort()
            f, bk = fw[len(fw) // 2], bw[len(bw) // 2]
            fbytes = nb * (3 + (res is not None))
            bbytes = nb * (5 + 3 * (res is not None))
            tag = "plain" if not relu else ("relu" if res is None else "relu+res")
            print(f"K5 {shape} {tag:8s}: fwd {f * 1000:7.1f} us {fbytes / f / 1e6:6.0f} GB/s | "
                  f"bwd {bk * 1000:7.1f} us {bbytes / bk / 1e6:6.0f} GB/s", flush=True)


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    if what in ("all", "layers"):
        layers()
    if what in ("all", "models"):
        models()
