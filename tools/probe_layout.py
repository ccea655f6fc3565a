"""Probe the model-side configuration (memory format) for the torch part of the step."""
import json
import torch
import torchvision
import sys
sys.path.insert(0, ".")
from paper_2110_12484_b200.workloads import UNet

torch.backends.cudnn.benchmark = True
dev = torch.device("cuda:0")
out = {}


def bench(name, model, x, y, lossf, iters=10):
    opt = torch.optim.SGD(model.parameters(), lr=0.01, momentum=0.9, fused=True)

    def step():
        with torch.autocast("cuda", torch.bfloat16):
            loss = lossf(model(x), y)
        loss.backward()
        opt.step()
        opt.zero_grad(set_to_none=True)
    for _ in range(4):
        step()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(iters):
        step()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / iters
    out[name] = {"ms": ms, "sps": x.shape[0] / ms * 1e3}
    print(name, out[name], flush=True)


ce = torch.nn.functional.cross_entropy
for fmt in ("cl", "nchw"):
    for bs in (128,):
        m = torchvision.models.resnet50(num_classes=102).to(dev)
        x = torch.randn(bs, 3, 224, 224, device=dev, dtype=torch.bfloat16)
        if fmt == "cl":
            m = m.to(memory_format=torch.channels_last)
            x = x.contiguous(memory_format=torch.channels_last)
        y = torch.randint(0, 102, (bs,), device=dev)
        bench(f"r50_{fmt}_bs{bs}", m, x, y, ce)
        del m
bce = torch.nn.functional.binary_cross_entropy_with_logits
for fmt in ("cl", "nchw"):
    m = UNet().to(dev)
    x = torch.randn(48, 3, 384, 384, device=dev, dtype=torch.bfloat16)
    if fmt == "cl":
        m = m.to(memory_format=torch.channels_last)
        x = x.contiguous(memory_format=torch.channels_last)
    y = (torch.rand(48, 1, 384, 384, device=dev) < 0.5).float()
    bench(f"unet_{fmt}_bs48", m, x, y, bce, iters=5)
    del m
print(json.dumps(out))
