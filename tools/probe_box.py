"""One-off box probe: host cores/RAM, pinned H2D bandwidth, ResNet-50 step time."""
import os, time, json, subprocess
import torch, torchvision
out = {}
out["cpu_count"] = os.cpu_count()
out["mem"] = open("/proc/meminfo").read().split("\n")[:3]
out["lscpu"] = subprocess.run(["lscpu"], capture_output=True, text=True).stdout.split("\n")[:20]
dev = torch.device("cuda:0")
out["free_total"] = torch.cuda.mem_get_info()
for nbytes in (19_267_584, 77_070_336, 1 << 30):
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    for _ in range(3): d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(10): d.copy_(h, non_blocking=True)
    e.record(); torch.cuda.synchronize()
    out[f"h2d_GBs_{nbytes}"] = nbytes * 10 / (s.elapsed_time(e) / 1e3) / 1e9
torch.backends.cudnn.benchmark = True
for fmt in ("cl",):
    m = torchvision.models.resnet50(num_classes=102).to(dev).to(memory_format=torch.channels_last)
    opt = torch.optim.SGD(m.parameters(), lr=0.01, momentum=0.9, weight_decay=5e-4)
    for bs in (128, 256):
        x = torch.randn(bs, 3, 224, 224, device=dev).to(memory_format=torch.channels_last)
        y = torch.randint(0, 102, (bs,), device=dev)
        def step():
            with torch.autocast("cuda", torch.bfloat16):
                loss = torch.nn.functional.cross_entropy(m(x), y)
            loss.backward()
            opt.step(); opt.zero_grad(set_to_none=True)
        for _ in range(5): step()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        for _ in range(10): step()
        e.record(); torch.cuda.synchronize()
        ms = s.elapsed_time(e) / 10
        out[f"r50_bf16_{fmt}_bs{bs}_ms"] = ms
        out[f"r50_bf16_{fmt}_bs{bs}_sps"] = bs / ms * 1e3
print(json.dumps(out, indent=1))
