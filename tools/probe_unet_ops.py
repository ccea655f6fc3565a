"""Which torch ops launch the U-Net step's remaining copy / elementwise kernels (profiler with shapes)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2110_12484_b200.workloads import WORKLOADS, build_model  # noqa: E402
from paper_2110_12484_b200.losses import compute_loss  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
w = WORKLOADS[cfg]
dev = torch.device("cuda")
torch.backends.cudnn.benchmark = True
m = build_model(w, ops="native").to(dev).to(memory_format=torch.channels_last).train()
n = w.micro or 16
x = torch.randn((n,) + w.sample_shape, device=dev).to(torch.bfloat16).contiguous(memory_format=torch.channels_last)
y = (torch.randint(0, w.n_classes, (n,), device=dev) if w.target == "classes"
     else (torch.rand((n, 1) + w.sample_shape[1:], device=dev) < 0.5).float())


def one():
    with torch.autocast("cuda", dtype=torch.bfloat16):
        loss = compute_loss(w.loss_kind, m(x), y)
    loss.backward()


for _ in range(3):
    one()
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity  # noqa: E402
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA], record_shapes=True) as prof:
    one()
    torch.cuda.synchronize()
for e in prof.events():
    if (e.name.startswith("aten::") and "conv" not in e.name and e.device_time_total > 150
            and e.cpu_parent is not None and not e.cpu_parent.name.startswith("aten::")):
        print(f"{e.name:20s} {e.device_time_total / 1000:8.3f} ms  {str(e.input_shapes)[:150]}  "
              f"{[str(t)[:12] for t in getattr(e, 'concrete_inputs', [])][:3]}")
        parent = e.cpu_parent
        chain = []
        while parent is not None and len(chain) < 6:
            chain.append(parent.name)
            parent = parent.cpu_parent
        print("      <- " + " <- ".join(chain))
