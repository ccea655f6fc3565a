"""Diagnose GPU-vs-fp64 gradient differences on ResNet-18 (per parameter; MBS vs plain torch GPU)."""
import copy
import sys
import os
import numpy as np
import torch
import torchvision
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_12484_b200 as mbs
from oracle import mbs_oracle as O
from oracle.hybrid import TorchGradFn

torch.backends.cuda.matmul.allow_tf32 = False
torch.backends.cudnn.allow_tf32 = False
det = len(sys.argv) > 1 and sys.argv[1] == "det"
if det:
    torch.backends.cudnn.deterministic = True
    torch.backends.cudnn.benchmark = False
cuda = torch.device("cuda:0")
torch.manual_seed(0)
net = torchvision.models.resnet18(num_classes=10)
g = torch.Generator().manual_seed(1)
x = torch.randn(20, 3, 32, 32, generator=g)
y = torch.randint(0, 10, (20,), generator=g)
ref = TorchGradFn(net, "cross_entropy")
names = ref.names
plan = O.plan_split(20, 8)
g64, _ = O.mini_batch_gradient(ref, {n: v.shape for n, v in ref.params().items()}, x.double().numpy(), y.numpy(),
                               plan, "exact_weighted")
# plain torch on GPU: same micro split, loss*factor, autograd accumulation
pn = copy.deepcopy(net).to(cuda).train()
for k, (lo, hi) in enumerate(plan.index_ranges):
    f = O.normalization_factor(plan, k, "exact_weighted")
    loss = torch.nn.functional.cross_entropy(pn(x[lo:hi].to(cuda)), y[lo:hi].to(cuda))
    (loss * f).backward()
plain = {n: p.grad.double().cpu().numpy() for n, p in pn.named_parameters()}
dn = copy.deepcopy(net).to(cuda)
params = mbs.ParameterSet(dn)
total, st = mbs.mini_batch_gradient(dn, params, x.to(cuda), y.to(cuda), mbs.plan_split(20, 8), "exact_weighted",
                                    "cross_entropy")
ours = {n: total[n].double().cpu().numpy() for n in names}


def rl(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)


fa = lambda d: np.concatenate([d[n].ravel() for n in names])
print("det" if det else "default", "overall ours", rl(fa(ours), fa(g64)), "plain", rl(fa(plain), fa(g64)),
      "ours-vs-plain", rl(fa(ours), fa(plain)))
worst = sorted(names, key=lambda n: -rl(ours[n], g64[n]))[:8]
for n in worst:
    print(f"{n:40s} ours {rl(ours[n], g64[n]):.2e} plain {rl(plain[n], g64[n]):.2e} o-p {rl(ours[n], plain[n]):.2e}")
