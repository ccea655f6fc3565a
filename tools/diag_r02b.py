"""Round-2 diagnosis (GPU): ResNet-18@32 fp32, ONE micro-batch of 8, K5 variants vs fp64 per tensor."""
import copy
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

torch.backends.cuda.matmul.allow_tf32 = False
torch.backends.cudnn.allow_tf32 = False
cuda = torch.device("cuda:0")


def rel(a, b):
    a, b = np.asarray(a, np.float64).ravel(), np.asarray(b, np.float64).ravel()
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def grads(net, x, y, dev, dtype):
    net = net.to(dev, dtype).train()
    for p in net.parameters():
        p.grad = None
    out = net(x.to(dev, dtype).contiguous(memory_format=torch.channels_last) if dev.type == "cuda" else x.to(dtype))
    loss = torch.nn.functional.cross_entropy(out, y.to(dev))
    loss.backward()
    return {n: p.grad.double().cpu().numpy() for n, p in net.named_parameters()}, out.detach().double().cpu().numpy()


def main():
    import torchvision
    from paper_2110_12484_b200 import bn as K5
    torch.manual_seed(0)
    net = torchvision.models.resnet18(num_classes=10)
    for scale in ("u8", "n01"):
        g = torch.Generator().manual_seed(11)
        x = torch.randint(0, 256, (8, 3, 32, 32), generator=g).float() if scale == "u8" else \
            torch.randn(8, 3, 32, 32, generator=g)
        y = torch.randint(0, 10, (8,), generator=g)
        g64, o64 = grads(copy.deepcopy(net), x, y, torch.device("cpu"), torch.float64)
        names = list(g64)
        flat64 = np.concatenate([g64[n].ravel() for n in names])
        res = {}
        gt, ot = grads(copy.deepcopy(net).to(memory_format=torch.channels_last), x, y, cuda, torch.float32)
        res["torch"] = (gt, ot)
        for dual in ("1", "0"):
            os.environ["MBS_K5_DUAL"] = dual
            m = K5.fuse_batchnorm(copy.deepcopy(net)).to(memory_format=torch.channels_last)
            res[f"k5_dual{dual}"] = grads(m, x, y, cuda, torch.float32)
        for k, (gk, ok) in res.items():
            flat = np.concatenate([gk[n].ravel() for n in names])
            worst = sorted(names, key=lambda n: -rel(gk[n], g64[n]))[:4]
            print(scale, k, "grad %.3e out %.3e" % (rel(flat, flat64), rel(ok, o64)),
                  [(n, "%.2e" % rel(gk[n], g64[n])) for n in worst], flush=True)
        # per-layer forward activations: hook every BN output, torch vs k5
        acts = {}
        for k, mk in (("torch", copy.deepcopy(net)), ("k5", K5.fuse_batchnorm(copy.deepcopy(net))),
                      ("f64", copy.deepcopy(net))):
            dev, dt = (torch.device("cpu"), torch.float64) if k == "f64" else (cuda, torch.float32)
            mk = mk.to(dev, dt).train()
            rec = {}
            hs = [mod.register_forward_hook(lambda mod, i, o, nm=nm: rec.__setitem__(nm, (o[0] if isinstance(o, tuple) else o).detach().double().cpu().numpy()))
                  for nm, mod in mk.named_modules() if isinstance(mod, torch.nn.BatchNorm2d)]
            xx = x.to(dev, dt)
            if dev.type == "cuda":
                xx = xx.contiguous(memory_format=torch.channels_last)
            mk(xx)
            for h in hs:
                h.remove()
            acts[k] = rec
        for nm in list(acts["f64"])[:8] + list(acts["f64"])[-4:]:
            print(scale, "act", nm, "torch %.2e k5 %.2e" % (rel(acts["torch"][nm], acts["f64"][nm]),
                                                          rel(acts["k5"][nm], acts["f64"][nm])))


if __name__ == "__main__":
    main()
