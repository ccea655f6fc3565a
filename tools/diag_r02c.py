"""Round-2 diagnosis (GPU): ResNet-18@32 fp32 with K5 — per-micro errors, fresh module vs reused module."""
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


def micro_grads(net, xk, yk, dev, dtype):
    for p in net.parameters():
        p.grad = None
    xx = xk.to(dev, dtype)
    if dev.type == "cuda":
        xx = xx.contiguous(memory_format=torch.channels_last)
    loss = torch.nn.functional.cross_entropy(net(xx), yk.to(dev))
    loss.backward()
    return np.concatenate([p.grad.double().cpu().numpy().ravel() for p in net.parameters()])


def main():
    import torchvision
    from paper_2110_12484_b200 import bn as K5
    torch.manual_seed(0)
    net = torchvision.models.resnet18(num_classes=10).train()
    g = torch.Generator().manual_seed(11)
    x = torch.randint(0, 256, (64, 3, 32, 32), dtype=torch.uint8, generator=g).float()
    y = torch.randint(0, 10, (64,), generator=g)
    n64 = copy.deepcopy(net).double()
    k5_reuse = K5.fuse_batchnorm(copy.deepcopy(net)).to(cuda).to(memory_format=torch.channels_last).train()
    t_reuse = copy.deepcopy(net).to(cuda).to(memory_format=torch.channels_last).train()
    for k in range(8):
        xk, yk = x[8 * k:8 * k + 8], y[8 * k:8 * k + 8]
        r64 = micro_grads(n64, xk, yk, torch.device("cpu"), torch.float64)
        fresh = micro_grads(K5.fuse_batchnorm(copy.deepcopy(net)).to(cuda).to(memory_format=torch.channels_last).train(),
                            xk, yk, cuda, torch.float32)
        reuse = micro_grads(k5_reuse, xk, yk, cuda, torch.float32)
        tre = micro_grads(t_reuse, xk, yk, cuda, torch.float32)
        print(k, "k5 fresh %.3e  k5 reused %.3e  torch reused %.3e" % (rel(fresh, r64), rel(reuse, r64),
                                                                       rel(tre, r64)), flush=True)
    # running stats after 8 micro-batches: K5 vs torch vs fp64
    for (n1, b1), (n2, b2), (n3, b3) in zip(k5_reuse.named_buffers(), t_reuse.named_buffers(), n64.named_buffers()):
        if "running_var" in n1 or "running_mean" in n1:
            print(n1, "k5 %.2e torch %.2e" % (rel(b1.double().cpu().numpy(), b3.numpy()),
                                              rel(b2.double().cpu().numpy(), b3.numpy())))
            break




def layers():
    """Micro 5: every block's output and input-gradient, K5 (MBS_K5_DUAL=0: blocks called as modules) vs fp64."""
    import torchvision
    os.environ["MBS_K5_DUAL"] = "0"
    from paper_2110_12484_b200 import bn as K5
    torch.manual_seed(0)
    net = torchvision.models.resnet18(num_classes=10).train()
    g = torch.Generator().manual_seed(11)
    x = torch.randint(0, 256, (64, 3, 32, 32), dtype=torch.uint8, generator=g).float()
    y = torch.randint(0, 10, (64,), generator=g)
    xk, yk = x[40:48], y[40:48]
    rec = {}
    for tag, m, dev, dt in (("f64", copy.deepcopy(net).double(), torch.device("cpu"), torch.float64),
                            ("k5", K5.fuse_batchnorm(copy.deepcopy(net)).to(cuda).to(memory_format=torch.channels_last),
                             cuda, torch.float32),
                            ("torch", copy.deepcopy(net).to(cuda).to(memory_format=torch.channels_last), cuda,
                             torch.float32)):
        r = rec[tag] = {}
        hs = []
        for nm, mod in m.named_modules():
            if (nm.count(".") == 1 and nm.startswith("layer")) or nm in ("avgpool", "fc"):
                def fh(mod, i, o, nm=nm):
                    r["out:" + nm] = o.detach().double().cpu().numpy()
                    if o.requires_grad:
                        o.register_hook(lambda g, nm=nm: r.__setitem__("gout:" + nm, g.detach().double().cpu().numpy()))
                hs.append(mod.register_forward_hook(fh))
        for p in m.parameters():
            p.grad = None
        xx = xk.to(dev, dt)
        if dev.type == "cuda":
            xx = xx.contiguous(memory_format=torch.channels_last)
        loss = torch.nn.functional.cross_entropy(m(xx), yk.to(dev))
        loss.backward()
        for h in hs:
            h.remove()
    for k in rec["f64"]:
        if k in rec["k5"]:
            print(k, "k5 %.2e torch %.2e" % (rel(rec["k5"][k], rec["f64"][k]), rel(rec["torch"].get(k, 0), rec["f64"][k])))
    # the layer4 BN inputs of micro 5: per-channel spread
    print("done")



def bn_case():
    """Micro 5, layer4.1.bn1 / bn2: K5 fwd+bwd on the captured fp32 inputs vs the same math in fp64."""
    import torchvision
    os.environ["MBS_K5_DUAL"] = "0"
    from paper_2110_12484_b200 import bn as K5
    torch.manual_seed(0)
    net = torchvision.models.resnet18(num_classes=10).train()
    g = torch.Generator().manual_seed(11)
    x = torch.randint(0, 256, (64, 3, 32, 32), dtype=torch.uint8, generator=g).float()
    y = torch.randint(0, 10, (64,), generator=g)
    xk, yk = x[40:48], y[40:48]
    m = K5.fuse_batchnorm(copy.deepcopy(net)).to(cuda).to(memory_format=torch.channels_last).train()
    cap = {}
    for nm in ("layer4.1.bn1", "layer4.1.bn2", "layer4.0.bn2", "layer4.0.bn1"):
        mod = m.get_submodule(nm)

        def pre(mod, args, nm=nm):
            cap[nm] = {"x": args[0].detach().clone(), "r": args[1].detach().clone() if len(args) > 1 and args[1] is not None else None}

        def post(mod, args, out, nm=nm):
            out.register_hook(lambda gr, nm=nm: cap[nm].__setitem__("dy", gr.detach().clone()))
        mod.register_forward_pre_hook(pre)
        mod.register_forward_hook(post)
    loss = torch.nn.functional.cross_entropy(m(xk.to(cuda).contiguous(memory_format=torch.channels_last)), yk.to(cuda))
    loss.backward()
    for nm, c in cap.items():
        mod = m.get_submodule(nm)
        xx = c["x"].clone().requires_grad_(True)
        rr = c["r"].clone().requires_grad_(True) if c["r"] is not None else None
        w = mod.weight.detach().clone().requires_grad_(True)
        b = mod.bias.detach().clone().requires_grad_(True)
        out = K5._MicroBatchNormFn.apply(xx, rr, w, b, None, None, 0.0, mod.eps, mod.fuse_relu, False, None)
        out.backward(c["dy"])
        # fp64 reference of the same op
        x64 = c["x"].double().requires_grad_(True)
        r64 = c["r"].double().requires_grad_(True) if c["r"] is not None else None
        w64 = mod.weight.detach().double().requires_grad_(True)
        b64 = mod.bias.detach().double().requires_grad_(True)
        mean = x64.mean((0, 2, 3), keepdim=True)
        var = x64.var((0, 2, 3), keepdim=True, unbiased=False)
        z = (x64 - mean) / torch.sqrt(var + mod.eps) * w64.view(1, -1, 1, 1) + b64.view(1, -1, 1, 1)
        if r64 is not None:
            z = z + r64
        o64 = torch.relu(z) if mod.fuse_relu else z
        o64.backward(c["dy"].double())
        print(nm, "rows", c["x"].shape, "out %.2e dx %.2e dw %.2e db %.2e" % (
            rel(out.detach().double().cpu(), o64.detach().cpu()), rel(xx.grad.double().cpu(), x64.grad.cpu()),
            rel(w.grad.double().cpu(), w64.grad.cpu()), rel(b.grad.double().cpu(), b64.grad.cpu())))
        if rr is not None:
            print("   dres %.2e" % rel(rr.grad.double().cpu(), r64.grad.cpu()))
            de = (rr.grad.double() - r64.grad).abs()
            idx = torch.nonzero(de > 1e-3 * float(r64.grad.abs().max()))
            print("   dres bad elements", idx[:10].tolist(), "ours", [float(rr.grad[tuple(i)]) for i in idx[:5]],
                  "ref", [float(r64.grad[tuple(i)]) for i in idx[:5]], "z64", [float(z[tuple(i)]) for i in idx[:5]],
                  "r", [float(c["r"][tuple(i)]) for i in idx[:5]], "out", [float(out[tuple(i)]) for i in idx[:5]])
        dxe = (xx.grad.double() - x64.grad).abs().amax((0, 2, 3))
        ch = int(dxe.argmax())
        print("   worst channel", ch, "dx err", float(dxe[ch]), "x", c["x"][:, ch].flatten().tolist()[:8],
              "z64", z[:, ch].flatten().tolist()[:8], "dy", c["dy"][:, ch].flatten().tolist()[:8],
              "var", float(var.flatten()[ch]))



def block_case():
    """Micro 5: block layer4.1 alone on the captured input / output-gradient: K5 block vs torch fp32 vs fp64."""
    import torchvision
    os.environ["MBS_K5_DUAL"] = "0"
    from paper_2110_12484_b200 import bn as K5
    torch.manual_seed(0)
    net = torchvision.models.resnet18(num_classes=10).train()
    g = torch.Generator().manual_seed(11)
    x = torch.randint(0, 256, (64, 3, 32, 32), dtype=torch.uint8, generator=g).float()
    y = torch.randint(0, 10, (64,), generator=g)
    xk, yk = x[40:48], y[40:48]
    m = K5.fuse_batchnorm(copy.deepcopy(net)).to(cuda).to(memory_format=torch.channels_last).train()
    cap = {}
    blk = m.layer4[1]
    blk.register_forward_pre_hook(lambda mod, a: cap.__setitem__("x", a[0].detach().clone()))
    def fh(mod, a, o):
        o.register_hook(lambda gr: cap.__setitem__("dy", gr.detach().clone()))
    blk.register_forward_hook(fh)
    loss = torch.nn.functional.cross_entropy(m(xk.to(cuda).contiguous(memory_format=torch.channels_last)), yk.to(cuda))
    loss.backward()
    print("captured x", cap["x"].shape, cap["x"].stride(), "dy", cap["dy"].stride())
    res = {}
    for tag, b, dt, dev in (("k5", copy.deepcopy(blk), torch.float32, cuda),
                            ("torch", copy.deepcopy(net.layer4[1]).to(cuda).to(memory_format=torch.channels_last),
                             torch.float32, cuda),
                            ("f64", copy.deepcopy(net.layer4[1]).double(), torch.float64, torch.device("cpu"))):
        b.train()
        xi = cap["x"].to(dev, dt).clone().requires_grad_(True)
        o = b(xi)
        o.backward(cap["dy"].to(dev, dt))
        res[tag] = (o.detach().double().cpu(), xi.grad.double().cpu(),
                    {n: p.grad.double().cpu() for n, p in b.named_parameters()})
    for tag in ("k5", "torch"):
        o, gx, gp = res[tag]
        print(tag, "out %.2e dx %.2e" % (rel(o, res["f64"][0]), rel(gx, res["f64"][1])),
              {n: "%.1e" % rel(gp[n], res["f64"][2][n]) for n in gp})
    # K5 block with the sub-steps exposed
    b = copy.deepcopy(blk)
    xi = cap["x"].clone().requires_grad_(True)
    h1 = b.conv1(xi)
    h1.retain_grad()
    a1 = b.bn1(h1)
    a1.retain_grad()
    h2 = b.conv2(a1)
    h2.retain_grad()
    o = b.bn2(h2, xi)
    o.backward(cap["dy"])
    b64 = copy.deepcopy(net.layer4[1]).double().train()
    x64 = cap["x"].double().cpu().requires_grad_(True)
    g1 = b64.conv1(x64)
    g1.retain_grad()
    c1 = b64.relu(b64.bn1(g1))
    c1.retain_grad()
    g2 = b64.conv2(c1)
    g2.retain_grad()
    o64 = b64.relu(b64.bn2(g2) + x64)
    o64.backward(cap["dy"].double().cpu())
    for nm, t, t64 in (("h1", h1, g1), ("a1", a1, c1), ("h2", h2, g2)):
        print(nm, "val %.2e grad %.2e" % (rel(t.detach().double().cpu(), t64.detach()),
                                          rel(t.grad.double().cpu(), t64.grad)), "strides", t.stride(),
              t.grad.stride())


if __name__ == "__main__":
    {"layers": layers, "bn": bn_case, "block": block_case}.get(sys.argv[1] if len(sys.argv) > 1 else "", main)()
