"""Probe (GPU box): first-layer conv cost with 3 input channels vs zero-padded to 4 / 8 (bf16, channels-last)."""
import torch
import torch.nn.functional as F


def bench(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def main():
    torch.backends.cudnn.benchmark = True
    dev = torch.device("cuda")
    for name, n, hw, cout, k, s, p in (("resnet50 conv1", 128, 224, 64, 7, 2, 3), ("unet inc conv", 48, 384, 64, 3, 1, 1)):
        for cin in (3, 4, 8):
            x = torch.randn(n, cin, hw, hw, device=dev, dtype=torch.bfloat16).contiguous(memory_format=torch.channels_last)
            w = torch.randn(cout, cin, k, k, device=dev, dtype=torch.bfloat16).contiguous(
                memory_format=torch.channels_last).requires_grad_(True)
            y = F.conv2d(x, w, None, s, p)
            g = torch.randn_like(y)

            def fwd():
                return F.conv2d(x, w, None, s, p)

            def fwdbwd():
                out = F.conv2d(x, w, None, s, p)
                out.backward(g)
            tf = bench(fwd)
            tb = bench(fwdbwd)
            print(f"{name} C_in={cin}: fwd {tf * 1e3:.0f} us, fwd+wgrad {tb * 1e3:.0f} us", flush=True)


if __name__ == "__main__":
    main()
