"""Probe (exploration, not product): does cuDNN's runtime fusion build on sm_100 for the ResNet conv-BN patterns?

(1) ConvBNfprop: relu(x * scale + bias) -> conv_fprop -> genstats (sum, sum of squares per output channel)
(2) ConvBNwgrad: relu(x * scale + bias) -> conv_wgrad(dy)
Times each against torch's conv (cuDNN) + the separate passes it would replace.
"""
import time

import cudnn
import torch

dev = torch.device("cuda:0")
torch.backends.cudnn.benchmark = True
handle = cudnn.create_handle()
print("cudnn backend", cudnn.backend_version())


def timeit(fn, it=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(it):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it * 1e3


for (n, c, h, k, r) in [(128, 64, 56, 64, 3), (128, 128, 28, 128, 3), (128, 256, 56, 64, 1), (128, 512, 28, 128, 1)]:
    x = torch.randn(n, c, h, h, device=dev, dtype=torch.bfloat16).to(memory_format=torch.channels_last)
    wt = (torch.randn(k, c, r, r, device=dev, dtype=torch.bfloat16) * 0.05).to(memory_format=torch.channels_last)
    sc = torch.rand(1, c, 1, 1, device=dev, dtype=torch.float32) + 0.5
    bi = torch.randn(1, c, 1, 1, device=dev, dtype=torch.float32) * 0.1
    pad = r // 2
    y = torch.empty(n, k, h, h, device=dev, dtype=torch.bfloat16).to(memory_format=torch.channels_last)
    s1 = torch.empty(1, k, 1, 1, device=dev, dtype=torch.float32)
    s2 = torch.empty(1, k, 1, 1, device=dev, dtype=torch.float32)
    try:
        g = cudnn.pygraph(io_data_type=cudnn.data_type.BFLOAT16, intermediate_data_type=cudnn.data_type.FLOAT,
                          compute_data_type=cudnn.data_type.FLOAT, handle=handle)
        X = g.tensor_like(x)
        W = g.tensor_like(wt)
        SC = g.tensor_like(sc)
        BI = g.tensor_like(bi)
        t = g.scale(input=X, scale=SC)
        t = g.bias(input=t, bias=BI)
        t = g.relu(input=t)
        t.set_data_type(cudnn.data_type.BFLOAT16)
        Y = g.conv_fprop(image=t, weight=W, padding=[pad, pad], stride=[1, 1], dilation=[1, 1])
        Y.set_output(True).set_data_type(cudnn.data_type.BFLOAT16)
        S1, S2 = g.genstats(input=Y)
        S1.set_output(True).set_data_type(cudnn.data_type.FLOAT)
        S2.set_output(True).set_data_type(cudnn.data_type.FLOAT)
        g.validate()
        g.build_operation_graph()
        g.create_execution_plans([cudnn.heur_mode.A, cudnn.heur_mode.FALLBACK])
        g.check_support()
        g.build_plans()
        ws = torch.empty(g.get_workspace_size(), device=dev, dtype=torch.uint8)
        pack = {X: x, W: wt, SC: sc, BI: bi, Y: y, S1: s1, S2: s2}
        us_f = timeit(lambda: g.execute(pack, ws, handle=handle))
        ref = torch.nn.functional.conv2d(torch.relu(x.float() * sc + bi).to(torch.bfloat16), wt, padding=pad)
        err = (ref.float() - y.float()).norm() / ref.float().norm()
        serr = (ref.float().sum(dim=(0, 2, 3)) - s1.flatten()).norm() / ref.float().sum(dim=(0, 2, 3)).norm()
        ok = f"fused {us_f:.1f} us  rel err y {err:.2e}  sum {serr:.2e}"
    except Exception as e:  # noqa: BLE001
        ok = f"fused FAILED: {type(e).__name__}: {str(e)[:300]}"
    xr = torch.relu(x.float() * sc + bi).to(torch.bfloat16)
    us_c = timeit(lambda: torch.nn.functional.conv2d(xr, wt, padding=pad))
    us_a = timeit(lambda: torch.relu(x * sc.to(torch.bfloat16) + bi.to(torch.bfloat16)))
    print(f"n{n} c{c} h{h} k{k} r{r}: torch conv {us_c:.1f} us, torch apply {us_a:.1f} us | {ok}")
