"""Isolated MBS kernel microbenchmarks (L2 flushed between launches), C2 / C3 layouts.

The flush READS a 512 MB buffer (L2 ends up full of clean lines): a write-flush
would leave ~126 MB of dirty lines whose write-back lands inside the next timed
kernel (19 us of extra traffic at 6.5 TB/s). ``--flush write`` keeps that mode.

python tools/kbench.py [--config c2] -> JSON with algorithmic GB/s per kernel.
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_12484_b200 as mbs  # noqa: E402
from paper_2110_12484_b200.streamer import Staging, stage_rows  # noqa: E402
from paper_2110_12484_b200.workloads import WORKLOADS, build_model  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--flush", default="read", choices=["read", "write"])
args = ap.parse_args()
w = WORKLOADS[args.config]
dev = torch.device("cuda:0")
model = build_model(w).to(dev).to(memory_format=torch.channels_last)
params = mbs.ParameterSet(model)
P = params.layout.n_params
flush = torch.ones(128 * 2 ** 20, dtype=torch.float32, device=dev)
flush_sink = torch.empty((), dtype=torch.float32, device=dev)
peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6650.0


def timeit(fn, nbytes):
    ts = []
    for i in range(args.iters + 3):
        if args.flush == "write":
            flush.fill_(float(i))
        else:
            torch.sum(flush, dim=(0,), out=flush_sink)
        torch.cuda._sleep(2_000_000)      # GPU busy ~1 ms: host-side launch overhead is off the clock
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(s.elapsed_time(e))
    ts.sort()
    med = ts[len(ts) // 2]
    return {"us_median": med * 1e3, "us_min": ts[0] * 1e3, "gbs": nbytes / (med / 1e3) / 1e9,
            "frac": nbytes / (med / 1e3) / 1e9 / peak, "bytes": nbytes}


out = {"P": P, "segments": len(params.layout.names), "peak_gbs": peak, "flush": args.flush}
acc = mbs.GradientAccumulator(params)
grads = [torch.randn(s, device=dev).contiguous(memory_format=torch.channels_last) if len(s) == 4 else
         torch.randn(s, device=dev) for s in params.layout.shapes]
grads = [g.as_strided(s, st) if tuple(g.stride()) == st else g for g, s, st in
         zip(grads, params.layout.shapes, params.layout.strides)]


def k1_assign():
    acc.begin(1 << 15)
    acc.add_tensors(grads, 0.125)


def k1_accum():
    acc.add_tensors(grads, 0.125)


def k1_last():
    acc.add_tensors(grads, 0.125, last=True)


acc.begin(1 << 15)
acc.add_tensors(grads, 0.125)
out["k1_assign"] = timeit(k1_assign, 8 * P)
acc.begin(1 << 15)
acc.add_tensors(grads, 0.125)
out["k1_accumulate"] = timeit(k1_accum, 12 * P)
out["k1_accumulate_norm"] = timeit(k1_last, 12 * P)
# shadow-weight mode (the bench): bf16 gradients for the conv / linear weights, fp32 for BN and biases
gmix = [g.to(torch.bfloat16) if g.dim() >= 2 else g for g in grads]
nb_g = sum(g.numel() * g.element_size() for g in gmix)


def k1m_assign():
    acc.begin(1 << 15)
    acc.add_tensors(gmix, 0.125)


acc.begin(1 << 15)
acc.add_tensors(gmix, 0.125)
out["k1_assign_bf16g"] = timeit(k1m_assign, nb_g + 4 * P)
acc.begin(1 << 15)
acc.add_tensors(gmix, 0.125)
out["k1_accumulate_bf16g"] = timeit(lambda: acc.add_tensors(gmix, 0.125), nb_g + 8 * P)
acc.begin(1 << 15)
acc.add_tensors(grads, 0.125)
gs = acc.as_gradient_set()
st = mbs.sgd_state(0.01, 0.9, 5e-4)
out["k3_sgd"] = timeit(lambda: mbs.apply_update(params, gs, st), 20 * P)
sa = mbs.adam_state(0.01, 5e-4)
out["k3_adam"] = timeit(lambda: mbs.apply_update(params, gs, sa), 28 * P)
x = torch.randint(0, 256, (w.micro if w.micro else 16,) + w.sample_shape, dtype=torch.uint8, device=dev)
n = x.shape[0]
E = x[0].numel()
out["k2_stage_u8_bf16_nhwc"] = timeit(lambda: stage_rows(x, torch.uint8, tuple(x.shape[1:]), None, 0, n,
                                                         Staging(torch.bfloat16, True), dev), n * E * 3)
out["k2_stage_u8_f32_nhwc"] = timeit(lambda: stage_rows(x, torch.uint8, tuple(x.shape[1:]), None, 0, n,
                                                        Staging(torch.float32, True), dev), n * E * 5)
out["k2_stage_u8_f32_nchw"] = timeit(lambda: stage_rows(x, torch.uint8, tuple(x.shape[1:]), None, 0, n,
                                                        Staging(torch.float32, False), dev), n * E * 5)
xf = torch.randn((n,) + w.sample_shape, device=dev)
out["k2_stage_f32_bf16_nhwc"] = timeit(lambda: stage_rows(xf, torch.float32, tuple(xf.shape[1:]), None, 0, n,
                                                          Staging(torch.bfloat16, True), dev), n * E * 6)
# reference points: torch ops moving the same bytes
out["torch_copy_P_f32"] = timeit(lambda: acc.flat.copy_(params.flat), 8 * P)
out["torch_add_P_f32"] = timeit(lambda: acc.flat.add_(params.flat, alpha=0.125), 12 * P)
print(json.dumps(out, indent=1))
