"""One profiled MBS mini-batch (C2 by default) between cudaProfilerStart/Stop, for ncu.

ncu --profile-from-start off ... python tools/profile_step.py [--config c2] [--host]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_12484_b200 as mbs  # noqa: E402
from paper_2110_12484_b200.streamer import Staging  # noqa: E402
from paper_2110_12484_b200.workloads import WORKLOADS, build_model, synthetic_data  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--host", action="store_true")
ap.add_argument("--warmup", type=int, default=2)
ap.add_argument("--model-ops", default="native", choices=["native", "torch"])
args = ap.parse_args()
w = WORKLOADS[args.config]
dev = torch.device("cuda:0")
torch.backends.cudnn.benchmark = True
model = build_model(w, ops=args.model_ops).to(dev).to(memory_format=torch.channels_last)
params = mbs.ParameterSet(model, shadow=torch.bfloat16)
plan = mbs.plan_split(w.mini, w.micro)
x, y = synthetic_data(w, w.mini, device="cpu" if args.host else dev)
if args.host:
    x, y = x.pin_memory(), y.pin_memory()
acc = mbs.GradientAccumulator(params)
st = mbs.sgd_state(0.01, 0.9, 5e-4) if w.optimizer == "sgd" else mbs.adam_state(0.01, 5e-4)
streamer = mbs.make_streamer(x, y, w.micro) if args.host else None
kw = dict(accumulator=acc, staging=Staging(torch.bfloat16, True), autocast_dtype=torch.bfloat16,
          streamer=streamer, prefetch=True, keep_outputs=False)
for _ in range(args.warmup):
    mbs.train_mini_batch(model, params, (x, y), plan, w.normalization, w.loss_kind, st, **kw)[1].resolve()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
s = mbs.train_mini_batch(model, params, (x, y), plan, w.normalization, w.loss_kind, st, **kw)[1]
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("loss", s.loss, "grad_norm", s.grad_norm)
if streamer:
    streamer.close()
