"""In-pipeline kernel shares of the MBS step (C2 by default) from CUPTI device timestamps (torch.profiler),
as the timed run executes it: micro steps replayed from CUDA graphs, PDL overlaps, warm L2. Complements the
ncu launch list (serialized, cold cache).

python tools/prof_pipeline.py [--config c2] [--minis 2]  -> table on stdout, JSON to gpurun_out/prof_pipeline.json
"""
import argparse
import collections
import json
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_12484_b200 as mbs  # noqa: E402
from paper_2110_12484_b200.streamer import Staging  # noqa: E402
from paper_2110_12484_b200.workloads import WORKLOADS, build_model, synthetic_data  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--minis", type=int, default=2)
ap.add_argument("--out", default="gpurun_out/prof_pipeline.json")
args = ap.parse_args()
w = WORKLOADS[args.config]
dev = torch.device("cuda:0")
torch.backends.cudnn.benchmark = True
model = build_model(w, ops="native").to(dev).to(memory_format=torch.channels_last)
params = mbs.ParameterSet(model, shadow=torch.bfloat16)
plan = mbs.plan_split(w.mini, w.micro)
x, y = synthetic_data(w, w.mini, device=dev)
acc = mbs.GradientAccumulator(params)
st = mbs.sgd_state(0.01, 0.9, 5e-4) if w.optimizer == "sgd" else mbs.adam_state(0.01, 5e-4)
kw = dict(accumulator=acc, staging=Staging(torch.bfloat16, True), autocast_dtype=torch.bfloat16, prefetch=True,
          keep_outputs=False)
for _ in range(3):
    mbs.train_mini_batch(model, params, (x, y), plan, w.normalization, w.loss_kind, st, **kw)[1].resolve()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    e0.record()
    for _ in range(args.minis):
        mbs.train_mini_batch(model, params, (x, y), plan, w.normalization, w.loss_kind, st, **kw)[1].resolve()
    e1.record()
    torch.cuda.synchronize()
wall_us = e0.elapsed_time(e1) * 1e3
kern = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
spans = sorted((e.time_range.start, e.time_range.end) for e in kern)
busy, cur_s, cur_e = 0.0, None, None
for s, e in spans:                                   # union of kernel intervals = device busy time
    if cur_e is None or s > cur_e:
        if cur_e is not None:
            busy += cur_e - cur_s
        cur_s, cur_e = s, e
    else:
        cur_e = max(cur_e, e)
if cur_e is not None:
    busy += cur_e - cur_s
agg = collections.defaultdict(lambda: [0, 0.0])
for e in kern:
    n = e.name.split("(")[0]
    agg[n][0] += 1
    agg[n][1] += e.time_range.end - e.time_range.start
tot = sum(v[1] for v in agg.values())


def family(n):
    if "k_bn" in n:
        return "K5 BatchNorm"
    if "k_maxpool" in n or "k_copy_channels" in n:
        return "K6 pool / skip join"
    if "k_im2col" in n:
        return "K7 stem im2col"
    if "k_accum" in n or "k_finalize" in n or "k_sumsq" in n:
        return "K1/K4 accumulate"
    if "k_stage" in n or "k_gather" in n:
        return "K2 staging"
    if "k_sgd" in n or "k_adam" in n:
        return "K3 optimizer"
    if "cutlass" in n or "nvjet" in n or "cudnn" in n or "gemm" in n.lower() or "conv" in n.lower():
        return "convolutions / GEMMs (cuDNN, cuBLAS)"
    return "other (torch elementwise, casts, loss)"


fam = collections.defaultdict(float)
for n, (c, t) in agg.items():
    fam[family(n)] += t
out = {"config": w.name, "mini_batches": args.minis, "wall_us": wall_us, "kernel_sum_us": tot, "busy_us": busy,
       "idle_frac": 1.0 - busy / wall_us if wall_us else None, "overlap_us": tot - busy,
       "families": {k: {"us": v, "share_of_kernel_time": v / tot} for k, v in sorted(fam.items(), key=lambda kv: -kv[1])},
       "top": [{"kernel": n[:100], "launches": c, "us": t, "share": t / tot}
               for n, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:30]]}
os.makedirs(os.path.dirname(args.out), exist_ok=True)
with open(args.out, "w") as f:
    json.dump(out, f, indent=1)
print(f"wall {wall_us / 1e3:.2f} ms, kernel sum {tot / 1e3:.2f} ms, device busy {busy / 1e3:.2f} ms "
      f"(idle {100 * out['idle_frac']:.1f} %, overlapped {(tot - busy) / 1e3:.2f} ms)")
for k, v in out["families"].items():
    print(f"{100 * v['share_of_kernel_time']:6.2f} %  {v['us'] / 1e3:8.2f} ms  {k}")
for t in out["top"][:15]:
    print(f"{100 * t['share']:6.2f} %  {t['launches']:5d}  {t['kernel']}")
