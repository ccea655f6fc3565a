"""Why does the MBS U-Net run hold a lower SM clock than the no-stream run under the power cap?
Runs, each for --seconds on HBM-resident data with nvidia-smi sampling clock / power / temperature:
  nos      - the no-stream baseline (bench.no_stream_baseline, native ops, graph, fused Adam per batch)
  mbs_1    - the MBS engine with mini = micro (one micro-batch per optimizer step: same schedule as nos)
  mbs_64   - the MBS engine with 64 micro-batches per mini-batch (the N1 shape)
  mbs_1_lr0 - mbs_1 with learning rate 1e-9 (an optimizer step per micro-batch that leaves the weights at init)
python tools/probe_power.py --config n1 --seconds 45
"""
import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2110_12484_b200 as mbs  # noqa: E402
from paper_2110_12484_b200.streamer import Staging  # noqa: E402
from paper_2110_12484_b200.workloads import WORKLOADS, build_model, synthetic_data  # noqa: E402


class Sampler:
    def __enter__(self):
        self.p = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw,temperature.gpu,clocks.mem",
                                   "--format=csv,noheader,nounits", "-lms", "200"], stdout=subprocess.PIPE, text=True)
        return self

    def __exit__(self, *a):
        self.p.terminate()
        out = self.p.communicate()[0]
        v = np.array([[float(t) for t in ln.split(",")] for ln in out.strip().splitlines() if ln.count(",") == 3])
        self.s = {"sm_mhz": float(np.median(v[:, 0])), "power_w": float(np.median(v[:, 1])),
                  "temp_c": float(np.median(v[:, 2])), "mem_mhz": float(np.median(v[:, 3])), "n": len(v)}


ap = argparse.ArgumentParser()
ap.add_argument("--config", default="n1")
ap.add_argument("--seconds", type=float, default=45.0)
ap.add_argument("--kinds", default="nos,mbs_1,mbs_64")
ap.add_argument("--reps", type=int, default=2)
args = ap.parse_args()
w = WORKLOADS[args.config]
dev = torch.device("cuda:0")
torch.backends.cudnn.benchmark = True
b = w.micro
x, y = synthetic_data(w, 64 * b, seed=0, device="cpu")
x, y = x.to(dev), y.to(dev)


def run_mbs(mini, lr=0.01):
    model = build_model(w, ops="native").to(dev).to(memory_format=torch.channels_last)
    params = mbs.ParameterSet(model, shadow=torch.bfloat16)
    acc = mbs.GradientAccumulator(params)
    st = mbs.sgd_state(lr, 0.9, 5e-4) if w.optimizer == "sgd" else mbs.adam_state(lr, 5e-4)
    staging = Staging(dtype=torch.bfloat16, channels_last=True, target_dtype=torch.float32)

    def epoch(e):
        return mbs.train_epoch(model, params, x, y, mini_batch_size=mini, micro_batch_size=b,
                               normalization=w.normalization, loss_kind=w.loss_kind, optimizer_state=st, seed=0,
                               epoch_index=e, shuffle=True, prefetch=True, accumulator=acc, staging=staging,
                               autocast_dtype=torch.bfloat16)
    epoch(0)
    torch.cuda.synchronize()
    n, t0 = 0, time.perf_counter()
    with Sampler() as s:
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        while time.perf_counter() - t0 < args.seconds:
            epoch(1 + n)
            n += 1
        e1.record()
        torch.cuda.synchronize()
    return {"value": n * x.shape[0] / (e0.elapsed_time(e1) / 1e3), **s.s}


for rep in range(args.reps):
    for kind in args.kinds.split(","):
        if kind == "nos":
            with Sampler() as s:
                r = bench.no_stream_baseline(w, dev, b, 3, 3, 1, ops="native", min_s=args.seconds, data=(x, y))
            r = {"value": r["value"], **s.s}
        else:
            r = run_mbs(b if kind.startswith("mbs_1") else 64 * b, lr=1e-9 if kind.endswith("lr0") else 0.01)
        torch.cuda.empty_cache()
        r["per_mhz"] = r["value"] / r["sm_mhz"]
        r["samples_per_joule"] = r["value"] / r["power_w"]
        print(json.dumps({"kind": kind, **{k: round(v, 4) for k, v in r.items()}}), flush=True)
