"""Does the no-stream baseline's data change its clock under the power cap? A/B: two synthetic batches
cycled (the old baseline) vs a pool of 64 distinct batches of the MBS run's dataset statistics, each run
for --seconds, alternated twice, with the SM clock sampled (bench.ClockSampler).

python tools/probe_nostream_data.py --config n1 --seconds 60
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2110_12484_b200.workloads import WORKLOADS, synthetic_data  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="n1")
ap.add_argument("--seconds", type=float, default=60.0)
args = ap.parse_args()
w = WORKLOADS[args.config]
dev = torch.device("cuda:0")
torch.backends.cudnn.benchmark = True
b = w.micro
x, y = synthetic_data(w, 64 * b, seed=0, device="cpu")
data = (x.to(dev), y.to(dev))
out = []
for rep in range(2):
    for kind in ("two_batches", "pool64"):
        with bench.ClockSampler(0) as ck:
            r = bench.no_stream_baseline(w, dev, b, 3, 3, 1, ops="native", min_s=args.seconds,
                                         data=data if kind == "pool64" else None)
        r.pop("events")
        r["clocks"] = ck.summary()
        r["kind"] = kind
        out.append(r)
        print(json.dumps({"kind": kind, "value": r["value"], "sm_mhz": r["clocks"]["sm_mhz"],
                          "per_mhz": r["value"] / r["clocks"]["sm_mhz"], "data": r["data"]}), flush=True)
