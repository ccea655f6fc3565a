"""A/B probe: bench.no_stream_baseline (C2) under the K5 cooperative-path switch."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2110_12484_b200.workloads import WORKLOADS  # noqa: E402

torch.backends.cudnn.benchmark = True
w = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
r = bench.no_stream_baseline(w, torch.device("cuda"), w.micro, 8, 3, 1, ops="native")
print(os.environ.get("MBS_K5_FUSED", "1"), os.environ.get("MBS_K5_FUSED_MB", "8"), r["value"], flush=True)
