#!/bin/bash
# K2 staging A/B: MBS_K2_PATH 0 = per-row kernels, 1 = grid-stride vector kernel, 2 = smem-staged NHWC
for p in 0 1 2; do
  MBS_K2_PATH=$p python tools/kbench.py --iters 30 > /tmp/kb.json 2>&1
  python - "$p" <<'PY'
import json, sys
d = json.load(open("/tmp/kb.json"))
print("path", sys.argv[1], " ".join(f"{k}={d[k]['us_median']:.1f}us/{d[k]['frac']:.3f}" for k in d if k.startswith("k2")))
PY
done
