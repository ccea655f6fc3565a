#!/bin/bash
# K2 staging A/B: MBS_K2_PATH 0 = per-row kernels, 1 = grid-stride vector kernel, 2 = smem-staged NHWC,
# 3 = bulk-async (TMA) ring; MBS_K2_TILE 2048|4096 for path 3
for pt in 2:4096 3:2048 4:2048; do
  MBS_K2_PATH=${pt%%:*} MBS_K2_TILE=${pt##*:} python tools/kbench.py --iters 30 > /tmp/kb.json 2>&1
  python - "$pt" <<'PY'
import json, sys
d = json.load(open("/tmp/kb.json"))
print("path", sys.argv[1], " ".join(f"{k}={d[k]['us_median']:.1f}us/{d[k]['frac']:.3f}" for k in d if k.startswith("k2")))
PY
done
