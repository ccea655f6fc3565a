#!/bin/bash
# K3 unroll (compiled variants) and K2 grid policy A/B via tools/kbench.py
for lib in paper_2110_12484_b200/libmbs_native.so build/variants/k3u1.so build/variants/k3u4.so; do
  MBS_NATIVE_LIB=$PWD/$lib python tools/kbench.py --iters 40 > /tmp/kb.json 2>&1
  python - "$lib" <<'PY'
import json, sys
d = json.load(open("/tmp/kb.json"))
print(sys.argv[1].split("/")[-1], " ".join(f"{k}={d[k]['us_median']:.1f}us/{d[k]['frac']:.3f}" for k in ("k3_sgd", "k3_adam", "k2_stage_u8_bf16_nhwc")))
PY
done
MBS_K2_GRID=resident python tools/kbench.py --iters 40 > /tmp/kb.json 2>&1
python - <<'PY'
import json
d = json.load(open("/tmp/kb.json"))
print("k2 grid=resident", " ".join(f"{k}={d[k]['us_median']:.1f}us/{d[k]['frac']:.3f}" for k in d if k.startswith("k2")))
PY
