#!/bin/bash
# K1 A/B: compiled variants (build/variants/*.so) x CTA tile (MBS_K1_TILE) via tools/kbench.py
for lib in paper_2110_12484_b200/libmbs_native.so build/variants/*.so; do
  for t in 0 8192 32768; do
    MBS_NATIVE_LIB=$PWD/$lib MBS_K1_TILE=$t python tools/kbench.py --iters 30 > /tmp/kb.json 2>&1
    python - "$lib" "$t" <<'PY'
import json, sys
d = json.load(open("/tmp/kb.json"))
print(sys.argv[1].split("/")[-1], "tile", sys.argv[2], " ".join(f"{k}={d[k]['us_median']:.1f}us/{d[k]['frac']:.3f}" for k in ("k1_assign", "k1_accumulate", "k1_accumulate_norm", "torch_add_P_f32")))
PY
  done
done
