#!/bin/bash
# K1 A/B: current tiled kernel vs the round's first chunk-per-CTA kernel vs the tiled kernel without a register cap
for lib in paper_2110_12484_b200/libmbs_native.so build/variants/chunk_old.so build/variants/tile_mb1.so; do
  for rep in 1 2; do
    MBS_NATIVE_LIB=$PWD/$lib python tools/kbench.py --iters 40 > /tmp/kb.json 2>&1
    python - "$lib" <<'PY'
import json, sys
d = json.load(open("/tmp/kb.json"))
print(sys.argv[1].split("/")[-1], " ".join(f"{k}={d[k]['us_median']:.1f}us/{d[k]['frac']:.3f}" for k in ("k1_assign", "k1_accumulate", "k1_accumulate_norm", "torch_add_P_f32")))
PY
  done
done
