#!/bin/bash
# K1 A/B under a READ flush (clean L2): compiled variants x CTA tile
run() { MBS_NATIVE_LIB=$PWD/$1 MBS_K1_TILE=$2 python tools/kbench.py --iters 40 > /tmp/kb.json 2>&1
  python - "$1" "$2" <<'PY'
import json, sys
d = json.load(open("/tmp/kb.json"))
print(sys.argv[1].split("/")[-1], "tile", sys.argv[2], " ".join(f"{k}={d[k]['us_median']:.1f}us/{d[k]['frac']:.3f}" for k in ("k1_assign", "k1_accumulate", "torch_add_P_f32")))
PY
}
run paper_2110_12484_b200/libmbs_native.so 8192
run paper_2110_12484_b200/libmbs_native.so 4096
run paper_2110_12484_b200/libmbs_native.so 16384
for v in ncacc plaing u2m8 u8 ncacc_plain; do run build/variants/$v.so 8192; done
