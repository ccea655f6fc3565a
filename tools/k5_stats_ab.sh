#!/bin/bash
# K5 statistics kernel: channel-vector group cap A/B (MBS_K5_STATS_GV) on the ResNet BN layer shapes (ncu, cold)
for gv in 256 64 32; do
  MBS_K5_STATS_GV=$gv timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_bn_reduce|k_bn_stats" --csv python tools/k5_ncu.py > /tmp/k5s_$gv.csv 2>/dev/null
  python - "$gv" <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(f"/tmp/k5s_{sys.argv[1]}.csv")) if len(r) > 10]
h = rows[0]; ki = h.index("Kernel Name"); vi = h.index("Metric Value")
t = [(r[ki].split("(")[0].split("::")[-1][:22], float(r[vi].replace(",", "")) / 1e3) for r in rows[1:]]
print("gv", sys.argv[1], " ".join(f"{k}:{v:.1f}" for k, v in t))
PY
done
