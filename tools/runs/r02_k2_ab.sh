# K2 flat variant A/B: 256-thread CTAs on 2048-pixel tiles (4 CTAs/SM) vs 128-thread CTAs on 1024-pixel tiles
timeout 600 python -m pytest tests/test_stage_gpu.py -q -m gpu -p no:cacheprovider -k every_path > gpurun_out/k2ab_tests.log 2>&1; tail -1 gpurun_out/k2ab_tests.log
for v in 0 128 0 128; do
  MBS_K2_FLAT=$v timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active \
      --clock-control none -k regex:"k_stage" --csv --log-file gpurun_out/k2ab_$v.csv python tools/profile_step.py > /dev/null 2>&1
  python - "$v" <<'PY'
import csv, sys
v = sys.argv[1]
rows = list(csv.reader(open(f"gpurun_out/k2ab_{v}.csv")))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]; h = rows[hi]
vi, mi, ui = h.index("Metric Value"), h.index("Metric Name"), h.index("Metric Unit")
t = [float(r[vi].replace(",", "")) * (1e-3 if r[ui] in ("ns", "nsecond") else 1) for r in rows[hi + 1:] if len(r) > vi and r[mi] == "gpu__time_duration.sum"]
print("MBS_K2_FLAT", v, "us", [round(x, 2) for x in t], "mean", round(sum(t) / len(t), 2))
PY
done
