# K2 warp-specialised kernel (MBS_K2_PATH=5, 8 or 16 px per lane) vs the flat kernel (4): bit-exactness, then
# the ncu launch-list time of every K2 launch of one C2 mini-batch (8 micro-batches), each variant twice
timeout 900 python -m pytest tests/test_stage_gpu.py -q -m gpu -p no:cacheprovider > gpurun_out/k2ws_tests.log 2>&1; tail -2 gpurun_out/k2ws_tests.log
for v in 4:8 5:8 5:16 4:8 5:8 5:16; do
  p=${v%%:*}; x=${v##*:}
  MBS_K2_PATH=$p MBS_K2_WS_PX=$x timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_active.avg,gpc__cycles_elapsed.max \
      --clock-control none -k regex:"k_stage" --csv --log-file gpurun_out/k2ws_${p}_${x}.csv python tools/profile_step.py > /dev/null 2>&1
  python - "$p" "$x" <<'PY'
import csv, sys
p, x = sys.argv[1:]
rows = list(csv.reader(open(f"gpurun_out/k2ws_{p}_{x}.csv")))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]; h = rows[hi]
vi, mi, ui, ki = h.index("Metric Value"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Kernel Name")
m = {}
for r in rows[hi + 1:]:
    if len(r) > vi: m.setdefault(r[mi], []).append(float(r[vi].replace(",", "")) * (1e-3 if r[ui] in ("ns", "nsecond") else 1))
t = m["gpu__time_duration.sum"]
print("PATH", p, "PX", x, rows[hi+1][ki][:40], "us", [round(v, 2) for v in t], "mean", round(sum(t) / len(t), 2),
      "GB/s", round(57802752 / (sum(t) / len(t)) / 1e3), "sm_active/elapsed", round(sum(m["sm__cycles_active.avg"]) / sum(m["gpc__cycles_elapsed.max"]), 3))
PY
done
