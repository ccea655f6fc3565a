# K2 vs same-byte torch kernels under ncu (launch list with DRAM bytes), cold L2 per launch (ncu default)
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_active.avg,gpc__cycles_elapsed.max \
    --clock-control none --csv --log-file gpurun_out/k2ref.csv python tools/k2_copy_ref.py > gpurun_out/k2ref.out 2>&1
tail -2 gpurun_out/k2ref.out
python - <<'PY'
import csv
rows = list(csv.reader(open("gpurun_out/k2ref.csv")))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]; h = rows[hi]
vi, mi, ui, ki, ii = h.index("Metric Value"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Kernel Name"), h.index("ID")
k = {}
for r in rows[hi + 1:]:
    if len(r) <= vi: continue
    v = float(r[vi].replace(",", ""))
    if r[ui] in ("ns", "nsecond"): v *= 1e-3
    if r[ui] in ("byte",): v *= 1e-6
    if r[ui] in ("Kbyte",): v *= 1e-3
    if r[ui] in ("Gbyte",): v *= 1e3
    k.setdefault((int(r[ii]), r[ki][:60]), {})[r[mi]] = v
for (i, n), m in sorted(k.items()):
    print(f"{i:3d} {n:60s} {m['gpu__time_duration.sum']:7.2f} us  rd {m['dram__bytes_read.sum']:6.1f} MB  wr {m['dram__bytes_write.sum']:6.1f} MB  active {m['sm__cycles_active.avg']/m['gpc__cycles_elapsed.max']:.2f}")
PY
