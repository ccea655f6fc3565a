# the remaining BASELINE configs at the final kernels: C1, C2 (fits HBM), C3 (U-Net 256/48, tail 16), C5 (U-Net@768 auto-sized)
for c in c1 c2 c3 c5; do
  timeout 1500 python bench.py --config $c --no-fp32-context --no-cpu-baseline > gpurun_out/c8_bench_$c.json 2> gpurun_out/c8_bench_$c.err
  echo "$c rc=$?"
done
python - <<'PY'
import json
for c in ["c1","c2","c3","c5"]:
    try:
        d=json.load(open(f"gpurun_out/c8_bench_{c}.json"))
        print(c, round(d["value"]), round(d["e2e"]["value"]), d.get("e2e_vs_no_stream"), (d.get("no_stream") or {}).get("value"), d.get("h2d_overlap_pct"), d["roofline"]["frac"], d["config"].get("autosize"), d["clocks"])
    except Exception as e: print(c, "ERR", e)
PY
