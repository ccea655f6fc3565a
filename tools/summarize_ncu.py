"""Summarise ncu outputs into profiles/: launch-list shares and full-set metrics of the MBS kernels.

python tools/summarize_ncu.py <launches.csv> <full.ncu-rep> <tag>
"""
import collections
import csv
import json
import subprocess
import sys

launches, rep, tag = sys.argv[1], sys.argv[2], sys.argv[3]
UNIT = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}

rows = list(csv.reader(open(launches)))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, ui, vi = h.index("Kernel Name"), h.index("Metric Unit"), h.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
total = 0.0
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    us = float(r[vi].replace(",", "")) * UNIT[r[ui]]
    total += us
    name = r[ki].split("(")[0]
    agg[name][0] += 1
    agg[name][1] += us
lines = [f"# ncu launch list ({tag}): one profiled MBS mini-batch (tools/profile_step.py)",
         "", f"launches: {sum(v[0] for v in agg.values())}, serialized cold-cache kernel time: {total / 1e3:.2f} ms",
         "", "| share | total us | launches | kernel |", "|---:|---:|---:|---|"]
for name, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:25]:
    lines.append(f"| {100 * us / total:.3f}% | {us:.1f} | {n} | `{name[:90]}` |")
mbs = {k: v for k, v in agg.items() if "mbs::" in k or k.split()[-1].startswith("k_")}
lines += ["", "MBS kernels (this repo):", "", "| share | total us | launches | kernel |", "|---:|---:|---:|---|"]
for name, (n, us) in sorted(mbs.items(), key=lambda kv: -kv[1][1]):
    lines.append(f"| {100 * us / total:.3f}% | {us:.1f} | {n} | `{name}` |")
lines.append(f"| **{100 * sum(v[1] for v in mbs.values()) / total:.3f}%** | {sum(v[1] for v in mbs.values()):.1f} | "
             f"{sum(v[0] for v in mbs.values())} | all MBS kernels |")
open(f"profiles/{tag}_launches.md", "w").write("\n".join(lines) + "\n")

raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
hh = rr[0]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum"]
idx = [hh.index(w) for w in want if w in hh]
units = [rr[1][i] for i in idx]
recs = []
for r in rr[2:]:
    recs.append({hh[i]: (r[i] if i == idx[0] else float(r[i].replace(",", ""))) for i in idx})
out = {"units": dict(zip([hh[i] for i in idx], units)), "kernels": recs}
json.dump(out, open(f"profiles/{tag}_ncu_full.json", "w"), indent=1)
md = [f"# ncu --set full ({tag}): MBS kernels, one mini-batch", "",
      "| kernel | us | DRAM read MB | DRAM write MB | DRAM % peak | regs | warps active % |", "|---|---:|---:|---:|---:|---:|---:|"]
for r in recs:
    md.append(f"| `{r['Kernel Name'][:60]}` | {r['gpu__time_duration.sum']:.1f} | {r['dram__bytes_read.sum']:.1f} | "
              f"{r['dram__bytes_write.sum']:.1f} | {r['gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed']:.1f} | "
              f"{r['launch__registers_per_thread']:.0f} | {r['sm__warps_active.avg.pct_of_peak_sustained_active']:.1f} |")
open(f"profiles/{tag}_ncu_full.md", "w").write("\n".join(md) + "\n")
acc = [r for r in recs if "k_accum<0, 0" in r["Kernel Name"]]   # acc += s*g (fp32 or MIXED bf16 grads)
if acc:
    mb = (acc[0]["dram__bytes_read.sum"] + acc[0]["dram__bytes_write.sum"])
    scale = 1e6 if units[idx.index(hh.index("dram__bytes_read.sum"))] == "Mbyte" else 1.0
    json.dump({"kernel": acc[0]["Kernel Name"][:40] + " (acc += s*g)", "dram_bytes_per_launch": mb * scale,
               "source": f"profiles/{tag}_ncu_full.json"}, open("profiles/ncu_k1_traffic.json", "w"), indent=1)
print("\n".join(lines[:8]))
print("\n".join(md))
