"""Print the markdown table of the bench lines committed under profiles/ (used for profiles/README.md)."""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ROWS = [("r01_bench_c2.json", "C2 ResNet-50 @224, 1024/128, SGD — one `train_epoch` call over 8 shuffled mini-batches"),
        ("r01_bench_c3.json", "C3 U-Net @384, 256/48 (ragged 16), Adam, bce_dice"),
        ("r01_bench_c4.json", "C4 ResNet-50, ONE mini-batch of 300,032 (2,344 × 128), 45.2 GB host-resident uint8"),
        ("r01_bench_c5.json", "C5 U-Net @768, micro auto-sized from measured HBM")]


def f(v, nd=0):
    return "—" if v is None else (f"{v:,.{nd}f}")


def main():
    print("| file | workload | value (HBM-resident) | e2e (host-streamed) | no-stream, same model | no-stream, stock torch ops "
          "| K1 frac | K5 frac | model FLOP frac | H2D overlap | clocks |")
    print("|---|---|---:|---:|---:|---:|---:|---:|---:|---:|---|")
    for name, what in ROWS:
        p = os.path.join(ROOT, "profiles", name)
        if not os.path.exists(p):
            continue
        d = json.load(open(p))
        nt = d.get("no_stream_torch_ops") or d.get("no_stream_torch_bn") or {}
        nts = f(nt.get("value")) + (f" (batch {nt['batch']})" if nt.get("batch") and nt["batch"] != d["config"]["micro_batch"] else "")
        auto = d["config"].get("autosize")
        if auto:
            what += f" (micro {auto['micro']}, mini {auto['mini']}, {auto['data_bytes_per_sample'] / 1e9:.2f} GB/sample)"
        ck = d.get("clocks") or {}
        print(f"| `{name}` | {what} | {f(d['value'])} | {f(d['e2e']['value'])} | {f(d['no_stream']['value'])} | {nts} "
              f"| {f(d['roofline']['frac'], 3)} | {f((d.get('roofline_k5') or {}).get('frac'), 3)} "
              f"| {f((d.get('model_flops') or {}).get('frac'), 3)} | {f(d.get('h2d_overlap_pct'), 1)} % "
              f"| {ck.get('sm_mhz')} MHz {','.join(ck.get('reasons') or []) or 'no throttle'} |")


if __name__ == "__main__":
    main()
