"""SPEC data-cli: experiment config, the run driver, metrics reports and the command line.

The reference declares ``mbstream = "mbstream.cli:main"`` (``pkg/pyproject.toml:15-16``) but ships no
``cli.py``; SPEC.md specifies the module. This is that module over the B200 path: ``run_experiment``
trains with ``engine.train_epoch`` (K1-K7, the streamer, CUDA graphs) and runs the no-MBS baseline iff
its mini-batch fits the device — the MEASURED device: per-sample bytes from a probe, capacity from
``cudaMemGetInfo`` or the configured ``memory.capacity_bytes`` — recording "Failed" otherwise (Tables
3-4). The "simulated" makespan of the SPEC is the MEASURED schedule here (``streaming.ScheduleTracer``).

Config text format: one ``key = value`` per line, dotted section prefixes, field names as
keys; floats are written with ``repr`` (shortest round-trip form), so a config round-trips bit-exactly.
CSV: fixed column order, header row, floats with 17 significant digits.
Exit codes: 0 success, 2 configuration error, 3 infeasible memory (even MBS cannot fit).
"""

from __future__ import annotations

import argparse
import csv
import dataclasses
import gc
import io
import json
import math
import os
import sys
import time
from dataclasses import dataclass, field

import numpy as np

from .datasets import DatasetSpec, make_dataset
from .errors import ConfigError, IdxFormatError, ModelDoesNotFitError

MODELS = ("resnet18", "resnet50", "unet", "convnet", "mlp")
OUTPUT_ROOT_ENV = "MBS_OUTPUT_ROOT"
CSV_COLUMNS = ("epoch", "mini_batch_index", "loss", "metric", "step_count", "wall_seconds", "makespan_seconds")


@dataclass
class ExperimentConfig:
    """fully serializable; every run embeds its resolved copy."""

    model: str = "convnet"
    model_ops: str = "native"
    dataset: DatasetSpec = field(default_factory=lambda: DatasetSpec("synthetic_classification", 256, (3, 32, 32),
                                                                      n_classes=10))
    loss: str = "cross_entropy"
    optimizer: str = "sgd"
    lr: float = 0.01
    momentum: float = 0.9
    weight_decay: float = 5e-4
    mini_batch_size: int = 64
    micro_batch_size: object = 8          # int, "auto" (fit_micro_batch on measured memory) or None (no MBS)
    normalization: str = "exact_weighted"
    epochs: int = 1
    seeds: tuple = (0,)
    precision: str = "bf16"               # "bf16" (autocast + bf16 shadow weights) or "fp32"
    capacity_bytes: int = 0               # 0: the measured free HBM
    output_dir: str = ""

    def validate(self) -> None:
        from .engine import NORMALIZATION_MODES
        from .losses import LOSS_KINDS
        self.dataset.validate()
        if self.model not in MODELS:
            raise ConfigError(f"model.name must be one of {MODELS}, got {self.model!r}")
        if self.model_ops not in ("native", "torch"):
            raise ConfigError("model.ops must be 'native' or 'torch'")
        if self.loss not in LOSS_KINDS:
            raise ConfigError(f"train.loss must be one of {LOSS_KINDS}")
        if self.optimizer not in ("sgd", "adam"):
            raise ConfigError("optim.kind must be 'sgd' or 'adam'")
        if not self.lr > 0 or self.momentum < 0 or self.weight_decay < 0:
            raise ConfigError("optim.lr must be > 0 and momentum / weight_decay >= 0")
        if self.mini_batch_size < 1 or self.epochs < 1 or not self.seeds:
            raise ConfigError("mbs.mini_batch_size and train.epochs must be >= 1, train.seeds non-empty")
        m = self.micro_batch_size
        if not (m is None or m == "auto" or (isinstance(m, int) and m >= 1)):
            raise ConfigError("mbs.micro_batch_size must be a positive integer, 'auto' or 'none'")
        if self.normalization not in NORMALIZATION_MODES:
            raise ConfigError(f"mbs.normalization must be one of {NORMALIZATION_MODES}")
        if self.precision not in ("bf16", "fp32"):
            raise ConfigError("train.precision must be 'bf16' or 'fp32'")
        if self.capacity_bytes < 0:
            raise ConfigError("memory.capacity_bytes must be >= 0")
        if (self.loss == "cross_entropy") != (self.dataset.kind != "synthetic_segmentation"):
            raise ConfigError("cross_entropy trains classification datasets; segmentation needs bce / bce_dice")


# ---------------------------------------------------------------------------
# config text format
# ---------------------------------------------------------------------------

_KEYS = (  # (key, path) in file order
    ("model.name", "model"), ("model.ops", "model_ops"),
    ("dataset.kind", "dataset.kind"), ("dataset.n_samples", "dataset.n_samples"),
    ("dataset.input_shape", "dataset.input_shape"), ("dataset.n_classes", "dataset.n_classes"),
    ("dataset.mask_shape", "dataset.mask_shape"), ("dataset.seed", "dataset.seed"), ("dataset.path", "dataset.path"),
    ("dataset.labels_path", "dataset.labels_path"), ("dataset.separation", "dataset.separation"),
    ("optim.kind", "optimizer"), ("optim.lr", "lr"), ("optim.momentum", "momentum"),
    ("optim.weight_decay", "weight_decay"),
    ("mbs.mini_batch_size", "mini_batch_size"), ("mbs.micro_batch_size", "micro_batch_size"),
    ("mbs.normalization", "normalization"),
    ("train.loss", "loss"), ("train.epochs", "epochs"), ("train.seeds", "seeds"), ("train.precision", "precision"),
    ("memory.capacity_bytes", "capacity_bytes"), ("run.output_dir", "output_dir"),
)
_TUPLES = {"dataset.input_shape", "dataset.mask_shape", "train.seeds"}
_INTS = {"dataset.n_samples", "dataset.n_classes", "dataset.seed", "mbs.mini_batch_size", "train.epochs",
         "memory.capacity_bytes"}
_FLOATS = {"dataset.separation", "optim.lr", "optim.momentum", "optim.weight_decay"}


def _fmt(key: str, v) -> str:
    if key in _TUPLES:
        return ",".join(str(int(t)) for t in v)
    if key in _FLOATS:
        return repr(float(v))
    if key == "mbs.micro_batch_size":
        return "none" if v is None else str(v)
    return str(v)


def _parse(key: str, text: str):
    t = text.strip()
    try:
        if key in _TUPLES:
            return tuple(int(p) for p in t.split(",") if p.strip()) if t else ()
        if key in _INTS:
            return int(t)
        if key in _FLOATS:
            return float(t)
        if key == "mbs.micro_batch_size":
            return None if t.lower() == "none" else ("auto" if t.lower() == "auto" else int(t))
    except ValueError:
        raise ConfigError(f"{key}: cannot parse {text!r}") from None
    return t


def dumps(cfg: ExperimentConfig) -> str:
    lines = []
    for key, path in _KEYS:
        obj = cfg
        for part in path.split("."):
            obj = getattr(obj, part)
        lines.append(f"{key} = {_fmt(key, obj)}")
    return "\n".join(lines) + "\n"


def loads(text: str) -> ExperimentConfig:
    known = dict(_KEYS)
    vals = {}
    for no, raw in enumerate(text.splitlines(), 1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        if "=" not in line:
            raise ConfigError(f"line {no}: expected 'key = value', got {raw!r}")
        key, val = (p.strip() for p in line.split("=", 1))
        if key not in known:
            raise ConfigError(f"line {no}: unknown key {key!r}")
        if key in vals:
            raise ConfigError(f"line {no}: duplicate key {key!r}")
        vals[key] = _parse(key, val)
    ds_fields = {k.split(".", 1)[1]: v for k, v in vals.items() if k.startswith("dataset.")}
    if "kind" not in ds_fields:
        raise ConfigError("dataset.kind is required")
    ds = DatasetSpec(**ds_fields)
    top = {known[k]: v for k, v in vals.items() if not k.startswith("dataset.")}
    cfg = ExperimentConfig(dataset=ds, **top)
    cfg.validate()
    return cfg


def load(path: str) -> ExperimentConfig:
    try:
        with open(path) as f:
            return loads(f.read())
    except OSError as e:
        raise ConfigError(f"cannot read config {path}: {e}") from None


# ---------------------------------------------------------------------------
# CSV (17 significant digits)
# ---------------------------------------------------------------------------

def _cell(v) -> str:
    if v is None:
        return ""
    if isinstance(v, float):
        return "nan" if math.isnan(v) else format(v, ".17g")
    return str(v)


def write_csv(path: str, rows: list, columns=CSV_COLUMNS) -> None:
    with open(path, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(columns)
        for r in rows:
            w.writerow([_cell(r.get(c)) for c in columns])


# ---------------------------------------------------------------------------
# models
# ---------------------------------------------------------------------------

def build_model(cfg: ExperimentConfig):
    from torch import nn
    from . import workloads
    ds = cfg.dataset
    shape = tuple(ds.input_shape)
    k = max(2, int(ds.n_classes))
    if cfg.model in ("resnet18", "resnet50"):
        import torchvision
        m = getattr(torchvision.models, cfg.model)(num_classes=k)
        if shape[0] != 3:
            m.conv1 = nn.Conv2d(shape[0], 64, 7, 2, 3, bias=False)
    elif cfg.model == "unet":
        m = workloads.UNet(shape[0], 1)
    elif cfg.model == "convnet":
        m = nn.Sequential(nn.Conv2d(shape[0], 16, 3, padding=1), nn.BatchNorm2d(16), nn.ReLU(), nn.MaxPool2d(2),
                          nn.Conv2d(16, 32, 3, padding=1), nn.BatchNorm2d(32), nn.ReLU(), nn.AdaptiveAvgPool2d(1),
                          nn.Flatten(), nn.Linear(32, k))
    else:
        m = nn.Sequential(nn.Flatten(), nn.Linear(int(np.prod(shape)), 64), nn.ReLU(), nn.Linear(64, k))
    if cfg.model_ops == "native":
        workloads.make_native(m)
    return m


def _metric(cfg):
    from . import losses
    if cfg.dataset.kind == "synthetic_segmentation":
        import torch
        return "iou", lambda out, y: losses.iou(torch.sigmoid(out.float()), y)
    return "accuracy", losses.accuracy


# ---------------------------------------------------------------------------
# the run driver
# ---------------------------------------------------------------------------

def _seed_for(seed: int, name: str) -> int:
    from .rng import stream_key
    return stream_key(seed, name) % (2 ** 63)


def _train(cfg, x, y, micro, seed, dev, tracer=True):
    """One training run (MBS when ``micro`` is an int, the no-MBS baseline when None): rows + wall + schedules."""
    import torch
    from . import engine, graphs, optim, streaming
    from .streamer import Staging
    from .tensor import ParameterSet
    torch.manual_seed(_seed_for(seed, "init"))
    model = build_model(cfg).to(dev)
    if x.dim() == 4:
        model = model.to(memory_format=torch.channels_last)
    bf16 = cfg.precision == "bf16"
    params = ParameterSet(model, shadow=torch.bfloat16 if bf16 else None)
    st = optim.sgd_state(cfg.lr, cfg.momentum, cfg.weight_decay) if cfg.optimizer == "sgd" else \
        optim.adam_state(cfg.lr, cfg.weight_decay)
    staging = Staging(torch.bfloat16 if bf16 else torch.float32, x.dim() == 4, target_dtype=torch.float32)
    _, metric = _metric(cfg)
    tr = streaming.ScheduleTracer(dev, nvtx=False) if tracer else None
    streamer = engine.make_streamer(x, y, micro or cfg.mini_batch_size) if x.device.type == "cpu" else None
    rows = []
    t0 = time.perf_counter()
    try:
        for e in range(cfg.epochs):
            te = time.perf_counter()
            es = engine.train_epoch(model, params, x, y, mini_batch_size=cfg.mini_batch_size,
                                    micro_batch_size=micro, normalization=cfg.normalization, loss_kind=cfg.loss,
                                    optimizer_state=st, seed=seed, epoch_index=e, prefetch=True, staging=staging,
                                    autocast_dtype=torch.bfloat16 if bf16 else None, streamer=streamer,
                                    metric_fn=metric, tracer=tr)
            wall = time.perf_counter() - te
            sch = tr.schedules()[-len(es.mini_losses):] if tr is not None else []
            base = es.step_count - len(es.mini_losses)
            for i, (lv, mv) in enumerate(zip(es.mini_losses, es.mini_metrics)):
                rows.append({"epoch": e, "mini_batch_index": i, "loss": float(lv), "metric": float(mv),
                             "step_count": base + i + 1, "wall_seconds": None,
                             "makespan_seconds": sch[i].makespan if i < len(sch) else None})
            sizes = np.asarray(es.mini_sizes, np.float64)
            rows.append({"epoch": e, "mini_batch_index": "epoch", "loss": float(es.mean_loss),
                         "metric": float(np.dot(es.mini_metrics, sizes) / sizes.sum()), "step_count": es.step_count,
                         "wall_seconds": wall,
                         "makespan_seconds": float(sum(s.makespan for s in sch)) if sch else None})
    finally:
        if streamer is not None:
            streamer.close()
        graphs.clear()
    total = time.perf_counter() - t0
    schedules = tr.schedules() if tr is not None else []
    del model, params, st
    return rows, total, schedules


def _probe_budget(cfg, x, y, dev):
    """Measured MemoryBudget of this config's model (memory.measure_budget), capacity overridden by config."""
    import torch
    from . import memory
    from .streamer import Staging, stage_rows
    gc.collect()                                  # a previous run's graphs / tensors are not this model's
    base = torch.cuda.memory_allocated(dev)
    torch.manual_seed(0)
    model = build_model(cfg).to(dev)
    if x.dim() == 4:
        model = model.to(memory_format=torch.channels_last)
    bf16 = cfg.precision == "bf16"
    st = Staging(torch.bfloat16 if bf16 else torch.float32, x.dim() == 4)

    def make_batch(k):
        k = min(k, x.shape[0])
        xb = stage_rows(x[:k].to(dev) if x.device.type == "cpu" else x[:k], x.dtype, tuple(x.shape[1:]), None, 0, k,
                        st, dev)
        yb = y[:k].to(dev)
        return xb, (yb.float() if yb.dtype == torch.uint8 else yb)
    n = min(8, x.shape[0])
    probe = (max(1, n // 2), n) if n >= 2 else (1, 2)
    b = memory.measure_budget(model, make_batch, cfg.loss, optimizer_kind=cfg.optimizer,
                              autocast_dtype=torch.bfloat16 if bf16 else None, probe=probe, baseline_bytes=base)
    if cfg.capacity_bytes:
        b = memory.MemoryBudget(capacity_bytes=int(cfg.capacity_bytes), param_bytes=b.param_bytes,
                                data_bytes_per_sample=b.data_bytes_per_sample,
                                fixed_overhead_bytes=b.fixed_overhead_bytes)
    del model
    torch.cuda.empty_cache()
    return b


def _unique_dir(root: str, stem: str) -> str:
    os.makedirs(root, exist_ok=True)
    i = 0
    while True:
        d = os.path.join(root, f"{stem}-{i:03d}")
        try:
            os.makedirs(d)
            return d
        except FileExistsError:
            i += 1


def run_experiment(cfg: ExperimentConfig, out_root: str | None = None) -> str:
    """train per config; write metrics.csv, summary.json, the resolved config, and the
    measured stream / memory reports into a fresh run directory; returns its path."""
    import torch
    from . import memory, streaming
    cfg.validate()
    if not torch.cuda.is_available():
        raise RuntimeError("run_experiment trains on the B200 path and needs a CUDA device")
    dev = torch.device("cuda", torch.cuda.current_device())
    root = out_root or cfg.output_dir or os.environ.get(OUTPUT_ROOT_ENV, "runs")
    x_np, y_np = make_dataset(dataclasses.replace(cfg.dataset, seed=cfg.dataset.seed))
    x, y = torch.from_numpy(np.ascontiguousarray(x_np)), torch.from_numpy(np.ascontiguousarray(y_np))
    x, y = x.pin_memory(), y.pin_memory()       # host-resident dataset, streamed by the native H2D streamer
    budget = _probe_budget(cfg, x, y, dev)
    micro = cfg.micro_batch_size
    if micro == "auto":
        micro = memory.auto_micro_batch(budget, cfg.mini_batch_size, build_model(cfg))
    elif micro is not None:
        micro = min(int(micro), cfg.mini_batch_size)
    if micro is not None and not budget.fits(micro):
        raise ModelDoesNotFitError(f"micro-batch {micro} needs {budget.bytes_for(micro)} bytes, capacity "
                                   f"{budget.capacity_bytes}")
    resolved = dataclasses.replace(cfg, micro_batch_size=micro)
    name = f"{cfg.model}-{cfg.dataset.kind.split('_')[-1]}-mini{cfg.mini_batch_size}-micro{micro or 'none'}"
    run = _unique_dir(root, name)
    with open(os.path.join(run, "config.txt"), "w") as f:
        f.write(dumps(resolved))
    metric_name, _ = _metric(cfg)
    baseline_fits = budget.fits(cfg.mini_batch_size)
    per_seed, base_seed, all_rows, base_rows = [], [], [], []
    mbs_sched = base_sched = None
    for seed in cfg.seeds:
        rows, wall, sch = _train(resolved, x, y, micro, seed, dev)
        for r in rows:
            r["seed"] = seed
        all_rows += rows
        ep = [r for r in rows if r["mini_batch_index"] == "epoch"]
        per_seed.append({"seed": seed, "final_metric": ep[-1]["metric"], "max_metric": max(r["metric"] for r in ep),
                         "final_loss": ep[-1]["loss"], "wall_seconds": wall})
        mbs_sched = sch[-1] if sch else mbs_sched
        if micro is not None and baseline_fits:
            try:
                brows, bwall, bsch = _train(resolved, x, y, None, seed, dev)
            except torch.OutOfMemoryError:
                baseline_fits = False
                torch.cuda.empty_cache()
            else:
                for r in brows:
                    r["seed"] = seed
                base_rows += brows
                bep = [r for r in brows if r["mini_batch_index"] == "epoch"]
                base_seed.append({"seed": seed, "final_metric": bep[-1]["metric"],
                                  "max_metric": max(r["metric"] for r in bep), "final_loss": bep[-1]["loss"],
                                  "wall_seconds": bwall})
                base_sched = bsch[-1] if bsch else base_sched
    cols = CSV_COLUMNS + ("seed",)
    write_csv(os.path.join(run, "metrics.csv"), all_rows, cols)
    if base_rows:
        write_csv(os.path.join(run, "baseline_metrics.csv"), base_rows, cols)

    def agg(rs):
        mx = np.asarray([r["max_metric"] for r in rs], np.float64)
        return {"max_metric_mean": float(mx.mean()), "max_metric_std": float(mx.std(ddof=1)) if len(mx) > 1 else 0.0,
                "final_metric_mean": float(np.mean([r["final_metric"] for r in rs])),
                "wall_seconds_mean": float(np.mean([r["wall_seconds"] for r in rs])), "per_seed": rs}
    summary = {"metric": metric_name, "mini_batch_size": cfg.mini_batch_size, "micro_batch_size": micro,
               "mbs": agg(per_seed),
               "baseline": (agg(base_seed) if base_seed else ("Failed" if micro is not None else "n/a (no MBS run)")),
               "config": dumps(resolved)}
    with open(os.path.join(run, "summary.json"), "w") as f:
        json.dump(summary, f, indent=1)
    with open(os.path.join(run, "memory_report.json"), "w") as f:
        json.dump({"capacity_bytes": budget.capacity_bytes, "resident_bytes": budget.resident_bytes,
                   "data_bytes_per_sample": budget.data_bytes_per_sample, "micro_batch": micro,
                   "mini_batch_fits": budget.fits(cfg.mini_batch_size),
                   "capacity_source": "memory.capacity_bytes" if cfg.capacity_bytes else "measured free HBM"}, f,
                  indent=1)
    if mbs_sched is not None:
        rep = streaming.overhead_report(mbs_sched, base_sched)
        with open(os.path.join(run, "stream_report.json"), "w") as f:
            json.dump({"mbs_makespan_s": rep.mbs_makespan, "baseline_makespan_s": rep.baseline_makespan,
                       "overhead_pct": rep.overhead_pct, "baseline_failed": rep.baseline_failed,
                       "h2d_overlap": streaming.overlap_fraction(mbs_sched),
                       "events": [dataclasses.astuple(e) for e in mbs_sched.events]}, f)
    return run


# ---------------------------------------------------------------------------
# reports
# ---------------------------------------------------------------------------

REPORT_COLUMNS = ("batch_size", "micro_batch_size", "metric_without_mbs", "metric_with_mbs", "time_without_s",
                  "time_with_s")


def compare_report(run_dirs: list, csv_path: str | None = None) -> str:
    """SPEC.md:519-527 / Tables 3-4: one row per run (mini-batch size), baseline cells "Failed" when the
    mini-batch did not fit; returns the aligned text table (and writes the CSV when ``csv_path``)."""
    if len(run_dirs) < 1:
        raise ConfigError("compare needs at least one run directory")
    rows, kinds = [], set()
    for d in run_dirs:
        try:
            with open(os.path.join(d, "summary.json")) as f:
                s = json.load(f)
        except OSError as e:
            raise ConfigError(f"{d}: not a run directory ({e})") from None
        kinds.add(s["metric"])
        b = s["baseline"]
        failed = not isinstance(b, dict)
        rows.append({"batch_size": s["mini_batch_size"], "micro_batch_size": s["micro_batch_size"],
                     "metric_without_mbs": "Failed" if failed else b["max_metric_mean"],
                     "metric_with_mbs": s["mbs"]["max_metric_mean"],
                     "time_without_s": "Failed" if failed else b["wall_seconds_mean"],
                     "time_with_s": s["mbs"]["wall_seconds_mean"]})
    if len(kinds) > 1:
        raise ConfigError(f"incompatible metric kinds: {sorted(kinds)}")
    rows.sort(key=lambda r: r["batch_size"])
    if csv_path:
        write_csv(csv_path, rows, REPORT_COLUMNS)
    cells = [list(REPORT_COLUMNS)] + [[_cell(r[c]) if not isinstance(r[c], float) else f"{r[c]:.6g}"
                                       for c in REPORT_COLUMNS] for r in rows]
    width = [max(len(row[i]) for row in cells) for i in range(len(REPORT_COLUMNS))]
    out = io.StringIO()
    for row in cells:
        out.write("  ".join(v.rjust(width[i]) for i, v in enumerate(row)) + "\n")
    return out.getvalue()


# ---------------------------------------------------------------------------
# command line
# ---------------------------------------------------------------------------

def main(argv: list | None = None) -> int:
    """``train <config>``, ``compare <dirs...>``, ``sweep <config> --mini-batch 16,32,...``,
    ``simulate-memory <config>``, ``simulate-stream <config>``."""
    ap = argparse.ArgumentParser(prog="mbstream")
    sub = ap.add_subparsers(dest="cmd", required=True)
    p = sub.add_parser("train")
    p.add_argument("config")
    p.add_argument("--out", default=None)
    p = sub.add_parser("compare")
    p.add_argument("dirs", nargs="+")
    p.add_argument("--csv", default=None)
    p = sub.add_parser("sweep")
    p.add_argument("config")
    p.add_argument("--mini-batch", required=True)
    p.add_argument("--out", default=None)
    p = sub.add_parser("simulate-memory")
    p.add_argument("config")
    p = sub.add_parser("simulate-stream")
    p.add_argument("config")
    args = ap.parse_args(argv)
    try:
        if args.cmd == "compare":
            print(compare_report(args.dirs, args.csv), end="")
            return 0
        cfg = load(args.config)
        if args.cmd == "train":
            print(run_experiment(cfg, args.out))
        elif args.cmd == "sweep":
            try:
                minis = [int(v) for v in args.mini_batch.split(",") if v.strip()]
            except ValueError:
                raise ConfigError(f"--mini-batch: cannot parse {args.mini_batch!r}") from None
            runs = [run_experiment(dataclasses.replace(cfg, mini_batch_size=m), args.out) for m in minis]
            print(compare_report(runs), end="")
        elif args.cmd == "simulate-memory":
            import torch
            x_np, y_np = make_dataset(cfg.dataset)
            b = _probe_budget(cfg, torch.from_numpy(x_np), torch.from_numpy(y_np), torch.device("cuda"))
            from . import memory
            print(json.dumps({"capacity_bytes": b.capacity_bytes, "resident_bytes": b.resident_bytes,
                              "data_bytes_per_sample": b.data_bytes_per_sample,
                              "fit_micro_batch": memory.fit_micro_batch(b),
                              "mini_batch_fits": b.fits(cfg.mini_batch_size)}))
        else:
            import torch
            from . import streaming
            x_np, y_np = make_dataset(cfg.dataset)
            n = min(len(x_np), 2 * cfg.mini_batch_size)
            one = dataclasses.replace(cfg, epochs=1, micro_batch_size=(None if cfg.micro_batch_size == "auto"
                                                                       else cfg.micro_batch_size))
            rows, wall, sch = _train(one, torch.from_numpy(x_np[:n]).pin_memory(), torch.from_numpy(y_np[:n]),
                                     one.micro_batch_size, cfg.seeds[0], torch.device("cuda"))
            s = sch[-1]
            print(json.dumps({"makespan_s": s.makespan, "h2d_overlap": streaming.overlap_fraction(s),
                              "events": [dataclasses.astuple(e) for e in s.events]}))
    except (ConfigError, IdxFormatError) as e:
        print(f"config error: {e}", file=sys.stderr)
        return 2
    except ModelDoesNotFitError as e:
        print(f"infeasible memory: {e}", file=sys.stderr)
        return 3
    return 0


if __name__ == "__main__":
    sys.exit(main())
