"""SPEC data-cli run driver on the B200 path: run directories, Failed baselines,
equivalence and reproducibility."""
import csv
import dataclasses
import json
import os

import pytest
import torch

from paper_2110_12484_b200 import cli
from paper_2110_12484_b200.datasets import DatasetSpec

pytestmark = pytest.mark.gpu


def _cfg(**kw):
    base = dict(model="convnet", dataset=DatasetSpec("synthetic_classification", 96, (3, 16, 16), n_classes=4,
                                                     seed=3), mini_batch_size=32, micro_batch_size=8, epochs=2,
                seeds=(1, 2), lr=0.05)
    base.update(kw)
    return cli.ExperimentConfig(**base)


def _rows(path):
    return list(csv.DictReader(open(path)))


def test_run_experiment_writes_the_run_directory(cuda, tmp_path):
    run = cli.run_experiment(_cfg(), str(tmp_path))
    for f in ("config.txt", "metrics.csv", "baseline_metrics.csv", "summary.json", "memory_report.json",
              "stream_report.json"):
        assert os.path.exists(os.path.join(run, f)), f
    rows = _rows(os.path.join(run, "metrics.csv"))
    assert len(rows) == 2 * 2 * (3 + 1)                     # seeds x epochs x (mini-batches + summary row)
    for seed in ("1", "2"):
        steps = [int(r["step_count"]) for r in rows if r["seed"] == seed and r["mini_batch_index"] != "epoch"]
        assert steps == list(range(1, 7))                   # monotone, one step per mini-batch
    s = json.load(open(os.path.join(run, "summary.json")))
    assert s["metric"] == "accuracy" and len(s["mbs"]["per_seed"]) == 2 and s["mbs"]["max_metric_std"] >= 0
    assert isinstance(s["baseline"], dict)                  # the 32-sample mini-batch fits: baseline was run
    assert cli.loads(open(os.path.join(run, "config.txt")).read()).micro_batch_size == 8
    assert json.load(open(os.path.join(run, "stream_report.json")))["mbs_makespan_s"] > 0


def test_baseline_failed_when_the_mini_batch_does_not_fit(cuda, tmp_path):
    """capacity where mini=32 fails the (measured) fit but micro 8 fits -> baseline "Failed"."""
    cfg = _cfg(seeds=(1,), epochs=1)
    x, y = (torch.from_numpy(a) for a in cli.make_dataset(cfg.dataset))
    b = cli._probe_budget(cfg, x, y, cuda)
    cap = b.resident_bytes + b.data_bytes_per_sample * 16       # 16 samples fit, 32 do not
    run = cli.run_experiment(dataclasses.replace(cfg, capacity_bytes=cap), str(tmp_path))
    s = json.load(open(os.path.join(run, "summary.json")))
    assert s["baseline"] == "Failed" and not os.path.exists(os.path.join(run, "baseline_metrics.csv"))
    assert "Failed" in cli.compare_report([run])
    auto = cli.run_experiment(dataclasses.replace(cfg, capacity_bytes=cap, micro_batch_size="auto"), str(tmp_path))
    assert 8 <= json.load(open(os.path.join(auto, "summary.json")))["micro_batch_size"] <= 16   # "auto" fits


def test_mbs_equals_no_mbs_without_batchnorm(cuda, tmp_path):
    """exact_weighted MBS vs the no-MBS baseline, same seed, BN-free model: equal per-epoch losses
    (fp32 here: 1e-5 relative; the SPEC's 1e-8 is the reference's float64)."""
    cfg = _cfg(model="mlp", precision="fp32", seeds=(1,), epochs=3)
    run = cli.run_experiment(cfg, str(tmp_path))
    a = [r for r in _rows(os.path.join(run, "metrics.csv")) if r["mini_batch_index"] == "epoch"]
    b = [r for r in _rows(os.path.join(run, "baseline_metrics.csv")) if r["mini_batch_index"] == "epoch"]
    for ra, rb in zip(a, b):
        assert abs(float(ra["loss"]) - float(rb["loss"])) <= 1e-5 * abs(float(rb["loss"]))


def test_run_is_reproducible_from_its_embedded_config(cuda, tmp_path, monkeypatch):
    monkeypatch.setattr(torch.backends.cudnn, "deterministic", True)
    monkeypatch.setattr(torch.backends.cudnn, "benchmark", False)
    run1 = cli.run_experiment(_cfg(seeds=(4,)), str(tmp_path / "a"))
    cfg2 = cli.load(os.path.join(run1, "config.txt"))
    assert cli.main(["train", os.path.join(run1, "config.txt"), "--out", str(tmp_path / "b")]) == 0
    run2 = [os.path.join(tmp_path / "b", d) for d in os.listdir(tmp_path / "b")][0]
    assert cli.dumps(cfg2) == open(os.path.join(run2, "config.txt")).read()
    keys = ("epoch", "mini_batch_index", "loss", "metric", "step_count", "seed")
    r1 = [{k: r[k] for k in keys} for r in _rows(os.path.join(run1, "metrics.csv"))]
    r2 = [{k: r[k] for k in keys} for r in _rows(os.path.join(run2, "metrics.csv"))]
    assert r1 == r2                                          # bit-identical (17 significant digits)


def test_segmentation_run_and_sweep(cuda, tmp_path):
    cfg = _cfg(model="unet", dataset=DatasetSpec("synthetic_segmentation", 24, (3, 32, 32), seed=2),
               loss="bce_dice", optimizer="adam", lr=1e-3, mini_batch_size=8, micro_batch_size=4, epochs=1,
               seeds=(0,))
    p = tmp_path / "seg.txt"
    p.write_text(cli.dumps(cfg))
    assert cli.main(["sweep", str(p), "--mini-batch", "8,12", "--out", str(tmp_path / "runs")]) == 0
    runs = sorted(os.path.join(tmp_path / "runs", d) for d in os.listdir(tmp_path / "runs"))
    assert len(runs) == 2
    text = cli.compare_report(runs)
    assert len(text.strip().splitlines()) == 3
    assert json.load(open(os.path.join(runs[0], "summary.json")))["metric"] == "iou"
