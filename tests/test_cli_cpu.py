"""SPEC data-cli on the CPU: config format, datasets, IDX loader, CSV, reports, exit codes."""
import csv
import dataclasses
import json
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

import paper_2110_12484_b200 as mbs
from paper_2110_12484_b200 import cli, datasets
from paper_2110_12484_b200.datasets import DatasetSpec

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_config_round_trips_bit_exactly():
    cfg = cli.ExperimentConfig(lr=0.1 + 0.2, weight_decay=1e-4 / 3, seeds=(1, 2, 3), micro_batch_size="auto",
                               dataset=DatasetSpec("synthetic_segmentation", 40, (3, 16, 16), mask_shape=(1, 16, 16),
                                                   seed=2 ** 64 - 1, separation=1 / 7),
                               loss="bce_dice", optimizer="adam", model="unet")
    text = cli.dumps(cfg)
    back = cli.loads(text)
    assert back == cfg
    assert back.lr == 0.1 + 0.2 and back.dataset.separation == 1 / 7       # floats bit-exact
    assert cli.dumps(back) == text
    assert cli.loads(cli.dumps(dataclasses.replace(cfg, micro_batch_size=None))).micro_batch_size is None


@pytest.mark.parametrize("text,msg", [
    ("dataset.kind = synthetic_classification\nbogus.key = 1\n", "unknown key"),
    ("dataset.kind = synthetic_classification\nmbs.mini_batch_size = x\n", "cannot parse"),
    ("mbs.mini_batch_size = 4\n", "dataset.kind is required"),
    ("dataset.kind = synthetic_classification\ndataset.kind = synthetic_classification\n", "duplicate"),
    ("dataset.kind = nope\n", "dataset.kind"),
    ("dataset.kind = synthetic_classification\ndataset.n_samples = 8\ndataset.input_shape = 4\n"
     "dataset.n_classes = 1\n", "n_classes"),
    ("dataset.kind = synthetic_classification\ndataset.n_samples = 8\ndataset.input_shape = 4\n"
     "dataset.n_classes = 2\nmbs.micro_batch_size = 0\n", "micro_batch_size"),
    ("dataset.kind = synthetic_classification\ndataset.n_samples = 0\ndataset.input_shape = 4\n"
     "dataset.n_classes = 2\n", "degenerate"),
    ("dataset.kind = synthetic_classification\nno equals sign\n", "key = value"),
])
def test_config_errors(text, msg):
    with pytest.raises(mbs.ConfigError, match=msg):
        cli.loads(text)


def test_classification_dataset_rules():
    spec = DatasetSpec("synthetic_classification", 33, (4,), n_classes=3, seed=5)
    x1, y1 = datasets.make_dataset(spec)
    x2, y2 = datasets.make_dataset(spec)
    assert x1[0].tobytes() == x2[0].tobytes() and np.array_equal(y1, y2)          # pure function of the spec
    assert sorted(np.bincount(y1).tolist()) == [11, 11, 11]                          # balanced
    assert not np.array_equal(datasets.make_dataset(dataclasses.replace(spec, seed=6))[0], x1)
    with pytest.raises(mbs.ConfigError):
        datasets.make_dataset(DatasetSpec("synthetic_classification", 0, (4,), n_classes=3))


def test_high_separation_is_linearly_separable():
    """separation set high -> a linear model reaches >= 99 % train accuracy in <= 20 epochs."""
    x, y = datasets.make_dataset(DatasetSpec("synthetic_classification", 300, (16,), n_classes=4, seed=1,
                                             separation=6.0))
    xt, yt = torch.from_numpy(x).double(), torch.from_numpy(y)
    lin = torch.nn.Linear(16, 4).double()
    opt = torch.optim.SGD(lin.parameters(), lr=0.1)
    for _ in range(20):
        opt.zero_grad()
        torch.nn.functional.cross_entropy(lin(xt), yt).backward()
        opt.step()
    assert mbs.accuracy(lin(xt).detach(), yt) >= 0.99


def test_segmentation_dataset_rules():
    spec = DatasetSpec("synthetic_segmentation", 12, (3, 20, 24), seed=3)
    x, m = datasets.make_dataset(spec)
    assert x.shape == (12, 3, 20, 24) and m.shape == (12, 1, 20, 24) and m.dtype == np.uint8
    assert set(np.unique(m)) <= {0, 1} and 0 < m.mean() < 1
    # masks are the exact ground truth of what was painted; the perfect-oracle predictor scores IoU 1.0
    assert mbs.iou(torch.from_numpy(m).float(), torch.from_numpy(m)) == 1.0
    assert np.array_equal((x.mean(axis=1, keepdims=True) > 0.5).astype(np.uint8), m)
    e = datasets.make_dataset(dataclasses.replace(spec, extra={"coverage": "empty"}))[1]
    f = datasets.make_dataset(dataclasses.replace(spec, extra={"coverage": "full"}))[1]
    assert not e.any() and f.all()
    with pytest.raises(mbs.ConfigError, match="spatial"):
        datasets.make_dataset(DatasetSpec("synthetic_segmentation", 4, (3, 8, 8), mask_shape=(1, 8, 9)))


def test_idx_loader(tmp_path):
    imgs = np.arange(10 * 4 * 3, dtype=np.uint8).reshape(10, 4, 3)
    labs = np.arange(10, dtype=np.uint8) % 7
    pi, pl = str(tmp_path / "i.idx"), str(tmp_path / "l.idx")
    datasets.write_idx(pi, imgs)
    datasets.write_idx(pl, labs)
    x, y = datasets.load_idx_images(pi, pl)
    assert x.shape == (10, 1, 4, 3) and x.dtype == np.float32 and np.allclose(x[:, 0] * 255.0, imgs)
    assert y.tolist() == labs.tolist()
    bad = tmp_path / "bad.idx"
    bad.write_bytes(b"\x00\x00\x08\x02" + (4).to_bytes(4, "big") * 2 + bytes(16))
    with pytest.raises(mbs.IdxFormatError, match="bad magic 0x00000802 at offset 0"):
        datasets.load_idx_images(str(bad))
    trunc = tmp_path / "t.idx"
    trunc.write_bytes(open(pi, "rb").read()[:-5])
    with pytest.raises(mbs.IdxFormatError, match="expected 136 bytes, got 131"):
        datasets.load_idx_images(str(trunc))
    datasets.write_idx(pl, labs[:9])
    with pytest.raises(mbs.IdxFormatError, match="9 labels for 10 images"):
        datasets.load_idx_images(pi, pl)


def test_csv_17_significant_digits(tmp_path):
    vals = [0.1 + 0.2, 1 / 3, 2.0 ** -40, 123456789.123456789, float("nan")]
    rows = [{"epoch": 0, "mini_batch_index": i, "loss": v, "metric": -v, "step_count": i + 1} for i, v in
            enumerate(vals)]
    p = str(tmp_path / "m.csv")
    cli.write_csv(p, rows)
    back = list(csv.DictReader(open(p)))
    assert list(back[0].keys()) == list(cli.CSV_COLUMNS)
    for r, v in zip(back, vals):
        assert (float(r["loss"]) == v) or (np.isnan(v) and r["loss"] == "nan")


def _fake_run(d, mini, micro, metric, base):
    os.makedirs(d)
    with open(os.path.join(d, "summary.json"), "w") as f:
        json.dump({"metric": metric, "mini_batch_size": mini, "micro_batch_size": micro,
                   "mbs": {"max_metric_mean": 0.9, "wall_seconds_mean": 2.0},
                   "baseline": base if base == "Failed" else {"max_metric_mean": 0.91, "wall_seconds_mean": 1.5}}, f)
    return d


def test_compare_report(tmp_path):
    a = _fake_run(str(tmp_path / "a"), 256, 16, "iou", "Failed")
    b = _fake_run(str(tmp_path / "b"), 16, 8, "iou", "ok")
    text = cli.compare_report([a, b], str(tmp_path / "t.csv"))
    lines = text.strip().splitlines()
    assert len(lines) == 3 and lines[1].split()[0] == "16" and "Failed" in lines[2]
    rows = list(csv.DictReader(open(tmp_path / "t.csv")))
    assert rows[1]["metric_without_mbs"] == "Failed" and rows[1]["time_without_s"] == "Failed"
    assert float(rows[0]["metric_without_mbs"]) == 0.91
    c = _fake_run(str(tmp_path / "c"), 32, 8, "accuracy", "ok")
    with pytest.raises(mbs.ConfigError, match="incompatible"):
        cli.compare_report([a, c])
    # two identical runs: identical rows (all deltas 0)
    d = _fake_run(str(tmp_path / "d"), 16, 8, "iou", "ok")
    assert cli.compare_report([b, d]).splitlines()[1] == cli.compare_report([b, d]).splitlines()[2]


def test_cli_exit_codes(tmp_path):
    bad = tmp_path / "bad.txt"
    bad.write_text("dataset.kind = synthetic_classification\nnot.a.key = 3\n")
    run = subprocess.run([sys.executable, "-m", "paper_2110_12484_b200.cli", "train", str(bad)], cwd=ROOT,
                         capture_output=True, text=True, timeout=300)
    assert run.returncode == 2 and "unknown key" in run.stderr
    run = subprocess.run([sys.executable, "-m", "paper_2110_12484_b200.cli", "compare", str(tmp_path / "none")],
                         cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert run.returncode == 2
    assert cli.main(["compare", _fake_run(str(tmp_path / "r"), 8, 4, "accuracy", "Failed")]) == 0
