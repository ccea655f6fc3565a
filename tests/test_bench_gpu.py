"""bench.py's GPU arm emits the driver's JSON contract (a short C1 run on cuda:0)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_gpu_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "c1", "--steps", "2",
                          "--warmup", "3", "--no-cpu-baseline", "--no-fp32-context"], capture_output=True, text=True,
                         timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "setup", "e2e", "roofline", "gpu_launches", "clocks",
              "h2d_overlap_pct", "accum_gbs", "no_stream"):
        assert k in line, k
    assert line["n_gpus"] == 1 and line["steps"] == 2 and line["warmup"] == 3 and line["value"] > 0
    assert line["config"]["workload"].startswith("resnet18") and line["config"]["mini_batch_per_gpu"] == 64
    assert "model" not in line["config"]                     # the config names the workload only
    e2e = line["e2e"]
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] >= 64 * 3 * 32 * 32 and e2e["d2h_bytes_per_step"] > 0
    r = line["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0.0 < r["frac"] < 1.5 and r["peak"] > 0
    assert r["frac"] == pytest.approx(r["achieved"] / r["peak"])
    assert line["gpu_launches"] > 0
    # the reference arm's config is the same workload object
    ref = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c1",
                          "--steps", "1", "--warmup", "3"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert ref.returncode == 0, ref.stderr[-2000:]
    rline = json.loads(ref.stdout.strip().splitlines()[-1])
    assert rline["config"] == line["config"]
