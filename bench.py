#!/usr/bin/env python
"""Benchmark: effective-batch samples/s of Micro-Batch Streaming on B200.

Default workload (BASELINE.json configs[1]): ResNet-50 @224 (102 classes,
synthetic Flower-102-shaped uint8 images), mini-batch 1024 streamed as
micro-batch 128, cross-entropy, SGD(0.01, 0.9, 5e-4), exact_weighted
normalisation. One STEP = one mini-batch: 8 micro-batch forward/backward
passes (bf16 autocast on cuDNN, fp32 master weights), 8 fused K1
normalise+accumulate passes, the loss/grad-norm finalize and one fused K3
optimizer step.

* ``value``  — inputs already resident in HBM (uint8), staged per micro-batch by K2.
* ``e2e``    — the same API fed from PINNED HOST memory: every step's micro-batches
  are copied H2D through the streamer inside the timed region, and every
  step's loss is read back (D2H).
* ``no_stream`` — plain torch training at batch = micro (128), data resident: the
  paper's "w/o MBS" run; ``stream_vs_no_stream`` = value / no_stream.
* ``roofline`` — K1 (the dominant MBS kernel) achieved algorithmic GB/s, timed
  live with CUDA events on its stream, vs the measured HBM copy peak.
* ``cpu_baseline`` — the CPU oracle port (float64 torch-CPU model + NumPy MBS
  arithmetic, the reference's algorithm) on a bounded sample, rank 0, N=1.

``--impl reference`` runs only that CPU reference path (all host threads).
Multi-GPU (torchrun): each rank streams its own mini-batch of 1024 (weak
scaling); the global plan's micro-batches are partitioned across ranks and
one NCCL all-reduce per mini-batch combines the accumulated gradients.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ---------------------------------------------------------------------------
# CPU reference arm (the oracle port: the reference's algorithm in float64)
# ---------------------------------------------------------------------------

def run_cpu_reference(w, steps: int, warmup: int, sample_n_b: int, sample_n_mu: int):
    """Time the float64 CPU oracle on a bounded sample of the workload; returns samples/s."""
    from oracle import mbs_oracle as O
    from oracle.hybrid import TorchGradFn
    from paper_2110_12484_b200.workloads import build_model, synthetic_data
    threads = os.cpu_count() or 1
    torch.set_num_threads(threads)
    torch.manual_seed(0)
    gf = TorchGradFn(build_model(w), w.loss_kind)
    st = O.OptState("sgd", 0.01, 0.9, 5e-4) if w.optimizer == "sgd" else O.OptState("adam", 0.01,
                                                                                       weight_decay=5e-4)
    acc = O.Accumulator({n: v.shape for n, v in gf.params().items()})
    x, y = synthetic_data(w, sample_n_b, seed=1)
    xn = x.double().numpy()
    yn = y.numpy()
    plan = O.plan_split(sample_n_b, sample_n_mu)
    params = gf.params()
    times = []
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        O.train_mini_batch(gf, params, xn, yn, plan, w.normalization, st, acc)
        dt = time.perf_counter() - t0
        if i >= warmup:
            times.append(dt)
    sps = sample_n_b * len(times) / sum(times)
    return sps, threads, float(np.mean(times))


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=16, help="samples per CPU-reference step")
    ap.add_argument("--model-ops", default="native", choices=["native", "torch"],
                    help="the model's BatchNorm(+ReLU/+skip add) and max-pool: K5/K6 sm_100a kernels or stock torch")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3

    from paper_2110_12484_b200.workloads import WORKLOADS
    w = WORKLOADS[args.config]
    ws, rank, local = _dist()

    if args.impl == "reference":
        if rank != 0:
            return
        n_mu = max(1, min(w.micro, args.cpu_sample // 2))
        sps, cores, step_s = run_cpu_reference(w, args.steps, max(1, min(args.warmup, 1)), args.cpu_sample, n_mu)
        sample = (f"{w.model} {w.sample_shape}: mini-batch {args.cpu_sample} streamed as micro {n_mu}, float64 "
                  f"torch-CPU model + NumPy MBS arithmetic (oracle port of engine.py/optim.py)")
        line = {"impl": "reference", "metric": "effective-batch samples/sec", "value": sps, "unit": "samples/s",
                "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": step_s * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic",
                "config": {"workload": w.name, "mini": w.mini, "micro": w.micro, "parallelism": "cpu"},
                "cpu_baseline": {"value": sps, "unit": "samples/s", "cores": cores, "kind": "port",
                                 "sample": sample},
                "e2e": {"value": sps, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    import paper_2110_12484_b200 as mbs
    from paper_2110_12484_b200.prof import TIMER
    from paper_2110_12484_b200.streamer import Staging
    from paper_2110_12484_b200.workloads import build_model, synthetic_data

    ndev = torch.cuda.device_count()
    dev = torch.device("cuda", local % max(1, ndev))
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(dev)
        backend = os.environ.get("MBS_DP_BACKEND", "nccl")   # gloo only for smoke runs of >1 rank per GPU
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    torch.cuda.set_device(dev)
    torch.backends.cudnn.benchmark = os.environ.get("MBS_BENCH_DETERMINISTIC", "0") != "1"
    torch.backends.cudnn.deterministic = not torch.backends.cudnn.benchmark   # reproducibility checks only
    torch.manual_seed(1234 + rank)

    model = build_model(w, ops=args.model_ops).to(dev).to(memory_format=torch.channels_last)
    params = mbs.ParameterSet(model, shadow=torch.bfloat16)   # bf16 shadow weights: K3 refreshes them, K1 reads bf16 grads
    staging = Staging(dtype=torch.bfloat16, channels_last=True)
    autocast = torch.bfloat16
    n_b, n_mu = w.mini, w.micro
    autosize = None
    if n_mu == 0:
        # config 5: micro-batch auto-sized to free HBM (memory.py:88-101 rule on measured bytes)
        from paper_2110_12484_b200 import memory
        from paper_2110_12484_b200.streamer import stage_rows

        def make_batch(k):
            xb, yb = synthetic_data(w, k, seed=99, device=dev)
            return stage_rows(xb, xb.dtype, tuple(xb.shape[1:]), None, 0, k, staging, dev), yb
        # probes at 4 / 8 samples and a 0.88 margin: at HBM-filling sizes the allocator's fragmentation
        # and the size-dependent cuDNN workspaces are not covered by the 0.92 default
        budget = memory.measure_budget(model, make_batch, w.loss_kind, optimizer_kind=w.optimizer,
                                       autocast_dtype=autocast, probe=(4, 8), safety=0.88)
        n_mu = memory.fit_micro_batch(budget)
        n_b = max(w.mini, 4 * n_mu)          # a mini-batch that cannot fit HBM without streaming
        autosize = {"capacity_bytes": budget.capacity_bytes, "resident_bytes": budget.resident_bytes,
                    "data_bytes_per_sample": budget.data_bytes_per_sample, "micro": n_mu, "mini": n_b}
        torch.cuda.empty_cache()
    plan = mbs.plan_split(n_b, n_mu)

    # The timed region is ONE epoch call over `steps` shuffled mini-batches: engine.train_epoch
    # (engine.py:276) at N=1, DataParallelMBS.train_epoch (each rank streams its own shard, one
    # all-reduce per global mini-batch) at N>1. Device rows are gathered by K2, host rows by the native
    # gather pool + H2D. Every mini-batch is >= 154 MB of uint8, so inputs exceed the 126 MB L2.
    warm_mini = min(n_b, 1024)           # warm-up mini-batches (C4's 300k-sample mini-batch is 66 s of compute)
    if ws > 1:
        warm_mini = n_b                  # the global plan needs every rank's local mini-batch to be whole micros
    n_data = max(args.steps * n_b, args.warmup * warm_mini)
    x_host, y_host = synthetic_data(w, n_data, seed=rank, pinned=True)
    x_dev, y_dev = x_host.to(dev), y_host.to(dev)

    dp = None
    if ws > 1:
        from paper_2110_12484_b200.dp import DataParallelMBS
        dp = DataParallelMBS(params, transport=os.environ.get("MBS_DP_TRANSPORT", "nccl"))

    def make_opt():
        return mbs.sgd_state(0.01, 0.9, 5e-4) if w.optimizer == "sgd" else mbs.adam_state(0.01, 5e-4)

    acc = mbs.GradientAccumulator(params)
    st = make_opt()
    streamer = mbs.make_streamer(x_host, y_host, n_mu, n_slots=3)
    cs = torch.cuda.current_stream(dev)

    def epoch(host: bool, n_steps: int, epoch_index: int, mini: int = n_b):
        xs, ys = (x_host, y_host) if host else (x_dev, y_dev)
        if dp is not None:
            res = dp.train_epoch(model, xs[:n_steps * mini], ys[:n_steps * mini], mini_batch_size=mini,
                                 micro_batch_size=n_mu, normalization=w.normalization, loss_kind=w.loss_kind,
                                 optimizer_state=st, seed=rank, epoch_index=epoch_index, accumulator=acc,
                                 staging=staging, autocast_dtype=autocast, streamer=streamer if host else None,
                                 prefetch=True)
            return [r.loss for r in res]
        es = mbs.train_epoch(model, params, xs[:n_steps * mini], ys[:n_steps * mini], mini_batch_size=mini,
                             micro_batch_size=n_mu, normalization=w.normalization, loss_kind=w.loss_kind,
                             optimizer_state=st, seed=rank, epoch_index=epoch_index, shuffle=True, prefetch=True,
                             accumulator=acc, staging=staging, autocast_dtype=autocast,
                             streamer=streamer if host else None)
        return es.mini_losses      # every mini-batch's loss, read back (D2H) inside the call

    def barrier():
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize(dev)

    def timed(host: bool, steps: int, warmup: int, k1_timer: bool):
        epoch(host, warmup, 1000 + int(host), warm_mini)
        barrier()
        TIMER.reset()
        TIMER.enabled = k1_timer
        if host:
            streamer.timings(flush=True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(cs)
        losses = epoch(host, steps, int(host))
        e1.record(cs)
        barrier()
        TIMER.enabled = False
        ms = e0.elapsed_time(e1)
        if ws > 1:
            t = torch.tensor([ms], device=dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            ms = float(t.item())
        return ms, losses

    # --- value: inputs resident in HBM (no per-kernel instrumentation inside the timed region) ---
    with ClockSampler(dev.index) as clocks:
        ms_dev, _ = timed(False, args.steps, args.warmup, k1_timer=False)
    launches_value = TIMER.launches
    # Per-kernel bandwidths (K1 accumulate, K2, K3, K4 and the model's K5 BatchNorm): two more
    # HBM-resident mini-batches, eager, with CUDA events around every launch on its stream. Kept out of
    # `value` so the events and the eager launches do not perturb the headline number.
    from paper_2110_12484_b200 import engine as _eng
    from paper_2110_12484_b200 import graphs as _graphs
    _graphs.clear()     # free the captured pools for the eager pass (re-captured in the e2e run's warm-up)
    graphs_on, _eng.CUDA_GRAPHS = _eng.CUDA_GRAPHS, False
    TIMER.reset()
    TIMER.enabled = True
    TIMER.k5 = args.model_ops == "native"
    epoch(False, 2, 2000, warm_mini)
    TIMER.enabled = TIMER.k5 = False
    _eng.CUDA_GRAPHS = graphs_on
    allstats = TIMER.summary()
    kstats = {k: v for k, v in allstats.items() if not k.startswith("k5_")}
    k5stats = {k: v for k, v in allstats.items() if k.startswith("k5_")}
    samples_total = n_b * args.steps * ws
    value = samples_total / (ms_dev / 1e3)

    # --- e2e: host-pinned inputs through the streamer ---
    ms_host, losses = timed(True, args.steps, args.warmup, k1_timer=False)
    launches_e2e = TIMER.launches
    e2e = samples_total / (ms_host / 1e3)
    tim = streamer.timings(flush=True)
    copy_ms = sum(t[1] for t in tim)
    blocked_ms = sum(t[2] for t in tim)
    h2d_bytes = sum(t[3] for t in tim) / max(1, args.steps)
    overlap = 100.0 * (1.0 - blocked_ms / copy_ms) if copy_ms > 0 else None
    h2d_gbs = (sum(t[3] for t in tim) / (copy_ms / 1e3) / 1e9) if copy_ms > 0 else None
    streamer.close()

    # --- no-stream baseline: plain torch training at batch = micro, data resident ---
    _graphs.clear()     # the MBS step's graph pools are not needed by the baselines
    nos = nos_torch = None
    for ops_ in (args.model_ops, "torch") if args.model_ops != "torch" else (args.model_ops,):
        b = n_mu        # halve the batch until the model fits (the stock model holds more per sample)
        r = None
        while b >= 1 and r is None:
            try:
                r = no_stream_baseline(w, dev, b, args.steps, args.warmup, ws, ops=ops_)
            except torch.OutOfMemoryError:
                b //= 2
            torch.cuda.empty_cache()
        if ops_ == args.model_ops:
            nos = r
        else:
            nos_torch = r

    # the reference's overhead report (streaming.py:130-149) on MEASURED schedules: the MBS step as
    # run (copy per micro from the streamer's events, compute per micro from the timed step) vs the
    # no-stream run processing the same samples
    from paper_2110_12484_b200 import streaming as SS
    k3 = next((v for k, v in kstats.items() if k.startswith("k3_")), {"avg_ms": 0.0})
    per_micro_ms = (ms_host / args.steps - k3["avg_ms"]) / plan.n_s_mu
    copies = [t[1] for t in tim[-plan.n_s_mu:]] if tim else [0.0] * plan.n_s_mu
    mbs_sched = SS.measured_schedule(copies, [per_micro_ms] * plan.n_s_mu, k3["avg_ms"], overlap=True)
    base_ms = n_b / nos["value"] * ws * 1e3 if nos else None
    base_sched = SS.measured_schedule([0.0], [base_ms], 0.0, overlap=False) if base_ms else None
    rep = SS.overhead_report(mbs_sched, base_sched)
    overhead = {"mbs_makespan_ms": rep.mbs_makespan * 1e3,
                "no_stream_makespan_ms": rep.baseline_makespan * 1e3 if rep.baseline_makespan else None,
                "overhead_pct": rep.overhead_pct,
                "how": "streaming.overhead_report on measured per-micro copy/compute times (e2e run) vs the "
                       "no-stream run's time for the same samples"}

    k1 = kstats.get("k1_accumulate", {})
    peak, peak_kind = _peaks()
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_k1_traffic.json")) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")
    except Exception:
        pass
    roofline = {"kernel": "k1_accumulate (mbs_accum_add)", "bound": "hbm", "achieved": k1.get("gbs"),
                "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                "frac": (k1.get("gbs") or 0.0) / peak, "traffic": traffic,
                "algorithmic_bytes_per_launch": k1.get("bytes_per_launch"), "avg_launch_us": (k1.get("avg_ms") or 0) * 1e3,
                "launches_timed": k1.get("launches"),
                "bytes_rule": "12 B/param (read g, read acc, write acc); 8 B/param on the first micro-batch "
                              "(acc = s*g); P = %d" % params.layout.n_params,
                "how": "CUDA events around every K1 launch of two extra HBM-resident mini-batches (eager), "
                       "outside the timed region",
                "note": "K1 is the kernel the north star names (accumulate); the dominant kernel of the step by "
                        "time is the model's K5 BatchNorm, reported in roofline_k5",
                "other_kernels": {k: {"gbs": v["gbs"], "avg_us": v["avg_ms"] * 1e3, "launches": v["launches"]}
                                  for k, v in kstats.items() if k != "k1_accumulate"}}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            _pk = json.load(f)
        tf_peak, tf_kind = float(_pk["bf16_tflops_sustained"]), "measured sustained bf16"
    except Exception:
        tf_peak, tf_kind = 1407.5, "fallback (SURVEY §8d sustained bf16)"
    from paper_2110_12484_b200.workloads import gflop_per_sample
    gfs = gflop_per_sample(w, dev)
    model_flops = {"bound": "tensor", "gflop_per_sample": gfs, "unit": "TFLOP/s",
                   "achieved": value * gfs / 1e3, "achieved_e2e": e2e * gfs / 1e3, "peak": tf_peak,
                   "peak_kind": tf_kind, "frac": value / ws * gfs / 1e3 / tf_peak,
                   "frac_e2e": e2e / ws * gfs / 1e3 / tf_peak, "peak_is": "per GPU (frac uses value / n_gpus)",
                   "how": "end-to-end samples/s x algorithmic fwd+bwd FLOP per sample (FlopCounterMode: the "
                          "model's convolutions/matmuls), against the bf16 dense peak"}
    roofline_k5 = None
    if k5stats:
        kb = sum(v["bytes_per_launch"] * v["launches"] for v in k5stats.values())
        kt = sum(v["total_ms"] for v in k5stats.values())
        roofline_k5 = {"kernel": "k5 micro-batch BatchNorm (+ReLU/+residual), forward and backward",
                       "bound": "hbm", "achieved": kb / (kt / 1e3) / 1e9, "peak": peak, "peak_kind": peak_kind,
                       "unit": "GB/s", "frac": kb / (kt / 1e3) / 1e9 / peak,
                       "ms_per_mini_batch": kt, "calls": {k: v["launches"] for k, v in k5stats.items()},
                       "per_call": {k: {"gbs": v["gbs"], "avg_us": v["avg_ms"] * 1e3} for k, v in k5stats.items()},
                       "bytes_rule": "per call over E activation elements of s bytes: forward 3*E*s (+E*s "
                                     "residual), backward 5*E*s (+2*E*s residual: the two-pass minimum); CUDA events around each "
                                     "3-kernel call, so small layers include launch gaps"}

    line = {"metric": "effective-batch samples/sec", "value": value, "unit": "samples/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_dev / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (uint8 images, random labels; random-init weights)",
            "config": {"workload": w.name, "model": w.model, "mini_batch_per_gpu": n_b, "micro_batch": n_mu,
                       "n_micro": plan.n_s_mu, "global_batch": n_b * ws, "parallelism": f"dp{ws}",
                       "normalization": w.normalization, "optimizer": w.optimizer,
                       "model_precision": "bf16 compute (autocast) on cuDNN/cuBLAS reading bf16 shadow weights that "
                                          "K3 writes; fp32 master weights, fp32 MBS accumulation",
                       "model_ops": ("BatchNorm(+ReLU/+skip add) on K5, max-pool (+U-Net skip join) on K6, stem "
                                     "conv as K7 im2col + GEMM (bn.py, pool.py, stem.py), micro-batch statistics; "
                                     "micro step replayed from a CUDA graph" if args.model_ops == "native"
                                     else "stock torch BatchNorm / max-pool / stem conv"),
                       "input": "uint8 NCHW staged to bf16 NHWC by K2",
                       "l2": ("inputs > L2: every mini-batch is %.0f MB of uint8" % (x_dev[:n_b].numel() / 1e6)) +
                             ", none reused within the timed region",
                       "api": ("engine.train_epoch" if ws == 1 else "dp.DataParallelMBS.train_epoch (per-rank "
                               "shards, one all-reduce per global mini-batch, transport=%s)" % dp.transport) +
                              " over `steps` shuffled mini-batches",
                       "autosize": autosize},
            "e2e": {"value": e2e, "unit": "samples/s", "h2d_bytes_per_step": int(h2d_bytes),
                    "d2h_bytes_per_step": 8 * (4 + 2 * plan.n_s_mu), "ms_per_step": ms_host / args.steps},
            "h2d_overlap_pct": overlap, "h2d_gbs": h2d_gbs, "accum_gbs": k1.get("gbs"),
            "no_stream": nos, "stream_vs_no_stream": value / nos["value"] if nos else None, "overhead": overhead,
            "no_stream_torch_ops": nos_torch, "roofline_k5": roofline_k5, "model_flops": model_flops,
            "e2e_vs_no_stream": e2e / nos["value"] if nos else None,
            "roofline": roofline, "gpu_launches": launches_value, "gpu_launches_e2e": launches_e2e,
            "clocks": clocks.summary(), "final_loss": losses[-1] if losses else None}

    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu_n_b = args.cpu_sample
        cpu_mu = max(1, cpu_n_b // 2)
        sps, cores, step_s = run_cpu_reference(w, 1, 1, cpu_n_b, cpu_mu)
        line["cpu_baseline"] = {"value": sps, "unit": "samples/s", "cores": cores, "kind": "port",
                                "sample": f"1 mini-batch of {cpu_n_b} as micro {cpu_mu}, {w.model} float64 "
                                          f"torch-CPU + NumPy MBS oracle, {step_s:.1f} s/step"}
    if rank == 0:
        print(json.dumps(line))
    if ws > 1:
        torch.distributed.destroy_process_group()


def no_stream_baseline(w, dev, batch, steps, warmup, ws, ops="torch", graph=True):
    """The paper's 'w/o MBS' run: plain torch training, batch = micro-batch, data resident in HBM.

    ``ops`` selects the same model definition as the MBS run (native K5/K6/K7 or stock torch ops).
    ``graph``: the whole training step (fwd + bwd + fused optimizer step) is replayed from one CUDA
    graph, like the MBS micro step — eager, this loop is host-bound on B200 and its number then
    tracks the host CPU rather than the GPU. Falls back to eager if capture fails."""
    from paper_2110_12484_b200.losses import compute_loss
    from paper_2110_12484_b200.workloads import build_model, synthetic_data
    torch.manual_seed(0)
    model = build_model(w, ops=ops).to(dev).to(memory_format=torch.channels_last)
    if w.optimizer == "sgd":
        opt = torch.optim.SGD(model.parameters(), lr=0.01, momentum=0.9, weight_decay=5e-4, fused=True)
    else:
        opt = torch.optim.Adam(model.parameters(), lr=0.01, weight_decay=5e-4, fused=True, capturable=graph)
    x, y = synthetic_data(w, 2 * batch, seed=7, device=dev)
    xs = [x[i * batch:(i + 1) * batch].to(torch.bfloat16).contiguous(memory_format=torch.channels_last)
          for i in range(2)]
    ys = [y[i * batch:(i + 1) * batch] for i in range(2)]
    sx, sy = xs[0].clone(), ys[0].clone()

    def step(cache=True):
        with torch.autocast("cuda", dtype=torch.bfloat16, cache_enabled=cache):
            loss = compute_loss(w.loss_kind, model(sx), sy)
        loss.backward()
        opt.step()
        return loss

    def one(i):
        sx.copy_(xs[i % 2])
        sy.copy_(ys[i % 2])
        step()
        opt.zero_grad(set_to_none=True)

    for i in range(warmup):
        one(i)
    torch.cuda.synchronize(dev)
    how = "torch fwd/bwd + fused torch.optim step per batch, bf16 autocast, data in HBM"
    if graph:
        try:
            side = torch.cuda.Stream(dev)
            side.wait_stream(torch.cuda.current_stream(dev))
            with torch.cuda.stream(side):
                for i in range(2):
                    one(i)
            torch.cuda.current_stream(dev).wait_stream(side)
            torch.cuda.synchronize(dev)
            opt.zero_grad(set_to_none=True)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                step(cache=False)

            def one(i):                                  # noqa: F811 - the graphed step
                sx.copy_(xs[i % 2])
                sy.copy_(ys[i % 2])
                g.replay()
            for i in range(2):
                one(i)
            how = "CUDA graph of torch fwd/bwd + fused torch.optim step per batch, bf16 autocast, data in HBM"
        except Exception as e:                           # noqa: BLE001
            print(f"no-stream baseline: graph capture failed ({type(e).__name__}: {e}); eager", file=sys.stderr)
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = steps * max(1, w.mini // batch)
    e0.record()
    for i in range(n):
        one(i)
    e1.record()
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1)
    del model, opt
    return {"value": batch * n * ws / (ms / 1e3), "unit": "samples/s", "batch": batch,
            "steps": n, "model_ops": ops, "how": how}


if __name__ == "__main__":
    main()
