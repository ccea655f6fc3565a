#!/usr/bin/env python
"""Benchmark: effective-batch samples/s of Micro-Batch Streaming on B200, batch > HBM.

Default workload (BASELINE.json ``configs[3]``, the config the metric "(batch > HBM)" is quoted on):
ResNet-50 @224 (102 classes, synthetic Flower-102-shaped uint8 images, random labels, random init),
ONE mini-batch of 300,032 samples per GPU streamed as 2,344 micro-batches of 128 — 45.2 GB
host-resident as uint8, 180.6 GB as the reference's float32 arrays (> the 180 GB of HBM) — cross
entropy, SGD(0.01, 0.9, 5e-4), exact_weighted normalisation. The host dataset is exactly one
mini-batch; every step is one epoch over it (reshuffled per epoch by ``epoch_index``, engine.py:300).
One STEP = one mini-batch: 2,344 micro forward/backward passes (bf16 autocast on cuDNN, bf16 shadow
weights), 2,344 fused K1 normalise+accumulate passes, the loss/grad-norm finalize and one fused K3
optimizer step. ``--config c2`` is the fits-in-HBM 1024/128 case.

* ``value``   — inputs resident in HBM (uint8), staged per micro-batch by K2.
* ``e2e``     — the same API fed from PINNED HOST memory: every micro-batch is copied H2D through the
  streamer inside the timed region and every mini-batch's loss is read back (D2H).
* ``no_stream`` — plain torch training at batch = micro, data resident (the paper's "w/o MBS" run);
  ``e2e_vs_no_stream`` is the north-star ratio; ``no_stream_weights_at_init`` is the same run with the
  weights held at init (lr 1e-9), the matched-power-state baseline (the weight trajectory, not MBS,
  sets the power-capped clock on synthetic data: profiles/r02_power_state.md).
* ``overhead`` — the reference's overhead report (streaming.py:130-149) on the MEASURED schedule of
  the timed e2e run (``streaming.ScheduleTracer``: CUDA events per micro-batch on the copy and
  compute streams), and the H2D overlap fraction from the same events.
* ``roofline`` — K1 (the accumulate kernel the north star names) achieved algorithmic GB/s, timed live
  with CUDA events on its stream, vs the measured HBM copy peak.
* ``precision_fp32`` — the same MBS stack in fp32 (TF32 off), the precision every oracle parity test
  also pins; context only.
* ``cpu_baseline`` — the CPU oracle port (float64 torch-CPU model + NumPy MBS arithmetic, the
  reference's algorithm) on a bounded sample, rank 0, N=1.

``--impl reference`` runs only that CPU reference path (all host threads) on the same workload config.
Multi-GPU (torchrun): each rank streams its own mini-batch (weak scaling); the global plan's
micro-batches are partitioned across ranks and one NCCL all-reduce per mini-batch combines the
accumulated gradients.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "effective-batch samples/sec"
E2E_BUDGET_S = 1200.0           # longest e2e timed region (see run_gpu)
HOST_DATA_CAP = 8 << 30          # host bytes per rank beyond which the dataset is ONE mini-batch
CPU_SAMPLE = (16, 8)             # the CPU reference's bounded sample: mini 16 streamed as micro 8


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
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
                 "--format=csv,noheader,nounits", "-lms", "500"],
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
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


class SharedHostPool:
    """The image pool of a multi-rank run, ONE copy per node: local rank 0 writes it into a shared file
    (``/dev/shm``, else ``/tmp``), every local rank maps it and page-locks its mapping (cudaHostRegister), and
    each rank streams it in its own rank-keyed order (dp.DataParallelMBS.train_epoch). C4 at 8 ranks would
    otherwise pin 8 x 45.2 GB = 361 GB of uint8 on a host with ~200 GB of RAM."""

    def __init__(self, w, n: int, local_rank: int, barrier):
        from paper_2110_12484_b200.workloads import synthetic_data
        self.shape = (n,) + tuple(w.sample_shape)
        self.nbytes = int(np.prod(self.shape))
        base = "/dev/shm" if os.path.isdir("/dev/shm") else "/tmp"
        st = os.statvfs(base)
        if st.f_bavail * st.f_frsize < 1.05 * self.nbytes:
            base = "/tmp"
        self.path = os.path.join(base, f"mbs_bench_pool_{w.name.replace('/', '_')}_{n}_{os.getppid()}.u8")
        self.owner = local_rank == 0
        if self.owner:
            x = torch.from_file(self.path, shared=True, size=self.nbytes, dtype=torch.uint8).view(self.shape)
            pool, _ = synthetic_data(w, min(n, 509), seed=0)
            for i in range(0, n, pool.shape[0]):
                k = min(pool.shape[0], n - i)
                x[i:i + k].copy_(pool[:k])
            del x
        barrier()
        self.x = torch.from_file(self.path, shared=True, size=self.nbytes, dtype=torch.uint8).view(self.shape)
        torch.cuda.cudart().cudaHostRegister(self.x.data_ptr(), self.nbytes, 0)
        self.where = base

    def close(self, barrier):
        try:
            torch.cuda.cudart().cudaHostUnregister(self.x.data_ptr())
        except Exception:
            pass
        del self.x
        barrier()
        if self.owner and os.path.exists(self.path):
            os.unlink(self.path)


def workload_config(w, n_b: int, n_mu: int, ws: int) -> dict:
    """The ``config`` object of BOTH arms' JSON lines: the workload only (identical in the two arms, so the
    driver can compare them); how each arm ran it is in the line's ``setup``."""
    from paper_2110_12484_b200 import engine
    plan = engine.plan_split(n_b, n_mu)
    row = int(np.prod(w.sample_shape))
    return {"workload": w.name, "input": "x".join(map(str, w.sample_shape)),
            "mini_batch_per_gpu": n_b, "micro_batch": n_mu, "n_micro": plan.n_s_mu,
            "micro_sizes_head_tail": [plan.sizes[0], plan.sizes[-1]], "global_batch": n_b * ws,
            "parallelism": f"dp{ws}", "normalization": w.normalization, "optimizer": w.optimizer,
            "loss": w.loss_kind,
            "mini_batch_bytes": {"uint8": n_b * row, "fp32_as_reference_holds_it": 4 * n_b * row},
            "l2": "inputs > L2: every mini-batch is %.1f GB of uint8, none reused within a step" % (n_b * row / 1e9)
            if n_b * row > (126 << 20) else "mini-batch fits L2 (no flush): CPU-sized config"}


# ---------------------------------------------------------------------------
# CPU reference arm (the oracle port: the reference's algorithm in float64)
# ---------------------------------------------------------------------------

def run_cpu_reference(w, steps: int, warmup: int, sample_n_b: int, sample_n_mu: int):
    """Time the float64 CPU oracle on a bounded sample of the workload; returns (samples/s, cores, s/step)."""
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
    yn = y.numpy().astype(np.float64) if w.target == "mask" else y.numpy()
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


def run_cpu_accumulate(shapes: dict, reps: int = 3):
    """SURVEY §8(d) CPU baseline (3): the reference's GradientAccumulator.add (engine.py:117-128, restated
    in the oracle: fp64 per-parameter ``sums[name] += g``) over one gradient of the workload's parameter
    shapes; algorithmic bytes 24 B/param (read g, read sum, write sum, fp64). Returns (GB/s, s/add)."""
    from oracle import mbs_oracle as O
    acc = O.Accumulator(shapes)
    rng = np.random.default_rng(0)
    g = {n: rng.standard_normal(s) for n, s in shapes.items()}
    n_params = sum(int(np.prod(s)) for s in shapes.values())
    acc.begin(reps + 1)
    acc.add(g)                                                 # warm-up (page faults)
    t0 = time.perf_counter()
    for _ in range(reps):
        acc.add(g)
    dt = (time.perf_counter() - t0) / reps
    return 24 * n_params / dt / 1e9, dt


def reference_arm(args, w, ws, rank):
    if rank != 0:
        return
    n_b, n_mu = CPU_SAMPLE
    n_mu = min(n_mu, w.micro or n_mu)
    sps, cores, step_s = run_cpu_reference(w, args.steps, args.warmup, n_b, n_mu)
    sample = (f"each step: one mini-batch of {n_b} {w.model} {'x'.join(map(str, w.sample_shape))} samples of "
              f"this workload streamed as micro-batches of {n_mu}, float64 torch-CPU model + NumPy MBS arithmetic "
              f"(oracle port of engine.py/optim.py); samples/s is per-sample, so it compares with the GPU arm's")
    line = {"impl": "reference", "metric": METRIC, "value": sps, "unit": "samples/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_s * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(w, w.mini, w.micro or 128, ws),
            "setup": {"model": w.model, "model_ops": "reference numerics (float64 CPU, oracle port)",
                      "api": "oracle.mbs_oracle.train_mini_batch (engine.py:233-261 restated)"},
            "reference_sample": {"mini_batch": n_b, "micro_batch": n_mu, "steps": args.steps,
                                 "warmup": args.warmup},
            "cpu_baseline": {"value": sps, "unit": "samples/s", "cores": cores, "kind": "port", "sample": sample},
            "e2e": {"value": sps, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4", choices=["c1", "c2", "c3", "c4", "c5", "n1"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-fp32-context", action="store_true")
    ap.add_argument("--mini", type=int, default=0, help="override the workload's mini-batch (builder runs only)")
    ap.add_argument("--model-ops", default="native", choices=["native", "torch"],
                    help="the model's BatchNorm(+ReLU/+skip add) and max-pool: K5/K6 sm_100a kernels or stock torch")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    from paper_2110_12484_b200.workloads import WORKLOADS
    w = WORKLOADS[args.config]
    ws, rank, local = _dist()
    if args.impl == "reference":
        reference_arm(args, w, ws, rank)
        return
    run_gpu(args, w, ws, rank, local)


def run_gpu(args, w, ws, rank, local):
    import paper_2110_12484_b200 as mbs
    from paper_2110_12484_b200 import engine as _eng
    from paper_2110_12484_b200 import graphs as _graphs
    from paper_2110_12484_b200 import streaming as SS
    from paper_2110_12484_b200.prof import TIMER
    from paper_2110_12484_b200.streamer import Staging
    from paper_2110_12484_b200.workloads import build_model, synthetic_data

    ndev = torch.cuda.device_count()
    dev = torch.device("cuda", local % max(1, ndev))
    torch.cuda.set_device(dev)
    if ws > 1:
        import torch.distributed as dist
        backend = os.environ.get("MBS_DP_BACKEND", "nccl")   # gloo only for smoke runs of >1 rank per GPU
        if backend == "nccl":
            os.environ.setdefault("NCCL_DEBUG", "INFO")       # communicator INIT lines: rank count / NVLS
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    torch.backends.cudnn.benchmark = os.environ.get("MBS_BENCH_DETERMINISTIC", "0") != "1"
    torch.backends.cudnn.deterministic = not torch.backends.cudnn.benchmark
    torch.manual_seed(1234 + rank)

    model = build_model(w, ops=args.model_ops).to(dev).to(memory_format=torch.channels_last)
    params = mbs.ParameterSet(model, shadow=torch.bfloat16)   # bf16 shadow weights: K3 refreshes them, K1 reads bf16 grads
    staging = Staging(dtype=torch.bfloat16, channels_last=True, target_dtype=torch.float32)
    autocast = torch.bfloat16
    n_b, n_mu = (args.mini or w.mini), w.micro
    autosize = None
    if n_mu == 0:
        # config 5: micro-batch auto-sized to free HBM (memory.py:88-101 rule on measured bytes)
        from paper_2110_12484_b200 import memory
        from paper_2110_12484_b200.streamer import stage_rows

        def make_batch(k):
            xb, yb = synthetic_data(w, k, seed=99, device=dev)
            return stage_rows(xb, xb.dtype, tuple(xb.shape[1:]), None, 0, k, staging, dev), \
                (yb.float() if yb.dtype == torch.uint8 else yb)
        budget = memory.measure_budget(model, make_batch, w.loss_kind, optimizer_kind=w.optimizer,
                                       autocast_dtype=autocast, probe=(4, 8), safety=0.88)
        n_mu = memory.auto_micro_batch(budget, max(n_b, 4 * memory.fit_micro_batch(budget)), model)
        n_b = max(n_b, 4 * n_mu)             # a mini-batch that cannot fit HBM without streaming
        autosize = {"capacity_bytes": budget.capacity_bytes, "resident_bytes": budget.resident_bytes,
                    "data_bytes_per_sample": budget.data_bytes_per_sample, "micro": n_mu, "mini": n_b}
        torch.cuda.empty_cache()
    plan = mbs.plan_split(n_b, n_mu)

    # host dataset per rank: whole mini-batches, at most HOST_DATA_CAP bytes unless ONE mini-batch is larger
    # (C4: exactly one 45.2 GB mini-batch, reshuffled every epoch)
    row = int(np.prod(w.sample_shape)) + (int(np.prod(w.sample_shape[1:])) if w.target == "mask" else 8)
    d_minis = max(1, min(args.steps, HOST_DATA_CAP // (n_b * row)))
    t_data = time.perf_counter()
    pool = None
    if ws > 1 and os.environ.get("MBS_SHARED_HOST_POOL", "1") != "0":
        def _barrier():
            torch.distributed.barrier()
        pool = SharedHostPool(w, d_minis * n_b, local, _barrier)
        x_host = pool.x
        y_host = synthetic_data(w, d_minis * n_b, seed=rank, pinned=True)[1]      # per-rank labels / masks
    else:
        x_host, y_host = synthetic_data(w, d_minis * n_b, seed=rank, pinned=True)
    x_dev, y_dev = x_host.to(dev), y_host.to(dev)
    t_data = time.perf_counter() - t_data
    warm_small = min(n_b, 1024)          # e2e warm-up: one small mini-batch through the (already warm) stack

    dp = None
    if ws > 1:
        from paper_2110_12484_b200.dp import DataParallelMBS
        dp = DataParallelMBS(params, transport=os.environ.get("MBS_DP_TRANSPORT", "nccl"))
        warm_small = n_b                 # the global plan needs every rank's local mini-batch to be whole micros

    def make_opt():
        return mbs.sgd_state(0.01, 0.9, 5e-4) if w.optimizer == "sgd" else mbs.adam_state(0.01, 5e-4)

    acc = mbs.GradientAccumulator(params)
    st = make_opt()
    streamer = mbs.make_streamer(x_host, y_host, n_mu, n_slots=3)
    cs = torch.cuda.current_stream(dev)

    def run_steps(host: bool, n_steps: int, epoch0: int, mini: int = n_b, tracer=None):
        """``n_steps`` mini-batches = epochs over the dataset (d_minis mini-batches each); losses read back."""
        xs, ys = (x_host, y_host) if host else (x_dev, y_dev)
        losses, s = [], 0
        while s < n_steps:
            take = min(d_minis if mini == n_b else max(1, xs.shape[0] // mini), n_steps - s)
            xe, ye = xs[:take * mini], ys[:take * mini]
            if dp is not None:
                res = dp.train_epoch(model, xe, ye, mini_batch_size=mini, micro_batch_size=n_mu,
                                     normalization=w.normalization, loss_kind=w.loss_kind, optimizer_state=st,
                                     seed=rank, epoch_index=epoch0 + s, accumulator=acc, staging=staging,
                                     autocast_dtype=autocast, streamer=streamer if host else None, prefetch=True)
                losses += [r.loss for r in res]
            else:
                es = mbs.train_epoch(model, params, xe, ye, mini_batch_size=mini, micro_batch_size=n_mu,
                                     normalization=w.normalization, loss_kind=w.loss_kind, optimizer_state=st,
                                     seed=rank, epoch_index=epoch0 + s, shuffle=True, prefetch=True,
                                     accumulator=acc, staging=staging, autocast_dtype=autocast,
                                     streamer=streamer if host else None, tracer=tracer)
                losses += es.mini_losses
            s += take
        return losses

    def barrier():
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize(dev)

    def timed(host: bool, steps: int, tracer=None):
        barrier()
        TIMER.reset()
        if host:
            streamer.timings(flush=True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        w0 = time.perf_counter()
        e0.record(cs)
        losses = run_steps(host, steps, 100 * int(host), tracer=tracer)
        e1.record(cs)
        barrier()
        wall = time.perf_counter() - w0
        ms = e0.elapsed_time(e1)
        if ws > 1:
            t = torch.tensor([ms], device=dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            ms = float(t.item())
        return ms, losses, wall

    # --- value: inputs resident in HBM; W full warm-up mini-batches first ---
    run_steps(False, args.warmup, 1000)
    with ClockSampler(dev.index) as clocks:
        ms_dev, _, wall_dev = timed(False, args.steps)
    launches_value = TIMER.launches
    samples_total = n_b * args.steps * ws
    value = samples_total / (ms_dev / 1e3)

    # --- per-kernel bandwidths: two more HBM-resident small mini-batches with CUDA events around every launch on
    # its stream, outside the timed regions. K1-K4 run outside the captured micro step, so they are timed in
    # the graph-replay pipeline the timed run uses (the host runs ahead of the GPU there, so no launch gap lands
    # between an event and its kernel); K5 lives inside the graph, so it is timed in a separate eager pass ---
    TIMER.reset()
    TIMER.enabled = True
    run_steps(False, 2, 2000, mini=warm_small)
    TIMER.enabled = False
    kstats = TIMER.summary()
    k5stats = {}
    if args.model_ops == "native":
        _graphs.clear()
        graphs_on, _eng.CUDA_GRAPHS = _eng.CUDA_GRAPHS, False
        TIMER.reset()
        TIMER.enabled = TIMER.k5 = True
        run_steps(False, 1, 2500, mini=warm_small)
        TIMER.enabled = TIMER.k5 = False
        _eng.CUDA_GRAPHS = graphs_on
        k5stats = {k: v for k, v in TIMER.summary().items() if k.startswith("k5_")}
        _graphs.clear()

    # --- e2e: host-pinned inputs through the streamer, the run's real schedule traced ---
    run_steps(True, 1, 3000, mini=warm_small)
    tracer = SS.ScheduleTracer(dev) if ws == 1 else None
    # the e2e run repeats the value run's K steps unless that alone would exceed E2E_BUDGET_S (a C4 step is
    # 26 s: K = 50 would double a 22-minute bench); then it times as many whole steps as fit (>= 1)
    step_s = ms_dev / 1e3 / args.steps
    e2e_steps = args.steps if step_s * args.steps <= E2E_BUDGET_S else max(1, int(E2E_BUDGET_S // step_s))
    with ClockSampler(dev.index) as clocks_e2e:
        ms_host, losses, wall_host = timed(True, e2e_steps, tracer)
    launches_e2e = TIMER.launches
    e2e = n_b * e2e_steps * ws / (ms_host / 1e3)
    tim = streamer.timings(flush=True)
    copy_ms = sum(t[1] for t in tim)
    blocked_ms = sum(t[2] for t in tim)
    h2d_bytes = sum(t[3] for t in tim) / max(1, e2e_steps)
    h2d_gbs = (sum(t[3] for t in tim) / (copy_ms / 1e3) / 1e9) if copy_ms > 0 else None
    streamer.close()
    scheds = tracer.schedules() if tracer is not None else []

    # --- no-stream baseline: plain torch training at batch = micro, data resident ---
    _graphs.clear()
    torch.cuda.empty_cache()             # the MBS graphs' pools back to the driver (C5 fills HBM by design)
    nos = nos_torch = None
    for ops_ in (args.model_ops, "torch") if args.model_ops != "torch" else (args.model_ops,):
        b = n_mu
        r = None
        while b >= 1 and r is None:
            try:
                with ClockSampler(dev.index) as ck:
                    # the same-model baseline runs as long as the timed e2e run (its power / clock state: a
                    # 30 s U-Net@384 run held 1,597 MHz against the 206 s MBS run's 1,492 under the power cap)
                    min_s = NO_STREAM_MIN_S if ops_ != args.model_ops else \
                        min(NO_STREAM_MAX_S, max(NO_STREAM_MIN_S, ms_host / 1e3))
                    r = no_stream_baseline(w, dev, b, args.steps, args.warmup, ws, ops=ops_, min_s=min_s,
                                           data=(x_dev, y_dev))
                r["clocks"] = ck.summary()
            except torch.OutOfMemoryError:
                b //= 2
            torch.cuda.empty_cache()
        if ops_ == args.model_ops:
            nos = r
        else:
            nos_torch = r
    # the same baseline with the weights held at init (lr 1e-9): the MBS run takes one optimizer step per
    # mini-batch, the baseline one per micro-batch, and on synthetic data the power a step draws depends on
    # the weight state — U-Net@384: the MBS engine at one micro per step runs 1,717 MHz / 1,289 samples/s
    # at lr 0.01 and 1,500 MHz / 1,165 at lr 1e-9, all at the 985 W cap (profiles/r02_power_state.md)
    nos_init = None
    if nos is not None:
        try:
            with ClockSampler(dev.index) as ck:
                nos_init = no_stream_baseline(w, dev, nos["batch"], args.steps, args.warmup, ws, ops=args.model_ops,
                                              data=(x_dev, y_dev), lr=1e-9)
            nos_init["clocks"] = ck.summary()
        except torch.OutOfMemoryError:
            nos_init = None
        torch.cuda.empty_cache()

    # --- the reference's overhead report on the measured schedules ---
    overhead = None
    if scheds:
        mk = [s.makespan for s in scheds]
        fr = [f for f in (SS.overlap_fraction(s) for s in scheds) if f is not None]
        per_kind = {}
        for s in scheds:
            for e in s.events:
                per_kind[e.kind] = per_kind.get(e.kind, 0.0) + (e.end - e.start)
        mbs_sched = scheds[-1]
        base_sched = None
        if nos:
            base_mk = n_b / (nos["value"] / ws)
            base_sched = SS.StreamSchedule(tuple(SS.StreamEvent(*e) for e in nos["events"]), base_mk, False)
        rep = SS.overhead_report(mbs_sched, base_sched)
        overhead = {"mbs_makespan_s": rep.mbs_makespan, "no_stream_makespan_s": rep.baseline_makespan,
                    "overhead_pct": rep.overhead_pct, "overhead_seconds": rep.overhead_seconds,
                    "mbs_makespan_s_per_mini_batch": mk, "h2d_overlap_pct": 100.0 * float(np.mean(fr)) if fr else None,
                    "seconds_per_mini_batch_by_kind": {k: v / len(scheds) for k, v in per_kind.items()},
                    "events_per_mini_batch": len(mbs_sched.events),
                    "how": "streaming.overhead_report (streaming.py:130-149) on the last timed e2e mini-batch's "
                           "StreamSchedule, recorded by streaming.ScheduleTracer (CUDA events per micro-batch: "
                           "transfer on the copy stream, forward / backward(+K1) / update on the compute stream); "
                           "baseline = the no-stream run's measured per-sample time x N_B (it ran "
                           f"{nos['samples'] if nos else 0} samples); overlap = 1 - (compute-stream wait on "
                           "copies) / (copy time), from the same events"}
        if nos_init:
            base_mk = n_b / (nos_init["value"] / ws)
            rep0 = SS.overhead_report(mbs_sched, SS.StreamSchedule(
                tuple(SS.StreamEvent(*e) for e in nos_init["events"]), base_mk, False))
            overhead["vs_weights_at_init"] = {"no_stream_makespan_s": rep0.baseline_makespan,
                                              "overhead_pct": rep0.overhead_pct,
                                              "overhead_seconds": rep0.overhead_seconds}

    k1 = kstats.get("k1_accumulate", {})
    peak, peak_kind = _peaks()
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_k1_traffic.json")) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")
    except Exception:
        pass
    gbytes = 2 if getattr(params, "shadow", None) is not None else 4
    roofline = {"kernel": "k1_accumulate (mbs_accum_add_typed)", "bound": "hbm", "achieved": k1.get("gbs"),
                "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                "frac": (k1.get("gbs") or 0.0) / peak, "traffic": traffic,
                "algorithmic_bytes_per_launch": k1.get("bytes_per_launch"),
                "avg_launch_us": (k1.get("avg_ms") or 0) * 1e3, "launches_timed": k1.get("launches"),
                "bytes_rule": (f"per parameter: read g ({gbytes} B: bf16 weight gradients of the shadow-weight "
                               "matmuls, fp32 for BN / bias) + read acc (4 B) + write acc (4 B); the first micro-batch "
                               "of a mini-batch assigns acc = s*g (no acc read); P = %d" % params.layout.n_params),
                "how": "CUDA events around every K1 launch (on its stream) of two extra HBM-resident mini-batches "
                       "run like the timed ones (micro step replayed from a CUDA graph, K1 after each replay), "
                       "outside the timed region",
                "other_kernels": {k: {"gbs": v["gbs"], "avg_us": v["avg_ms"] * 1e3, "launches": v["launches"],
                                      "bytes_per_launch": v["bytes_per_launch"]}
                                  for k, v in kstats.items() if k != "k1_accumulate"}}
    if x_dev.dim() == 4 and x_dev.dtype == torch.uint8:
        roofline["other_kernels"]["k2_stage_back_to_back"] = k2_back_to_back(x_dev, staging, dev, n_mu)
        roofline["other_kernels"]["k2_stage_back_to_back"]["frac"] = \
            roofline["other_kernels"]["k2_stage_back_to_back"]["gbs"] / peak
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
                   "how": "samples/s x algorithmic fwd+bwd FLOP per sample (FlopCounterMode: the model's "
                          "convolutions/matmuls), against the bf16 dense peak"}
    roofline_k5 = None
    if k5stats:
        kb = sum(v["bytes_per_launch"] * v["launches"] for v in k5stats.values())
        kt = sum(v["total_ms"] for v in k5stats.values())
        roofline_k5 = {"kernel": "k5 micro-batch BatchNorm (+ReLU/+residual), forward and backward (model side)",
                       "bound": "hbm", "achieved": kb / (kt / 1e3) / 1e9, "peak": peak, "unit": "GB/s",
                       "frac": kb / (kt / 1e3) / 1e9 / peak, "ms_per_small_mini_batch": kt}

    precision = {"dtype": "bf16",
                 "detail": "bf16 autocast compute on cuDNN/cuBLAS reading bf16 shadow weights that K3 writes; bf16 "
                           "weight gradients widened by K1; fp32 master weights, fp32 MBS accumulation, fp32 "
                           "optimizer state; inputs uint8 staged exactly to bf16",
                 "parity": "pinned to the float64 oracle in tests/test_bench_stack_parity_gpu.py (this exact stack, "
                           "bf16 and fp32, at C1 / ResNet-50@224 / U-Net@384 shapes)"}

    fp32_ctx = None
    if not args.no_fp32_context and ws == 1:
        _graphs.clear()
        torch.cuda.empty_cache()
        try:
            fp32_ctx = fp32_context(w, dev, n_mu, warm_small, args.model_ops, x_dev, y_dev)
        except torch.OutOfMemoryError as e:                # context only: never lose the line to it
            fp32_ctx = {"unavailable": f"OutOfMemoryError: {str(e)[:120]}"}
        torch.cuda.empty_cache()

    config = workload_config(w, n_b, n_mu, ws)
    setup = {"model": w.model,
             "model_ops": "BatchNorm(+ReLU/+skip add) on K5, max-pool (+U-Net skip join) on K6, stem conv as K7 "
                          "im2col + GEMM, micro-batch statistics; micro step replayed from CUDA graphs"
                          if args.model_ops == "native" else "stock torch"}
    setup.update({"precision": precision["detail"], "autosize": autosize,
                   "host_dataset": {"mini_batches": d_minis, "samples": d_minis * n_b,
                                    "bytes": int(x_host.numel() * x_host.element_size() +
                                                 y_host.numel() * y_host.element_size()),
                                    "pinned": True, "setup_s": t_data,
                                    "images": ("one page-locked copy per node in %s, mapped by every rank; each "
                                               "rank streams it in its own order" % pool.where) if pool else
                                              "per rank, page-locked"},
                   "steps_are": "one mini-batch each; an epoch over the host dataset every "
                                f"{d_minis} steps, reshuffled by epoch_index",
                   "warmup_is": f"{args.warmup} full mini-batches before the HBM-resident (value) run; 1 mini-batch "
                                f"of {warm_small} through the host streamer before the e2e run",
                   "api": ("engine.train_epoch" if ws == 1 else "dp.DataParallelMBS.train_epoch (per-rank shards, "
                           "one all-reduce per global mini-batch, transport=%s over the %s process group)"
                           % (dp.transport, torch.distributed.get_backend()))})
    line = {"metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_dev / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (uint8 images, random labels / masks; random-init weights)",
            "config": config, "setup": setup,
            "e2e": {"value": e2e, "unit": "samples/s", "h2d_bytes_per_step": int(h2d_bytes),
                    "d2h_bytes_per_step": 8 * (4 + 2 * plan.n_s_mu), "ms_per_step": ms_host / e2e_steps,
                    "steps": e2e_steps, "wall_s": wall_host},
            "e2e_vs_no_stream": e2e / nos["value"] if nos else None,
            # both runs sit at the power cap; their median SM clocks differ by a few % (U-Net: MBS 1492 vs
            # no-stream 1597 MHz), so the ratio per clock is stated beside the raw one
            "e2e_vs_no_stream_per_clock": _per_clock(e2e, clocks_e2e.summary(), nos),
            "e2e_vs_no_stream_weights_at_init": e2e / nos_init["value"] if nos_init else None,
            "value_vs_no_stream": value / nos["value"] if nos else None,
            "h2d_overlap_pct": (overhead or {}).get("h2d_overlap_pct"),
            "h2d_overlap_pct_streamer": 100.0 * (1.0 - blocked_ms / copy_ms) if copy_ms > 0 else None,
            "h2d_gbs": h2d_gbs, "accum_gbs": k1.get("gbs"),
            "no_stream": {k: v for k, v in (nos or {}).items() if k != "events"} or None,
            "no_stream_torch_ops": {k: v for k, v in (nos_torch or {}).items() if k != "events"} or None,
            "no_stream_weights_at_init": {k: v for k, v in (nos_init or {}).items() if k != "events"} or None,
            "overhead": overhead, "roofline": roofline, "roofline_k5": roofline_k5, "model_flops": model_flops,
            "precision": precision, "precision_fp32": fp32_ctx,
            "gpu_launches": launches_value, "gpu_launches_e2e": launches_e2e,
            "clocks": clocks.summary(), "clocks_e2e": clocks_e2e.summary(),
            "final_loss": losses[-1] if losses else None, "value_wall_s": wall_dev}

    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu_n_b, cpu_mu = CPU_SAMPLE
        sps, cores, step_s = run_cpu_reference(w, 1, 1, cpu_n_b, cpu_mu)
        line["cpu_baseline"] = {"value": sps, "unit": "samples/s", "cores": cores, "kind": "port",
                                "sample": f"1 mini-batch of {cpu_n_b} as micro {cpu_mu} (after 1 warm-up), {w.model} "
                                          f"float64 torch-CPU + NumPy MBS oracle, {step_s:.1f} s/step"}
        shapes = {n: tuple(params[n].shape) for n in params.names()}
        agbs, adt = run_cpu_accumulate(shapes)
        line["cpu_baseline"]["accum_gbs"] = {"value": agbs, "unit": "GB/s", "cores": 1, "kind": "port",
                                             "sample": f"GradientAccumulator.add of one {params.layout.n_params}-"
                                                       f"parameter fp64 gradient, 24 B/param, {adt * 1e3:.0f} ms/add"}
    if rank == 0:
        print(json.dumps(line))
    if ws > 1:
        if pool is not None:
            del x_host
            pool.close(torch.distributed.barrier)
        torch.distributed.destroy_process_group()


def k2_back_to_back(x_dev, staging, dev, n_mu: int, reps: int = 16) -> dict:
    """K2 (gather by index + u8 -> bf16 NHWC) timed as ``reps`` back-to-back launches between two events on a
    pre-filled stream (host launch gaps off the clock), each over a DIFFERENT shuffled micro-batch of the
    HBM-resident dataset into its own output, so sources and outputs are cold (reps x the micro-batch bytes
    >> L2). Event resolution is ~2 us here, too coarse for one ~10 us launch; this amortises it."""
    from paper_2110_12484_b200.streamer import stage_rows
    n = x_dev.shape[0]
    reps = max(1, min(reps, n // n_mu))
    g = torch.Generator(device=dev).manual_seed(7)
    rows = torch.randperm(n, generator=g, device=dev)[:reps * n_mu].contiguous()
    outs = [staging.out_tensor(n_mu, tuple(x_dev.shape[1:]), dev) for _ in range(reps)]
    shape = tuple(x_dev.shape[1:])
    ms = []
    for _ in range(3):
        torch.cuda.synchronize(dev)
        torch.cuda._sleep(20_000_000)                  # ~10 ms of GPU work: every launch below is queued
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for r in range(reps):
            stage_rows(x_dev, x_dev.dtype, shape, rows[r * n_mu:(r + 1) * n_mu], 0, n_mu, staging, dev, out=outs[r])
        e1.record()
        torch.cuda.synchronize(dev)
        ms.append(e0.elapsed_time(e1) / reps)
    us = 1e3 * float(np.median(ms))
    nbytes = n_mu * int(np.prod(shape)) * (x_dev.element_size() + outs[0].element_size())
    return {"gbs": nbytes / (us / 1e6) / 1e9, "avg_us": us, "launches": reps, "bytes_per_launch": nbytes,
            "how": f"{reps} back-to-back launches over distinct shuffled micro-batches, median of 3"}


def fp32_context(w, dev, n_mu, mini, model_ops, x_dev, y_dev):
    """The MBS stack at fp32 (fp32 weights, staging and compute, TF32 off): the precision the oracle pins."""
    import paper_2110_12484_b200 as mbs
    from paper_2110_12484_b200.streamer import Staging
    from paper_2110_12484_b200.workloads import build_model
    tf = (torch.backends.cuda.matmul.allow_tf32, torch.backends.cudnn.allow_tf32)
    torch.backends.cuda.matmul.allow_tf32 = torch.backends.cudnn.allow_tf32 = False
    try:
        torch.manual_seed(5)
        model = build_model(w, ops=model_ops).to(dev).to(memory_format=torch.channels_last)
        params = mbs.ParameterSet(model)
        st = mbs.sgd_state(0.01, 0.9, 5e-4) if w.optimizer == "sgd" else mbs.adam_state(0.01, 5e-4)
        staging = Staging(torch.float32, True, target_dtype=torch.float32)
        n = 3 * mini

        def run(e):
            return mbs.train_epoch(model, params, x_dev[:n], y_dev[:n], mini_batch_size=mini, micro_batch_size=n_mu,
                                   normalization=w.normalization, loss_kind=w.loss_kind, optimizer_state=st, seed=0,
                                   epoch_index=e, staging=staging)
        run(0)
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run(1)
        e1.record()
        torch.cuda.synchronize(dev)
        ms = e0.elapsed_time(e1)
        del model, params, st
        return {"value": n / (ms / 1e3), "unit": "samples/s", "dtype": "f32 (TF32 off)", "mini_batch": mini,
                "micro_batch": n_mu, "mini_batches_timed": 3, "warmup_mini_batches": 3,
                "how": "same MBS stack (K1-K7, CUDA graphs, HBM-resident uint8 staged to fp32) at the precision "
                       "every oracle parity test also pins; context only"}
    finally:
        torch.backends.cuda.matmul.allow_tf32, torch.backends.cudnn.allow_tf32 = tf


NO_STREAM_MIN_S = 30.0          # the no-stream baseline runs at least this long (same power / clock state as MBS)
NO_STREAM_MAX_S = 300.0         # ... and as long as the timed e2e run, up to this
NO_STREAM_POOL = 64             # distinct batches the baseline cycles through
NO_STREAM_POOL_BYTES = 2 << 30  # ... within this many staged bytes (C5's auto-sized micro-batch leaves no room)


def _per_clock(e2e, e2e_clocks: dict, nos: dict | None):
    """(e2e / its median SM MHz) / (no-stream / its median SM MHz), or None when a clock is missing."""
    try:
        a, b = float(e2e_clocks["sm_mhz"]), float(nos["clocks"]["sm_mhz"])
        return (e2e / a) / (nos["value"] / b)
    except (TypeError, KeyError, ValueError, ZeroDivisionError):
        return None


def no_stream_baseline(w, dev, batch, steps, warmup, ws, ops="torch", graph=True, min_s=NO_STREAM_MIN_S, data=None,
                       lr=0.01):
    """The paper's 'w/o MBS' run: plain torch training, batch = micro-batch, data resident in HBM.

    ``ops`` selects the same model definition as the MBS run (native K5/K6/K7 or stock torch ops).
    ``graph``: the whole training step (fwd + bwd + fused optimizer step) is replayed from one CUDA
    graph, like the MBS micro step — eager, this loop is host-bound on B200 and its number then
    tracks the host CPU rather than the GPU. Falls back to eager if capture fails. Every step is
    bracketed by CUDA events (the baseline's measured "compute" schedule). It runs for at least
    ``min_s`` seconds: a sub-second burst would be timed at boost clocks the minutes-long MBS run under
    the power cap does not see. ``lr``: 0.01 is the run's own learning rate; 1e-9 keeps the weights at
    their initial values (the matched-weight-state run, see bench's ``no_stream_weights_at_init``). ``data``: the MBS run's own (HBM-resident) dataset; the baseline then cycles
    through its first NO_STREAM_POOL batches (pre-staged to bf16 NHWC, untimed) instead of two synthetic
    ones, so both runs train on data of the same statistics (two repeated batches are memorised within
    seconds; the shrinking gradients then lower the power draw and flatter the baseline's clock)."""
    from paper_2110_12484_b200.losses import compute_loss
    from paper_2110_12484_b200.workloads import build_model, synthetic_data
    torch.manual_seed(0)
    model = build_model(w, ops=ops).to(dev).to(memory_format=torch.channels_last)
    if w.optimizer == "sgd":
        opt = torch.optim.SGD(model.parameters(), lr=lr, momentum=0.9, weight_decay=5e-4, fused=True)
    else:
        opt = torch.optim.Adam(model.parameters(), lr=lr, weight_decay=5e-4, fused=True, capturable=graph)
    if data is not None and data[0].shape[0] >= 2 * batch:
        x, y = data
        staged = batch * (x[0].numel() * 2 + (y[0].numel() * 4 if y.dim() > 1 else 8))   # bf16 image + target
        n_pool = max(2, min(NO_STREAM_POOL, x.shape[0] // batch, NO_STREAM_POOL_BYTES // staged))
    else:
        x, y = synthetic_data(w, 2 * batch, seed=7, device=dev)
        n_pool = 2
    xs = [x[i * batch:(i + 1) * batch].to(torch.bfloat16).contiguous(memory_format=torch.channels_last)
          for i in range(n_pool)]
    ys = [y[i * batch:(i + 1) * batch] for i in range(n_pool)]
    ys = [t.float() if t.dtype == torch.uint8 else t for t in ys]
    sx, sy = xs[0].clone(), ys[0].clone()

    def step(cache=True):
        with torch.autocast("cuda", dtype=torch.bfloat16, cache_enabled=cache):
            loss = compute_loss(w.loss_kind, model(sx), sy)
        loss.backward()
        opt.step()
        return loss

    def one(i):
        sx.copy_(xs[i % n_pool])
        sy.copy_(ys[i % n_pool])
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
                sx.copy_(xs[i % n_pool])
                sy.copy_(ys[i % n_pool])
                g.replay()
            for i in range(2):
                one(i)
            how = "CUDA graph of torch fwd/bwd + fused torch.optim step per batch, bf16 autocast, data in HBM"
        except Exception as e:                           # noqa: BLE001
            print(f"no-stream baseline: graph capture failed ({type(e).__name__}: {e}); eager", file=sys.stderr)
    torch.cuda.synchronize(dev)
    n = steps * max(1, min(w.mini, 1024) // batch)
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0.record()
    for i in range(3):
        one(i)
    c1.record()
    torch.cuda.synchronize(dev)
    n = max(n, int(math.ceil(min_s / (c0.elapsed_time(c1) / 3e3))))
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(n + 1)]
    evs[0].record()
    for i in range(n):
        one(i)
        evs[i + 1].record()
    torch.cuda.synchronize(dev)
    ms = evs[0].elapsed_time(evs[-1])
    events = [("compute", i, evs[0].elapsed_time(evs[i]) / 1e3, evs[0].elapsed_time(evs[i + 1]) / 1e3)
              for i in range(n)]
    del model, opt
    return {"value": batch * n * ws / (ms / 1e3), "unit": "samples/s", "batch": batch, "steps": n,
            "samples": batch * n, "model_ops": ops, "how": how, "events": events,
            "data": (f"the first {n_pool} batches ({n_pool * batch} samples) of the MBS run's dataset, cycled"
                     if data is not None and data[0].shape[0] >= 2 * batch else "two synthetic batches, cycled")}


if __name__ == "__main__":
    main()
