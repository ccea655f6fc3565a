"""Data-parallel MBS across the GPUs of one node: one all-reduce per mini-batch.

The reference is single-device; this layer is new. The
micro-batches of one mini-batch are independent until the sum
(``engine.py:206-216``, Eq. 13), so the GLOBAL plan ``plan_split(N_B, N_mu)``
is partitioned into contiguous blocks of whole micro-batches, one block per
rank (at most one micro-batch of imbalance). Each rank:

1. streams its own micro-batches and accumulates them with K1 using the
   GLOBAL normalisation factors (``size_k / N_B`` or ``1 / N_Smu``) — so BN
   micro-batch membership, and therefore every per-micro gradient, is exactly
   the single-device one;
2. on its LAST micro-batch, accumulates gradient BUCKETS as autograd produces
   them (post-accumulate-grad hooks) and immediately launches an async NCCL
   SUM all-reduce of that bucket's slice of the flat accumulator (in a fixed
   bucket order), so the all-reduce overlaps the rest of the backward
    — or, with ``transport="peer"``, runs the last K1 and the
   all-reduce as ONE kernel over CUDA-IPC peer memory (K1C, ``mbs_peer.cu``);
3. after the last bucket, recomputes the grad norm of the reduced sum (the
   optimizer's non-finite guard), all-reduces the tiny loss record, merges the
   BN running statistics so they equal the single-device sequential ones
   (``BNStatSync``, one small all-reduce), and runs the identical K3 step on
   every rank.

The pure functions (partition, factors, buckets, stats combination) carry the
logic and are exercised on CPU with the gloo backend (tests/test_dp_gloo.py).
"""

from __future__ import annotations

import math
from contextlib import nullcontext

import numpy as np
import torch

from .engine import (GradientAccumulator, MicroBatchPlan, MiniBatchStats, _as_tensor, _micro_source, make_streamer,
                     normalization_factor, plan_split, weight_cast_cache, _graph_dest, _graph_for)
from .losses import compute_loss
from .optim import apply_update
from .tensor import ParameterSet


def partition_micro_batches(plan: MicroBatchPlan, world: int) -> list:
    """Contiguous blocks of whole micro-batch indices per rank: [(k0, k1), ...] (at most 1 of imbalance)."""
    if world < 1:
        raise ValueError("world size must be positive")
    q, r = divmod(plan.n_s_mu, world)
    out, k = [], 0
    for i in range(world):
        n = q + (1 if i < r else 0)
        out.append((k, k + n))
        k += n
    return out


def rank_samples(plan: MicroBatchPlan, block: tuple) -> tuple:
    """Global sample range [lo, hi) covered by a block of micro-batches."""
    k0, k1 = block
    if k1 <= k0:
        return (0, 0)
    return (plan.index_ranges[k0][0], plan.index_ranges[k1 - 1][1])


def local_factors(plan: MicroBatchPlan, block: tuple, mode: str) -> list:
    """GLOBAL normalisation factors of this rank's micro-batches (engine.py:81-91 on the global plan)."""
    return [normalization_factor(plan, k, mode) for k in range(*block)]


def weak_scaling_plan(n_b_per_rank: int, n_mu: int, world: int) -> MicroBatchPlan:
    """Global plan when every rank holds its own n_b_per_rank samples (must split on micro boundaries)."""
    if world > 1 and n_b_per_rank % n_mu:
        raise ValueError("weak scaling needs the per-rank mini-batch to be a multiple of the micro-batch")
    return plan_split(n_b_per_rank * world, n_mu)


def bucket_ranges(numels: tuple, bucket_elems: int) -> list:
    """Contiguous segment ranges [(s0, s1), ...] of ~bucket_elems, listed from the LAST segment backwards
    (the order autograd produces gradients in)."""
    out, hi, acc = [], len(numels), 0
    for i in range(len(numels) - 1, -1, -1):
        acc += numels[i]
        if acc >= bucket_elems:
            out.append((i, hi))
            hi, acc = i, 0
    if hi > 0:
        out.append((0, hi))
    return out


def combine_loss_record(losses_local: list, factors_local: list, weights_local: list, block: tuple, n_s_mu: int,
                        n_b: int) -> np.ndarray:
    """Per-rank vector [lsum/N_B, raw losses (global slots), normalised losses] to be SUM-all-reduced."""
    v = np.zeros(1 + 2 * n_s_mu)
    k0, _ = block
    for j, (l, f, wgt) in enumerate(zip(losses_local, factors_local, weights_local)):
        v[0] += wgt * l
        v[1 + k0 + j] = l
        v[1 + n_s_mu + k0 + j] = l * f
    v[0] /= n_b
    return v


def bn_merge_coefficients(momentum, block: tuple, n_s_mu: int) -> tuple:
    """Coefficients that turn per-rank BN running statistics into the single-device sequential ones.

    torch BN (and the reference, ``nn.py:329-332``) updates a running statistic
    once per micro-batch, r <- (1-m) r + m s_k, in plan order. Starting every
    rank from the same r0, rank r's block of n_r micro-batches ends at
    R_r = c^n_r r0 + L_r (c = 1-m, L_r its own terms), and the single-device
    run over all K micro-batches ends at c^K r0 + sum_r c^(K-k1_r) L_r. So the
    exchange is ONE SUM all-reduce of contrib_r = a (R_r - b r0), followed by
    R = g r0 + sum, with (a, b, g) = (c^(K-k1_r), c^n_r, c^K) returned here.
    ``momentum=None`` (cumulative average) is handled on device by the caller.
    """
    k0, k1 = block
    c = 1.0 - float(momentum)
    return c ** (n_s_mu - k1), c ** (k1 - k0), c ** n_s_mu


class BNStatSync:
    """Makes data-parallel BN running statistics equal the single-device MBS run.

    Each rank sees only its own micro-batches, so without this its
    ``running_mean/var`` follow a different EMA than the single-device run.
    ``snapshot()`` before the rank's first micro-batch forward, ``merge()``
    after its last: one SUM all-reduce of a flat buffer of every BN running
    statistic (ResNet-50: 53 layers, 53,120 values) recovers the sequential
    single-device statistics exactly up to fp32 rounding, and
    ``num_batches_tracked`` advances by the GLOBAL micro-batch count.
    """

    def __init__(self, model: torch.nn.Module, dist, group=None):
        bn = torch.nn.modules.batchnorm._BatchNorm
        self.mods = [m for m in model.modules()
                     if isinstance(m, bn) and m.track_running_stats and m.running_mean is not None]
        self.dist, self.group = dist, group
        self._coef = {}
        self._r0 = None
        self._n0 = None

    def _bufs(self):
        return [t for m in self.mods for t in (m.running_mean, m.running_var)]

    def snapshot(self):
        if not self.mods:
            return
        with torch.no_grad():
            self._r0 = torch.cat([t.reshape(-1) for t in self._bufs()])
            self._n0 = torch.stack([m.num_batches_tracked for m in self.mods])

    def merge(self, block: tuple, n_s_mu: int):
        """contrib = A*local - B*r0 (SUM-all-reduced), then r = (G*r0 + sum) * D, per BN layer:
        EMA layers (a, a*b, g, 1) from ``bn_merge_coefficients``; cumulative-average layers
        (n0+n_r, n0, n0, 1/(n0+K)) with n0 = num_batches_tracked before the step (on device)."""
        if not self.mods:
            return
        with torch.no_grad():
            r0 = self._r0
            dev, dt = r0.device, r0.dtype
            n_r = block[1] - block[0]
            key = (block, n_s_mu)
            if key not in self._coef:
                ema = [bn_merge_coefficients(m.momentum if m.momentum is not None else 0.0, block, n_s_mu)
                       for m in self.mods]
                host = torch.tensor([[a, a * b, g, 1.0] for a, b, g in ema], dtype=torch.float64)
                cma = torch.tensor([m.momentum is None for m in self.mods])
                counts = torch.tensor([2 * m.running_mean.numel() for m in self.mods])
                self._coef[key] = (host.to(dev), cma.to(dev), counts.to(dev), bool(cma.any()))
            host, cma, counts, any_cma = self._coef[key]
            coef = host
            if any_cma:
                n0 = self._n0.double()
                alt = torch.stack([n0 + n_r, n0, n0, 1.0 / (n0 + n_s_mu)], dim=1)
                coef = torch.where(cma[:, None], alt, host)
            A, B, G, D = torch.repeat_interleave(coef.to(dt), counts, dim=0).unbind(1)
            local = torch.cat([t.reshape(-1) for t in self._bufs()])
            contrib = A * local - B * r0
            self.dist.all_reduce(contrib, group=self.group)
            new = (G * r0 + contrib) * D
            bufs = self._bufs()
            torch._foreach_copy_(bufs, [p.view_as(t) for p, t in zip(new.split([t.numel() for t in bufs]), bufs)])
            for m, n0 in zip(self.mods, self._n0):
                m.num_batches_tracked.copy_(n0 + n_s_mu)


class _Result:
    """MiniBatchStats-compatible view of the combined global statistics."""

    def __init__(self, vec_dev: torch.Tensor, norm2_dev: torch.Tensor, n_s_mu: int):
        self._n = n_s_mu
        self._host = torch.empty(vec_dev.numel() + 1, dtype=torch.float64, pin_memory=True)
        self._host[:-1].copy_(vec_dev, non_blocking=True)
        self._host[-1:].copy_(norm2_dev.reshape(1), non_blocking=True)
        self._ev = torch.cuda.Event()
        self._ev.record()
        self.step_count = 0
        self._r = None

    def resolve(self):
        if self._r is None:
            self._ev.synchronize()
            h = self._host.tolist()
            n = self._n
            self._r = dict(loss=h[0], losses_raw=h[1:1 + n], losses_normalized=h[1 + n:1 + 2 * n], norm2=h[-1])
            if not (math.isfinite(h[-1]) and all(math.isfinite(v) for v in h[:-1])):
                from .errors import NonFiniteError
                raise NonFiniteError(-1, "non-finite accumulated gradient or micro-batch loss; no update was applied")
        return self._r

    loss = property(lambda s: s.resolve()["loss"])
    losses_raw = property(lambda s: s.resolve()["losses_raw"])
    losses_normalized = property(lambda s: s.resolve()["losses_normalized"])
    grad_norm = property(lambda s: math.sqrt(s.resolve()["norm2"]))
    n_micro = property(lambda s: s._n)
    outputs = None


class PeerExchange:
    """Symmetric exchange buffers for the fused K1 + all-reduce over peer memory (``mbs_peer_*``).

    Every rank allocates its buffer in the native library, exports CUDA IPC
    handles, and maps every peer's buffer (NVLink/NVSwitch P2P inside a node;
    ranks sharing one GPU also work, which is how it is tested on one B200).
    """

    def __init__(self, numel: int, group=None):
        import ctypes

        import torch.distributed as dist
        from . import _native as N
        self.N = N
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        h = ctypes.c_void_p()
        N.check(N.lib().mbs_peer_create(self.rank, self.world, int(numel), ctypes.byref(h)), "mbs_peer_create")
        self.handle = h
        mine = (ctypes.c_char * N.PEER_HANDLE_BYTES)()
        N.check(N.lib().mbs_peer_handle(h, mine), "mbs_peer_handle")
        allh = [None] * self.world
        dist.all_gather_object(allh, bytes(mine), group=group)
        buf = (ctypes.c_char * (N.PEER_HANDLE_BYTES * self.world)).from_buffer_copy(b"".join(allh))
        N.check(N.lib().mbs_peer_open(h, buf), "mbs_peer_open")
        dist.barrier(group=group)

    def error(self) -> bool:
        import ctypes
        v = ctypes.c_int()
        self.N.check(self.N.lib().mbs_peer_status(self.handle, ctypes.byref(v)), "mbs_peer_status")
        return bool(v.value)

    def close(self):
        if getattr(self, "handle", None):
            self.N.lib().mbs_peer_destroy(self.handle)
            self.handle = None


class DataParallelMBS:
    """Per-rank driver of data-parallel micro-batch streaming.

    ``transport="nccl"`` (default): bucket-wise K1 from post-accumulate-grad hooks + async NCCL
    all-reduce overlapped with the last backward. ``transport="peer"``: the last micro-batch's K1
    and the all-reduce are ONE kernel over peer memory (``PeerExchange``, K1C).
    """

    def __init__(self, params: ParameterSet, process_group=None, bucket_mb: float = 32.0, transport: str = "nccl",
                 bn_stats: str = "sequential"):
        import torch.distributed as dist
        if transport not in ("nccl", "peer"):
            raise ValueError(f"unknown transport {transport!r}")
        if bn_stats not in ("sequential", "local"):
            raise ValueError(f"unknown bn_stats mode {bn_stats!r}")
        self.bn_stats = bn_stats
        self._bn = {}
        self.dist = dist
        self.params = params
        self.group = process_group
        self.world = dist.get_world_size(process_group)
        self.rank = dist.get_rank(process_group)
        self.transport = transport
        self.peer = PeerExchange(params.layout.total, process_group) if transport == "peer" else None
        self.buckets = bucket_ranges(params.layout.numels, max(1, int(bucket_mb * 2 ** 20 / 4)))
        self._seg_bucket = {}
        for b, (s0, s1) in enumerate(self.buckets):
            for s in range(s0, s1):
                self._seg_bucket[s] = b

    def _slice(self, acc: GradientAccumulator, s0: int, s1: int) -> torch.Tensor:
        lay = acc.layout
        lo = lay.offsets[s0]
        hi = lay.offsets[s1 - 1] + lay.numels[s1 - 1]
        return acc.flat[lo:hi]

    def train_mini_batch(self, model, batch, n_b_per_rank: int, n_mu: int, normalization: str, loss_kind: str,
                         optimizer_state, *, accumulator: GradientAccumulator, staging=None, autocast_dtype=None,
                         streamer=None, prefetch=True, loss_from_logits=True, dice_smoothing=1.0,
                         lr_for_step=None):
        """Weak-scaling step: this rank's batch holds its own n_b_per_rank samples (= its block of the global plan)."""
        plan = weak_scaling_plan(n_b_per_rank, n_mu, self.world)
        block = partition_micro_batches(plan, self.world)[self.rank]
        lo, hi = rank_samples(plan, block)
        x, y = (_as_tensor(t) for t in batch)
        if x.shape[0] != hi - lo:
            raise ValueError(f"rank {self.rank} holds {x.shape[0]} samples, its block of the plan needs {hi - lo}")
        jobs = [(None, plan.index_ranges[k][0] - lo, plan.sizes[k]) for k in range(*block)]
        own = None
        if x.device.type == "cpu" and streamer is None:
            streamer = own = make_streamer(x, y, n_mu)
        try:
            dest = _graph_dest(model, accumulator, loss_kind, autocast_dtype, loss_from_logits, dice_smoothing,
                               "fused")
            source = iter(_micro_source(x, y, jobs, staging, prefetch, streamer, dest))
            return self._step(model, plan, block, source, normalization, loss_kind, optimizer_state, accumulator,
                              autocast_dtype, loss_from_logits, dice_smoothing, lr_for_step)
        finally:
            if own is not None:
                own.close()

    def train_epoch(self, model, x, y, *, mini_batch_size: int, micro_batch_size: int, normalization: str,
                    loss_kind: str, optimizer_state, seed: int, epoch_index: int, accumulator: GradientAccumulator,
                    shuffle: bool = True, staging=None, autocast_dtype=None, streamer=None, prefetch=True,
                    loss_from_logits=True, dice_smoothing=1.0, lr_for_step=None) -> list:
        """One weak-scaling epoch: every rank walks ITS shard (x, y) in its own shuffled order.

        Rank r's order is the reference's named stream extended by the rank,
        ``named_stream(seed, f"shuffle/epoch{e}/rank{r}")`` (rng.py:26-28); global
        mini-batch m is the union of every rank's m-th local mini-batch of
        ``mini_batch_size`` samples, split by the global plan. All of the
        rank's micro-batches of the epoch stream as one sequence (cross-step
        prefetch). Returns the per-mini-batch statistics (resolved).
        """
        from .rng import named_stream
        x, y = _as_tensor(x), _as_tensor(y)
        n = x.shape[0]
        if n == 0:
            raise ValueError("dataset is empty")
        if n % mini_batch_size:
            raise ValueError("weak-scaling epochs need whole local mini-batches on every rank")
        on_device = x.device.type == "cuda"
        order = (named_stream(seed, f"shuffle/epoch{epoch_index}/rank{self.rank}").permutation(n) if shuffle
                 else np.arange(n))
        order_dev = torch.from_numpy(order.astype(np.int64)).to(x.device) if (on_device and shuffle) else None
        plan = weak_scaling_plan(mini_batch_size, micro_batch_size, self.world)
        block = partition_micro_batches(plan, self.world)[self.rank]
        lo, _ = rank_samples(plan, block)
        jobs = []
        for start in range(0, n, mini_batch_size):
            for k in range(*block):
                a, b = plan.index_ranges[k]
                a, b = start + a - lo, start + b - lo
                if not shuffle:
                    jobs.append((None, a, b - a))
                elif on_device:
                    jobs.append((order_dev[a:b], 0, b - a))
                else:
                    jobs.append((order[a:b], 0, b - a))
        own = None
        if not on_device and streamer is None:
            streamer = own = make_streamer(x, y, micro_batch_size)
        out = []
        try:
            dest = _graph_dest(model, accumulator, loss_kind, autocast_dtype, loss_from_logits, dice_smoothing,
                               "fused")
            source = iter(_micro_source(x, y, jobs, staging, prefetch, streamer, dest))
            for _ in range(0, n, mini_batch_size):
                r = self._step(model, plan, block, source, normalization, loss_kind, optimizer_state, accumulator,
                               autocast_dtype, loss_from_logits, dice_smoothing, lr_for_step)
                out.append(r)
            for r in out:
                r.resolve()
        finally:
            if own is not None:
                own.close()
        return out

    def _step(self, model, plan, block, source, normalization, loss_kind, optimizer_state, acc, autocast_dtype,
              loss_from_logits, dice_smoothing, lr_for_step):
        """Consume this rank's micro-batches of one global mini-batch from `source`, exchange, step."""
        n_local = block[1] - block[0]
        acc.begin(n_local)
        ctx = torch.autocast("cuda", dtype=autocast_dtype) if autocast_dtype is not None else nullcontext()
        model.train()
        bn = None
        if self.bn_stats == "sequential" and self.world > 1:
            bn = self._bn.get(id(model))
            if bn is None:
                bn = self._bn[id(model)] = BNStatSync(model, self.dist, self.group)
            bn.snapshot()
        losses, factors, weights = [], [], []
        works = []
        plist = acc._plist
        cast_cache = weight_cast_cache(autocast_dtype)    # one weight cast per mini-batch (engine.py)
        cast_cache.__enter__()
        try:
            self._micro_loop(model, plan, block, source, normalization, loss_kind, acc, ctx, loss_from_logits,
                             dice_smoothing, n_local, losses, factors, weights, works, plist, autocast_dtype)
        finally:
            cast_cache.__exit__(None, None, None)
        return self._exchange_and_step(model, plan, block, optimizer_state, acc, n_local, losses, factors, weights,
                                       works, bn, lr_for_step)

    def _micro_loop(self, model, plan, block, source, normalization, loss_kind, acc, ctx, loss_from_logits,
                    dice_smoothing, n_local, losses, factors, weights, works, plist, autocast_dtype=None):
        for j in range(n_local):
            xk, yk = next(source)
            k = block[0] + j
            f = normalization_factor(plan, k, normalization)
            last = j == n_local - 1
            if not last:
                # every micro-batch but the rank's last replays the captured micro step (engine.py); the
                # last interleaves K1 buckets and all-reduces with its backward through hooks: eager
                g = _graph_for(model, acc, loss_kind, xk, yk, autocast_dtype, loss_from_logits, dice_smoothing,
                               "fused", False, headroom=2.3)
                if g is not None:
                    loss = g.replay(xk, yk)
                    losses.append(loss.detach().float().clone())   # the static loss is overwritten next replay
                    factors.append(f)
                    weights.append(float(plan.sizes[k]))
                    acc.add_pointer_table(g.ptrs, f, loss=loss, loss_factor=f, loss_weight=plan.sizes[k])
                    continue
            with ctx:
                out = model(xk)
                loss = compute_loss(loss_kind, out, yk, from_logits=loss_from_logits, dice_smoothing=dice_smoothing)
            losses.append(loss.detach().float())
            factors.append(f)
            weights.append(float(plan.sizes[k]))
            if not last:
                loss.backward()
                acc.add_module_grads(f, loss=loss, loss_factor=f, loss_weight=plan.sizes[k])
                continue
            if self.peer is not None:
                loss.backward()
                acc.add_allreduce(self.peer, f, loss=loss, loss_factor=f, loss_weight=plan.sizes[k])
                continue
            # last micro-batch: bucket-wise K1 + async all-reduce, overlapped with the rest of backward.
            # All-reduces are issued strictly in self.buckets order (a bucket that completes early waits
            # for its predecessors), so every rank — including one without a micro-batch — issues the
            # identical collective sequence.
            pending = {b: s1 - s0 for b, (s0, s1) in enumerate(self.buckets)}
            done = set()
            nxt = [0]
            handles = []

            def launch_ready():
                while nxt[0] in done:
                    s0, s1 = self.buckets[nxt[0]]
                    works.append(self.dist.all_reduce(self._slice(acc, s0, s1), group=self.group, async_op=True))
                    nxt[0] += 1

            def hook(p, _idx={id(q): i for i, q in enumerate(plist)}):
                s = _idx[id(p)]
                b = self._seg_bucket[s]
                pending[b] -= 1
                if pending[b] == 0:
                    s0, s1 = self.buckets[b]
                    acc.add_tensors([plist[i].grad for i in range(s0, s1)], f, seg_begin=s0, last=False,
                                    loss=loss if s0 == 0 else None, loss_factor=f, loss_weight=plan.sizes[k])
                    for i in range(s0, s1):
                        plist[i].grad = None
                    done.add(b)
                    launch_ready()

            for p in plist:
                handles.append(p.register_post_accumulate_grad_hook(hook))
            try:
                loss.backward()
            finally:
                for h in handles:
                    h.remove()
            if any(v != 0 for v in pending.values()):
                from .errors import AccumulatorOverflowError
                raise AccumulatorOverflowError("a parameter received no gradient on the last micro-batch")
            launch_ready()

    def _exchange_and_step(self, model, plan, block, optimizer_state, acc, n_local, losses, factors, weights,
                           works, bn, lr_for_step):
        for wk in works:
            wk.wait()
        if n_local == 0:
            acc.begin(0)
            if self.peer is not None:     # no micro-batch here: still take part in the exchange
                acc.add_allreduce(self.peer, 1.0, from_module=False)
            else:                         # same bucket sequence as the working ranks, zeros contributed
                acc._materialize()
                for s0, s1 in self.buckets:
                    self.dist.all_reduce(self._slice(acc, s0, s1), group=self.group)
        # grad norm of the REDUCED sum (the optimizer's guard) + the global loss record
        stats_dev = acc.finalize(plan.n_b, recompute_norm=True)
        rec = torch.zeros(1 + 2 * plan.n_s_mu, dtype=torch.float64, device=acc.flat.device)
        if losses:
            lv = torch.stack(losses).double()
            k0 = block[0]
            wv = torch.tensor(weights, dtype=torch.float64, device=lv.device)
            fv = torch.tensor(factors, dtype=torch.float64, device=lv.device)
            rec[0] = (wv * lv).sum() / plan.n_b
            rec[1 + k0:1 + k0 + n_local] = lv
            rec[1 + plan.n_s_mu + k0:1 + plan.n_s_mu + k0 + n_local] = lv * fv
        self.dist.all_reduce(rec, group=self.group)
        if bn is not None:
            bn.merge(block, plan.n_s_mu)
        total = acc.as_gradient_set()
        res = _Result(rec, stats_dev[0], plan.n_s_mu)
        res.resolve()        # NonFiniteError before the update on every rank (reference: nn.py:578-579)
        if lr_for_step is not None:
            optimizer_state.lr = lr_for_step(optimizer_state.step_count)
        apply_update(self.params, total, optimizer_state)
        res.step_count = optimizer_state.step_count
        return res
