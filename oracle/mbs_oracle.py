"""CPU oracle for the Micro-Batch Streaming hot path — TEST INFRASTRUCTURE ONLY.

This module is a float64 NumPy restatement of the reference package
``mbstream`` (``/root/reference/pkg/src/mbstream``) restricted to the hot path
named by ``BASELINE.json.north_star``: the micro-batch plan, the epoch
shuffle/gather, the loss normalisation, the gradient accumulator, the grad-norm,
the optimizer step and the auto-sizer. Every function cites the reference
``file:line`` it restates.

Rules:

* Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
  ``--impl reference`` leg may import this module, and only as the checker or
  the CPU baseline. The product package ``paper_2110_12484_b200`` never imports
  it; the product fails loudly when its CUDA extension is missing.
* Parity is PINNED: ``tests/test_oracle_golden.py`` checks this module against
  fixtures produced by the real reference (``tests/golden/make_golden.py``
  imports ``/root/reference/pkg/src`` in the build container) and, when the
  reference tree is present, against the reference directly.

The one third-party algorithm on the path is NumPy's Philox bit generator plus
``Generator.permutation`` (numpy >= 1.24 per ``pkg/pyproject.toml:10``; 2.3.5
here). It is used as-is, exactly as ``rng.py:26-28`` does.
"""

from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass, field

import numpy as np

NORMALIZATION_MODES = ("paper_faithful", "exact_weighted", "off")  # engine.py:34
PROB_CLAMP = 1e-12  # losses.py:17


# --------------------------------------------------------------------------
# rng.py — named counter-based streams
# --------------------------------------------------------------------------

def stream_key(seed: int, name: str) -> int:
    """rng.py:18-23 — Philox key = little-endian int of SHA-256(f"{seed}/{name}")[:16]."""
    if seed < 0:
        raise ValueError("seed must be non-negative")
    digest = hashlib.sha256(f"{seed}/{name}".encode("utf-8")).digest()
    return int.from_bytes(digest[:16], "little")


def named_stream(seed: int, name: str) -> np.random.Generator:
    """rng.py:26-28."""
    return np.random.Generator(np.random.Philox(key=stream_key(seed, name)))


def epoch_order(n: int, seed: int, epoch_index: int, shuffle: bool = True) -> np.ndarray:
    """engine.py:300-303 — the per-epoch sample order."""
    if shuffle:
        return named_stream(seed, f"shuffle/epoch{epoch_index}").permutation(n)
    return np.arange(n)


# --------------------------------------------------------------------------
# engine.py — plan, normalisation, accumulator, micro-batch slicing
# --------------------------------------------------------------------------

@dataclass(frozen=True)
class Plan:
    """engine.py:37-53 (MicroBatchPlan)."""

    n_b: int
    n_mu: int
    n_s_mu: int
    sizes: tuple
    index_ranges: tuple


def plan_split(n_b: int, n_mu: int) -> Plan:
    """engine.py:56-78."""
    if n_b < 1 or n_mu < 1:
        raise ValueError("batch sizes must be positive")
    if n_b < n_mu:                       # engine.py:66-67
        n_mu = n_b
    n_s_mu = math.ceil(n_b / n_mu)       # engine.py:68
    sizes = [n_mu] * (n_b // n_mu)       # engine.py:69
    if n_b % n_mu:                       # engine.py:70-71
        sizes.append(n_b % n_mu)
    ranges, start = [], 0
    for s in sizes:                      # engine.py:72-76
        ranges.append((start, start + s))
        start += s
    return Plan(n_b, n_mu, n_s_mu, tuple(sizes), tuple(ranges))


def normalization_factor(plan: Plan, k: int, mode: str) -> float:
    """engine.py:81-91."""
    if not 0 <= k < plan.n_s_mu:
        raise ValueError("micro-batch index out of range")
    if mode == "paper_faithful":
        return 1.0 / plan.n_s_mu
    if mode == "exact_weighted":
        return plan.sizes[k] / plan.n_b
    if mode == "off":
        return 1.0
    raise ValueError(f"unknown normalization mode {mode!r}")


class Accumulator:
    """engine.py:100-131 — fp64 per-parameter running sums in plan order."""

    def __init__(self, shapes: dict, expected: int | None = None):
        self.sums = {n: np.zeros(s) for n, s in shapes.items()}
        self.micro_batches_seen = 0
        self.expected = expected

    def begin(self, expected: int) -> None:          # engine.py:110-115
        for a in self.sums.values():
            a.fill(0.0)
        self.micro_batches_seen = 0
        self.expected = expected

    def add(self, grads: dict) -> None:              # engine.py:117-128
        if self.expected is not None and self.micro_batches_seen >= self.expected:
            raise OverflowError("accumulator overflow")
        if set(grads) != set(self.sums):
            raise KeyError("gradient keys do not match accumulator parameters")
        for name, g in grads.items():
            self.sums[name] += np.asarray(g, dtype=np.float64)
        self.micro_batches_seen += 1


def micro_batch_rows(order: np.ndarray, mini_start: int, plan: Plan, k: int) -> np.ndarray:
    """engine.py:310-311 then 149-151: dataset rows of micro k of the mini-batch at mini_start."""
    lo, hi = plan.index_ranges[k]
    return np.asarray(order[mini_start: mini_start + plan.n_b])[lo:hi]


def stage_micro(x: np.ndarray, rows: np.ndarray) -> np.ndarray:
    """engine.py:311 + 150 — ``np.ascontiguousarray(x[idx][lo:hi])`` (bytes unchanged)."""
    return np.ascontiguousarray(x[rows])


def mini_loss(sizes, losses_raw, n_b: int) -> float:
    """engine.py:221 — exact sample-weighted mean of raw micro losses."""
    return float(sum(s * v for s, v in zip(sizes, losses_raw)) / n_b)


# --------------------------------------------------------------------------
# tensor.py — grad norm
# --------------------------------------------------------------------------

def l2_norm(grads: dict) -> float:
    """tensor.py:126-130 — sqrt of the sequential sum of per-parameter dot products."""
    total = 0.0
    for g in grads.values():
        g = np.asarray(g, dtype=np.float64).ravel()
        total += float(np.dot(g, g))
    return float(np.sqrt(total))


# --------------------------------------------------------------------------
# optim.py — SGD momentum / Adam with coupled weight decay
# --------------------------------------------------------------------------

@dataclass
class OptState:
    """optim.py:17-37."""

    kind: str
    lr: float
    momentum: float = 0.0
    weight_decay: float = 0.0
    adam_beta1: float = 0.9
    adam_beta2: float = 0.999
    adam_eps: float = 1e-8
    step_count: int = 0
    velocity: dict = field(default_factory=dict)
    first_moment: dict = field(default_factory=dict)
    second_moment: dict = field(default_factory=dict)


def sgd_step(params: dict, grads: dict, st: OptState) -> None:
    """optim.py:52-65 (mutates params in place)."""
    for name, grad in grads.items():
        w = params[name]
        g = grad + st.weight_decay * w if st.weight_decay else np.asarray(grad, np.float64)
        v = st.velocity.get(name)
        if v is None:
            v = np.zeros_like(w)
            st.velocity[name] = v
        v *= st.momentum
        v += g
        w -= st.lr * v
    st.step_count += 1


def adam_step(params: dict, grads: dict, st: OptState) -> None:
    """optim.py:68-93 (mutates params in place)."""
    t = st.step_count + 1
    b1, b2 = st.adam_beta1, st.adam_beta2
    c1, c2 = 1.0 - b1 ** t, 1.0 - b2 ** t
    for name, grad in grads.items():
        w = params[name]
        g = grad + st.weight_decay * w if st.weight_decay else np.asarray(grad, np.float64)
        m = st.first_moment.get(name)
        if m is None:
            m = np.zeros_like(w)
            v = np.zeros_like(w)
            st.first_moment[name] = m
            st.second_moment[name] = v
        else:
            v = st.second_moment[name]
        m *= b1
        m += (1.0 - b1) * g
        v *= b2
        v += (1.0 - b2) * g * g
        w -= st.lr * (m / c1) / (np.sqrt(v / c2) + st.adam_eps)
    st.step_count = t


def apply_update(params: dict, grads: dict, st: OptState) -> None:
    """optim.py:96-101."""
    (sgd_step if st.kind == "sgd" else adam_step)(params, grads, st)


def linear_lr(initial_lr: float, step: int, total_steps: int) -> float:
    """optim.py:104-110."""
    if total_steps <= 0:
        raise ValueError("total_steps must be positive")
    if not 0 <= step <= total_steps:
        raise ValueError("step out of range")
    return max(0.0, initial_lr * (1.0 - step / total_steps))


# --------------------------------------------------------------------------
# losses.py — mean-reduced losses: (value, dL/doutput)
# --------------------------------------------------------------------------

def _sigmoid(z):
    """losses.py:64-69."""
    out = np.empty_like(z)
    pos = z >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-z[pos]))
    ez = np.exp(z[~pos])
    out[~pos] = ez / (1.0 + ez)
    return out


def _mse(o, t):                      # losses.py:72-75
    d = o - t
    return float(np.mean(d * d)), 2.0 * d / d.size


def _cross_entropy(logits, classes):  # losses.py:78-87
    n = logits.shape[0]
    sh = logits - logits.max(axis=1, keepdims=True)
    lp = sh - np.log(np.exp(sh).sum(axis=1, keepdims=True))
    idx = np.arange(n)
    val = float(-lp[idx, classes].mean())
    g = np.exp(lp)
    g[idx, classes] -= 1.0
    return val, g / n


def _bce_probs(p, t):                 # losses.py:90-95
    c = np.clip(p, PROB_CLAMP, 1.0 - PROB_CLAMP)
    val = float(-np.mean(t * np.log(c) + (1.0 - t) * np.log1p(-c)))
    g = (c - t) / (c * (1.0 - c)) / p.size
    g[p != c] = 0.0
    return val, g


def _bce_logits(z, t):                # losses.py:98-102
    val = float(np.mean(np.maximum(z, 0.0) - z * t + np.log1p(np.exp(-np.abs(z)))))
    return val, (_sigmoid(z) - t) / z.size


def _dice_soft(p, t, s):              # losses.py:105-114
    n = p.shape[0]
    pf, gf = p.reshape(n, -1), t.reshape(n, -1)
    num = 2.0 * (pf * gf).sum(axis=1) + s
    den = pf.sum(axis=1) + gf.sum(axis=1) + s
    val = float(np.mean(1.0 - num / den))
    g = -(2.0 * gf * den[:, None] - num[:, None]) / (den[:, None] ** 2) / n
    return val, g.reshape(p.shape)


def compute_loss(kind: str, out, target, from_logits: bool = True, dice_smoothing: float = 1.0):
    """losses.py:184-207 (+ mean_loss 122-156): returns (value, dL/dout)."""
    out = np.asarray(out, dtype=np.float64)
    if kind == "mse":
        return _mse(out, np.asarray(target, np.float64))
    if kind == "cross_entropy":
        return _cross_entropy(out, np.asarray(target).astype(np.int64))
    if kind == "bce":
        t = np.asarray(target, np.float64)
        return _bce_logits(out, t) if from_logits else _bce_probs(out, t)
    if kind == "bce_dice":
        t = np.asarray(target, np.float64)
        if from_logits:
            p = _sigmoid(out)
            bv, bg = _bce_logits(out, t)
            dv, dg = _dice_soft(p, t, dice_smoothing)
            return bv + dv, bg + dg * p * (1.0 - p)
        bv, bg = _bce_probs(out, t)
        dv, dg = _dice_soft(out, t, dice_smoothing)
        return bv + dv, bg + dg
    raise ValueError(f"unknown loss kind {kind!r}")


# --------------------------------------------------------------------------
# memory.py — auto-sizing rule
# --------------------------------------------------------------------------

def fit_micro_batch(capacity_bytes: int, resident_bytes: int, per_sample_bytes: int) -> int:
    """memory.py:88-101 — n = (capacity - resident) // per_sample, >= 1 or raise."""
    n = (capacity_bytes - resident_bytes) // per_sample_bytes
    if n < 1:
        raise MemoryError("model does not fit")
    return int(n)


# --------------------------------------------------------------------------
# streaming.py — two-slot schedule (the ideal the real streamer is held to)
# --------------------------------------------------------------------------

def simulate_stream(transfer, fwd, bwd, update: float, overlap: bool):
    """streaming.py:78-111 given per-micro durations; returns (makespan, events)."""
    n = len(transfer)
    ev = []
    if not overlap:
        t = 0.0
        for k in range(n):
            ev.append(("transfer", k, t, t + transfer[k])); t += transfer[k]
            ev.append(("forward", k, t, t + fwd[k])); t += fwd[k]
            ev.append(("backward", k, t, t + bwd[k])); t += bwd[k]
        ev.append(("update", -1, t, t + update))
        return t + update, ev
    te, ce = [0.0] * n, [0.0] * n
    for k in range(n):
        t0 = max(te[k - 1] if k >= 1 else 0.0, ce[k - 2] if k >= 2 else 0.0)
        te[k] = t0 + transfer[k]
        ev.append(("transfer", k, t0, te[k]))
        c0 = max(te[k], ce[k - 1] if k >= 1 else 0.0)
        ev.append(("forward", k, c0, c0 + fwd[k]))
        ce[k] = c0 + fwd[k] + bwd[k]
        ev.append(("backward", k, c0 + fwd[k], ce[k]))
    u0 = ce[n - 1]
    ev.append(("update", -1, u0, u0 + update))
    return u0 + update, ev


# --------------------------------------------------------------------------
# engine.py:179-230 / 233-261 / 276-335 — the loops, with a pluggable model
# --------------------------------------------------------------------------

def mini_batch_gradient(grad_fn, shapes: dict, x, y, plan: Plan, normalization: str,
                        acc: Accumulator | None = None):
    """engine.py:179-230.

    ``grad_fn(xk, yk, seed) -> (loss_value, grads_dict, out)`` is the model's
    forward + loss + backward with the backward seeded by ``seed`` exactly as
    ``backward(tape, factor)`` (engine.py:214-215 -> nn.py:596).
    """
    if x.shape[0] != plan.n_b:
        raise ValueError("batch/plan size mismatch")
    acc = acc if acc is not None else Accumulator(shapes)
    acc.begin(plan.n_s_mu)
    raw, normed, outs = [], [], []
    for k in range(plan.n_s_mu):
        lo, hi = plan.index_ranges[k]
        xk, yk = np.ascontiguousarray(x[lo:hi]), np.ascontiguousarray(y[lo:hi])
        f = normalization_factor(plan, k, normalization)
        val, grads, out = grad_fn(xk, yk, f)
        acc.add(grads)
        raw.append(val)
        normed.append(val * f)
        outs.append(out)
    total = dict(acc.sums)
    stats = dict(losses_raw=raw, losses_normalized=normed,
                 loss=mini_loss(plan.sizes, raw, plan.n_b), grad_norm=l2_norm(total),
                 n_micro=plan.n_s_mu, outputs=np.concatenate(outs, axis=0))
    return total, stats


def train_mini_batch(grad_fn, params: dict, x, y, plan: Plan, normalization: str,
                     st: OptState, acc: Accumulator | None = None, lr_for_step=None):
    """engine.py:233-261."""
    total, stats = mini_batch_gradient(grad_fn, {n: p.shape for n, p in params.items()},
                                       x, y, plan, normalization, acc)
    if lr_for_step is not None:
        st.lr = lr_for_step(st.step_count)
    apply_update(params, total, st)
    stats["step_count"] = st.step_count
    return stats


def train_epoch(grad_fn, params: dict, x, y, *, mini_batch_size: int, micro_batch_size,
                normalization: str, st: OptState, seed: int, epoch_index: int,
                shuffle: bool = True, lr_for_step=None):
    """engine.py:276-335 (metrics omitted)."""
    n = x.shape[0]
    if n == 0:
        raise ValueError("dataset is empty")
    order = epoch_order(n, seed, epoch_index, shuffle)
    acc = Accumulator({k: v.shape for k, v in params.items()})
    losses, sizes, all_stats = [], [], []
    for start in range(0, n, mini_batch_size):
        idx = order[start:start + mini_batch_size]
        n_mu = micro_batch_size if micro_batch_size is not None else len(idx)
        plan = plan_split(len(idx), n_mu)
        s = train_mini_batch(grad_fn, params, x[idx], y[idx], plan, normalization, st, acc,
                             lr_for_step)
        losses.append(s["loss"])
        sizes.append(len(idx))
        all_stats.append(s)
    return dict(mini_losses=losses, mini_sizes=sizes,
                mean_loss=float(np.dot(losses, sizes) / n), step_count=st.step_count,
                mini_stats=all_stats)
