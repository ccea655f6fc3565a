"""Generate golden fixtures from the REAL reference package (build container only).

Run:  python tests/golden/make_golden.py
Needs ``/root/reference/pkg/src`` (the reference ``mbstream`` namespace package,
pure NumPy). Writes small JSON / NPZ fixtures next to this script; they are
committed, so the tests and the GPU box never need the reference tree.

Everything here calls the reference's own public functions:
``plan_split`` (engine.py:56), ``normalization_factor`` (engine.py:81),
``stream_key`` / ``named_stream`` (rng.py:18-28), ``GradientAccumulator``
(engine.py:100), ``GradientSet.l2_norm`` (tensor.py:126), ``apply_update``
(optim.py:96), ``build_model`` / ``forward`` / ``backward`` (nn.py),
``mini_batch_gradient`` / ``train_mini_batch`` / ``train_epoch``
(engine.py:179/233/276), ``fit_micro_batch`` (memory.py:88) and
``simulate_stream`` (streaming.py:78).
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

from mbstream import engine, memory, nn, optim, rng, streaming  # noqa: E402
from mbstream.tensor import GradientSet, ParameterSet, Tensor  # noqa: E402


def _spec_to_json(spec):
    out = []
    for e in spec:
        d = {"type": type(e).__name__}
        d.update(e.__dict__)
        out.append(d)
    return out


def gen_plans():
    cases = [(16, 8), (10, 8), (4, 8), (64, 8), (1024, 128), (256, 48), (33, 16), (1, 1),
             (7, 3), (1, 5), (5, 1), (300032, 128), (299999, 128), (100, 7), (48, 48), (49, 48)]
    rs = np.random.RandomState(0)
    for _ in range(60):
        cases.append((int(rs.randint(1, 3000)), int(rs.randint(1, 400))))
    plans = []
    for n_b, n_mu in cases:
        p = engine.plan_split(n_b, n_mu)
        factors = {m: [engine.normalization_factor(p, k, m).hex() for k in range(p.n_s_mu)]
                   for m in engine.NORMALIZATION_MODES} if p.n_s_mu <= 64 else None
        plans.append({"n_b": n_b, "n_mu_in": n_mu, "n_mu": p.n_mu, "n_s_mu": p.n_s_mu,
                      "sizes": list(p.sizes) if p.n_s_mu <= 64 else None,
                      "sizes_head_tail": [p.sizes[0], p.sizes[-1]],
                      "ranges_last": list(p.index_ranges[-1]), "factors_hex": factors})
    errors = []
    for n_b, n_mu in [(0, 1), (1, 0), (-3, 2), (4, -1)]:
        try:
            engine.plan_split(n_b, n_mu)
            errors.append([n_b, n_mu, None])
        except ValueError:
            errors.append([n_b, n_mu, "ValueError"])
    return {"plans": plans, "errors": errors}


def gen_rng():
    keys = {f"{s}|{n}": hex(rng.stream_key(s, n))
            for s in (0, 1, 2, 7, 12345)
            for n in ("shuffle/epoch0", "shuffle/epoch1", "shuffle/epoch3", "data/x", "init/layer0.weight")}
    perms = {}
    for seed in (0, 1, 2):
        for epoch in (0, 1, 2):
            for n in (1, 10, 33, 100, 1024):
                perms[f"{seed}|{epoch}|{n}"] = rng.named_stream(seed, f"shuffle/epoch{epoch}").permutation(n).tolist()
    return {"keys": keys, "perms": perms}


def gen_accum_optim():
    """Accumulator + grad norm + SGD/Adam over fp32-representable random grads."""
    rs = np.random.RandomState(1)
    shapes = {"a.weight": (7, 5), "a.bias": (5,), "b.weight": (3, 2, 3, 3), "b.bias": (3,)}
    params0 = {n: rs.randn(*s).astype(np.float32).astype(np.float64) for n, s in shapes.items()}
    n_micro = 3
    micro = [{n: rs.randn(*s).astype(np.float32).astype(np.float64) for n, s in shapes.items()}
             for _ in range(n_micro)]
    ps = ParameterSet((n, Tensor(v.copy(), grad_required=True)) for n, v in params0.items())
    acc = engine.GradientAccumulator(ps)
    acc.begin(n_micro)
    for g in micro:
        engine.accumulate(acc, GradientSet(dict(g)))
    total = {n: a.copy() for n, a in acc.as_gradient_set().items()}
    norm = acc.as_gradient_set().l2_norm()
    overflow = False
    try:
        acc.add(GradientSet(dict(micro[0])))
    except Exception as exc:  # AccumulatorOverflowError
        overflow = type(exc).__name__
    out = {"shapes": {n: list(s) for n, s in shapes.items()}, "n_micro": n_micro,
           "norm": norm.hex(), "overflow_error": overflow}
    arrays = {f"p0/{n}": v for n, v in params0.items()}
    for k, g in enumerate(micro):
        for n, v in g.items():
            arrays[f"g{k}/{n}"] = v
    for n, v in total.items():
        arrays[f"total/{n}"] = v
    for kind, st in (("sgd", optim.sgd_state(0.1, 0.9, 5e-4)),
                     ("sgd_nomom", optim.OptimizerState(kind="sgd", lr=0.05)),
                     ("adam", optim.adam_state(0.01, 5e-4)),
                     ("adam_nowd", optim.adam_state(0.003, 0.0, 0.8, 0.99, 1e-6))):
        p = ParameterSet((n, Tensor(v.copy(), grad_required=True)) for n, v in params0.items())
        for step in range(3):
            optim.apply_update(p, GradientSet({n: micro[step][n] for n in shapes}), st)
            for n in shapes:
                arrays[f"{kind}/step{step}/{n}"] = p[n].data.copy()
        out[f"{kind}_step_count"] = st.step_count
    return out, arrays


MODELS = {
    # name: (spec, input_shape, loss_kind, target kind, n_b, n_mu, optimizer)
    "convbn_ce": ([nn.Conv2d(3, 4, 3, 1, 1), nn.BatchNorm(4), nn.Relu(), nn.MaxPool2d(2),
                   nn.Flatten(), nn.Dense(64, 5)], (3, 8, 8), "cross_entropy", "classes5",
                  10, 4, "sgd"),
    "conv_ce": ([nn.Conv2d(3, 6, 3, 1, 1), nn.Relu(), nn.MaxPool2d(2), nn.Conv2d(6, 4, 3, 1, 0),
                 nn.Relu(), nn.Flatten(), nn.Dense(16, 5)], (3, 8, 8), "cross_entropy", "classes5",
                16, 4, "sgd"),
    "mlp_mse": ([nn.Dense(6, 8), nn.Relu(), nn.Dense(8, 3)], (6,), "mse", "dense3",
                12, 5, "adam"),
    "seg_bce_dice": ([nn.Conv2d(2, 4, 3, 1, 1), nn.Relu(), nn.Conv2d(4, 1, 3, 1, 1)], (2, 6, 6),
                     "bce_dice", "mask", 7, 3, "adam"),
    # a 1x1 feature map into BatchNorm with a 1-sample tail micro-batch (9/4 -> [4, 4, 1]): one value per
    # channel, legal in the reference (eps-guarded; biased running variance nn.py:329-332)
    "bn1_tail": ([nn.Conv2d(3, 4, 4, 1, 0), nn.BatchNorm(4), nn.Relu(), nn.Flatten(), nn.Dense(4, 5)],
                 (3, 4, 4), "cross_entropy", "classes5", 9, 4, "sgd"),
}


def _targets(kind, n, seed):
    g = rng.named_stream(seed, "data/y")
    if kind == "classes5":
        return g.integers(0, 5, size=n)
    if kind == "dense3":
        return g.standard_normal((n, 3))
    if kind == "mask":
        return (g.random((n, 1, 6, 6)) < 0.5).astype(np.float64)
    raise ValueError(kind)


def _state(kind):
    return optim.sgd_state(0.01, 0.9, 5e-4) if kind == "sgd" else optim.adam_state(0.01, 5e-4)


def gen_e2e():
    meta, arrays = {}, {}
    for name, (spec, in_shape, loss_kind, tkind, n_b, n_mu, okind) in MODELS.items():
        seed = 3
        params0, model = nn.build_model(spec, in_shape, seed)
        x = rng.named_stream(seed, "data/x").standard_normal((2 * n_b,) + in_shape)
        y = _targets(tkind, 2 * n_b, seed)
        arrays[f"{name}/x"] = x
        arrays[f"{name}/y"] = y
        for n, t in params0.items():
            arrays[f"{name}/p0/{n}"] = t.data.copy()
        meta[name] = {"spec": _spec_to_json(spec), "input_shape": list(in_shape),
                      "loss_kind": loss_kind, "n_b": n_b, "n_mu": n_mu, "optimizer": okind,
                      "param_names": params0.names(), "modes": {}}
        plan = engine.plan_split(n_b, n_mu)
        for mode in engine.NORMALIZATION_MODES:
            params = params0.copy()
            model.reset_state()
            st = _state(okind)
            acc = engine.GradientAccumulator(params)
            mstats = []
            for mb in range(2):
                xb, yb = x[mb * n_b:(mb + 1) * n_b], y[mb * n_b:(mb + 1) * n_b]
                if mb == 0:
                    total, s0 = engine.mini_batch_gradient(model, params, xb, yb, plan, mode,
                                                           loss_kind)
                    for n, g in total.items():
                        arrays[f"{name}/{mode}/grad0/{n}"] = g.copy()
                    model.reset_state()
                params, s = engine.train_mini_batch(model, params, (xb, yb), plan, mode,
                                                    loss_kind, st, accumulator=acc)
                mstats.append({"losses_raw": [v.hex() for v in s.losses_raw],
                               "losses_normalized": [v.hex() for v in s.losses_normalized],
                               "loss": s.loss.hex(), "grad_norm": s.grad_norm.hex(),
                               "n_micro": s.n_micro, "step_count": s.step_count})
                arrays[f"{name}/{mode}/out{mb}"] = s.outputs.copy()
                for n, t in params.items():
                    arrays[f"{name}/{mode}/p{mb + 1}/{n}"] = t.data.copy()
            meta[name]["modes"][mode] = mstats
        # full-batch (no-MBS) gradient: plan_split(n_b, n_b)
        model.reset_state()
        full, sf = engine.mini_batch_gradient(model, params0.copy(), x[:n_b], y[:n_b],
                                              engine.plan_split(n_b, n_b), "paper_faithful",
                                              loss_kind)
        for n, g in full.items():
            arrays[f"{name}/full/grad0/{n}"] = g.copy()
    return meta, arrays


def gen_epoch():
    spec, in_shape = MODELS["conv_ce"][0], (3, 8, 8)
    seed = 5
    params, model = nn.build_model(spec, in_shape, seed)
    n = 33
    x = rng.named_stream(seed, "data/x").standard_normal((n,) + in_shape)
    y = rng.named_stream(seed, "data/y").integers(0, 5, size=n)
    arrays = {"x": x, "y": y}
    for nme, t in params.items():
        arrays[f"p0/{nme}"] = t.data.copy()
    st = optim.sgd_state(0.05, 0.9, 5e-4)
    meta = {"spec": _spec_to_json(spec), "input_shape": list(in_shape), "n": n,
            "mini": 16, "micro": 8, "seed": seed, "epochs": []}
    for epoch in range(2):
        es = engine.train_epoch(model, params, x, y, mini_batch_size=16, micro_batch_size=8,
                                normalization="exact_weighted", loss_kind="cross_entropy",
                                optimizer_state=st, seed=seed, epoch_index=epoch,
                                lr_for_step=lambda s: optim.linear_lr(0.05, s, 10),
                                keep_mini_stats=True)
        meta["epochs"].append({"mini_losses": [v.hex() for v in es.mini_losses],
                               "mean_loss": es.mean_loss.hex(), "mini_sizes": es.mini_sizes,
                               "step_count": es.step_count,
                               "n_micro": [s.n_micro for s in es.mini_stats]})
        for nme, t in params.items():
            arrays[f"e{epoch}/{nme}"] = t.data.copy()
    return meta, arrays


def gen_epoch_metrics():
    """train_epoch(metric_fn=...) (engine.py:276-335, metric at engine.py:323-324): accuracy on a classifier and
    iou / dice (losses.py:239-259, MaskPair of sigmoid(logits) and the mask) on a segmenter, two epochs each."""
    from mbstream import losses
    meta, arrays = {}, {}
    cases = {
        "conv_ce": (MODELS["conv_ce"][0], (3, 8, 8), "cross_entropy", "classes5", 37, 16, 8, "sgd",
                    lambda o, t: losses.accuracy(o, t)),
        "seg_bce_dice": (MODELS["seg_bce_dice"][0], (2, 6, 6), "bce_dice", "mask", 21, 8, 3, "adam",
                         lambda o, t: losses.iou(losses.MaskPair(1.0 / (1.0 + np.exp(-o)), t))),
    }
    for name, (spec, in_shape, loss_kind, tkind, n, mini, micro, okind, metric) in cases.items():
        seed = 9
        params, model = nn.build_model(spec, in_shape, seed)
        x = rng.named_stream(seed, "data/x").standard_normal((n,) + in_shape)
        y = _targets(tkind, n, seed)
        arrays[f"{name}/x"] = x
        arrays[f"{name}/y"] = y
        for nme, t in params.items():
            arrays[f"{name}/p0/{nme}"] = t.data.copy()
        st = _state(okind)
        m = {"spec": _spec_to_json(spec), "input_shape": list(in_shape), "loss_kind": loss_kind, "n": n,
             "mini": mini, "micro": micro, "seed": seed, "optimizer": okind, "epochs": []}
        for epoch in range(2):
            es = engine.train_epoch(model, params, x, y, mini_batch_size=mini, micro_batch_size=micro,
                                    normalization="exact_weighted", loss_kind=loss_kind, optimizer_state=st,
                                    seed=seed, epoch_index=epoch, metric_fn=metric)
            m["epochs"].append({"mini_metrics": es.mini_metrics, "mini_losses": [v.hex() for v in es.mini_losses],
                                "mini_sizes": es.mini_sizes, "step_count": es.step_count})
        meta[name] = m
    return meta, arrays


def gen_misc():
    out = {}
    # SPEC.md:343-344 scalar example y = w x
    spec = [nn.Dense(1, 1, bias=False)]
    params, model = nn.build_model(spec, (1,), 0)
    params["layer0.weight"].data[...] = 1.0
    x = np.array([[1.0], [2.0], [3.0], [4.0]])
    y = np.array([[2.0], [3.0], [5.0], [4.0]])
    plan = engine.plan_split(4, 2)
    for mode in ("paper_faithful", "off"):
        g, _ = engine.mini_batch_gradient(model, params, x, y, plan, mode, "mse")
        out[f"wx_{mode}"] = float(g["layer0.weight"].ravel()[0])
    # memory.py fit_micro_batch
    fits = []
    for cap, res, per in [(1000, 100, 300), (901, 0, 901), (900, 0, 901), (10**12, 5 * 10**9, 123457)]:
        b = memory.MemoryBudget(capacity_bytes=cap, param_bytes=res, data_bytes_per_sample=per)
        try:
            fits.append([cap, res, per, memory.fit_micro_batch(b)])
        except Exception as exc:
            fits.append([cap, res, per, type(exc).__name__])
    out["fit_micro_batch"] = fits
    # streaming.py simulate_stream, SPEC.md:433-434 style
    sims = []
    rs = np.random.RandomState(4)
    for _ in range(20):
        nb, nmu = int(rs.randint(1, 40)), int(rs.randint(1, 12))
        p = engine.plan_split(nb, nmu)
        c = streaming.CostModel(float(rs.rand() * 1e-3), float(rs.rand()), float(rs.rand()),
                                float(rs.rand()), float(rs.rand() * 0.1), float(rs.rand() * 0.1))
        bps = int(rs.randint(1, 1000))
        for ov in (False, True):
            s = streaming.simulate_stream(p, c, bps, overlap=ov)
            sims.append({"n_b": nb, "n_mu": nmu, "cost": list(c.__dict__.values()), "bps": bps,
                         "overlap": ov, "makespan": s.makespan.hex(),
                         "events": [[e.kind, e.index, e.start.hex(), e.end.hex()] for e in s.events]})
    out["simulate_stream"] = sims
    out["linear_lr"] = [[0.1, s, 10, optim.linear_lr(0.1, s, 10).hex()] for s in range(11)]
    return out


def main():
    with open(os.path.join(HERE, "plans.json"), "w") as f:
        json.dump(gen_plans(), f)
    with open(os.path.join(HERE, "rng.json"), "w") as f:
        json.dump(gen_rng(), f)
    meta, arrays = gen_accum_optim()
    with open(os.path.join(HERE, "accum_optim.json"), "w") as f:
        json.dump(meta, f, indent=1)
    np.savez_compressed(os.path.join(HERE, "accum_optim.npz"), **arrays)
    meta, arrays = gen_e2e()
    with open(os.path.join(HERE, "e2e.json"), "w") as f:
        json.dump(meta, f, indent=1)
    np.savez_compressed(os.path.join(HERE, "e2e.npz"), **arrays)
    meta, arrays = gen_epoch()
    with open(os.path.join(HERE, "epoch.json"), "w") as f:
        json.dump(meta, f, indent=1)
    np.savez_compressed(os.path.join(HERE, "epoch.npz"), **arrays)
    with open(os.path.join(HERE, "misc.json"), "w") as f:
        json.dump(gen_misc(), f)
    meta, arrays = gen_epoch_metrics()
    with open(os.path.join(HERE, "epoch_metrics.json"), "w") as f:
        json.dump(meta, f, indent=1)
    np.savez_compressed(os.path.join(HERE, "epoch_metrics.npz"), **arrays)
    meta, arrays = gen_losses_metrics()
    with open(os.path.join(HERE, "losses.json"), "w") as f:
        json.dump(meta, f, indent=1)
    np.savez_compressed(os.path.join(HERE, "losses.npz"), **arrays)
    print("golden fixtures written to", HERE)


def gen_losses_metrics():
    """Reference losses (value) and metrics on small random inputs (losses.py:72-263)."""
    from mbstream import losses
    rs = np.random.RandomState(8)
    out, arrays = {"losses": [], "metrics": []}, {}
    for i in range(6):
        n = int(rs.randint(1, 6))
        logits = rs.randn(n, 5) * 3
        cls = rs.randint(0, 5, size=n)
        z = rs.randn(n, 1, 4, 4) * 2
        t = (rs.rand(n, 1, 4, 4) < 0.5).astype(np.float64)
        d = rs.randn(n, 3)
        td = rs.randn(n, 3)
        p = 1.0 / (1.0 + np.exp(-z))
        for nm, v in (("logits", logits), ("cls", cls), ("z", z), ("t", t), ("d", d), ("td", td)):
            arrays[f"l{i}/{nm}"] = v
        rec = {"i": i,
               "mse": losses.compute_loss("mse", d, td).value.hex(),
               "cross_entropy": losses.compute_loss("cross_entropy", logits, cls).value.hex(),
               "bce_logits": losses.compute_loss("bce", z, t, from_logits=True).value.hex(),
               "bce_probs": losses.compute_loss("bce", p, t, from_logits=False).value.hex(),
               "bce_dice_logits": losses.compute_loss("bce_dice", z, t, from_logits=True).value.hex(),
               "bce_dice_probs": losses.compute_loss("bce_dice", p, t, from_logits=False).value.hex(),
               "accuracy": losses.accuracy(logits, cls)}
        pair = losses.MaskPair(p, t)
        for thr in (0.3, 0.5):
            for per in (False, True):
                rec[f"dice_{thr}_{per}"] = losses.dice_coefficient(pair, thr, per)
                rec[f"iou_{thr}_{per}"] = losses.iou(pair, thr, per)
        out["losses"].append(rec)
    # empty masks -> 1.0 (losses.py:224-233)
    z0 = np.zeros((2, 1, 3, 3))
    pair0 = losses.MaskPair(z0, z0)
    out["empty"] = [losses.dice_coefficient(pair0), losses.iou(pair0, per_image=True)]
    return out, arrays


if __name__ == "__main__":
    main()
