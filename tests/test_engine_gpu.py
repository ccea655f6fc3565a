"""End-to-end parity of the B200 MBS loop with the REAL reference (golden fixtures).

The fixtures hold the reference's own mini_batch_gradient / train_mini_batch /
train_epoch outputs (float64) for reference-expressible models
(tests/golden/make_golden.py). Tolerances follow SURVEY.md §8c's layered
contract: accumulated gradient rel-L2 <= 1e-5 for BN-free models (fp32 vs
fp64), <= 1e-4 with BatchNorm at micro-batch 4 (fp32 noise floor),
post-step weights rel-L2 <= 1e-5, per-micro losses rel 1e-6.
"""
import numpy as np
import pytest
import torch

import paper_2110_12484_b200 as mbs
from tests.golden_io import fhex, load_json, load_npz
from tests.gpu_util import rel_l2
from tests.refmodels import build_torch, load_ref_params, to_ref

pytestmark = pytest.mark.gpu

MODELS = ["convbn_ce", "conv_ce", "mlp_mse", "seg_bce_dice"]
GRAD_TOL = {"convbn_ce": 1e-4, "conv_ce": 1e-5, "mlp_mse": 1e-5, "seg_bce_dice": 1e-5}


def _model(meta, a, name, cuda):
    torch.manual_seed(0)
    mod = build_torch(meta["spec"], tuple(meta["input_shape"])).to(cuda)
    load_ref_params(mod, meta["spec"], {n: a[f"{name}/p0/{n}"] for n in meta["param_names"]})
    params = mbs.ParameterSet(mod)
    return mod, params


def _xy(a, name, meta, lo, hi, cuda, host=False):
    x = torch.from_numpy(a[f"{name}/x"][lo:hi])
    y = torch.from_numpy(a[f"{name}/y"][lo:hi])
    if meta["loss_kind"] != "cross_entropy":
        y = y.float()
    x = x.float()
    if host:
        return x.contiguous(), y.contiguous()
    return x.to(cuda), y.to(cuda)


def _opt(meta):
    return mbs.sgd_state(0.01, 0.9, 5e-4) if meta["optimizer"] == "sgd" else mbs.adam_state(0.01, 5e-4)


@pytest.mark.parametrize("name", MODELS)
@pytest.mark.parametrize("mode", ["paper_faithful", "exact_weighted", "off"])
def test_mini_batch_gradient_matches_reference(cuda, name, mode):
    meta = load_json("e2e.json")[name]
    a = load_npz("e2e.npz")
    mod, params = _model(meta, a, name, cuda)
    n_b = meta["n_b"]
    plan = mbs.plan_split(n_b, meta["n_mu"])
    x, y = _xy(a, name, meta, 0, n_b, cuda)
    total, stats = mbs.mini_batch_gradient(mod, params, x, y, plan, mode, meta["loss_kind"])
    got = to_ref(meta["spec"], {tn: total[tn] for tn in params.names()})
    flat_g = np.concatenate([got[k].ravel() for k in sorted(got)])
    flat_w = np.concatenate([a[f"{name}/{mode}/grad0/{k}"].ravel() for k in sorted(got)])
    assert rel_l2(flat_g, flat_w) <= GRAD_TOL[name]
    ms = meta["modes"][mode][0]
    np.testing.assert_allclose(stats.losses_raw, [fhex(v) for v in ms["losses_raw"]], rtol=1e-5)
    np.testing.assert_allclose(stats.losses_normalized, [fhex(v) for v in ms["losses_normalized"]], rtol=1e-5)
    assert stats.loss == pytest.approx(fhex(ms["loss"]), rel=1e-5)
    assert stats.grad_norm == pytest.approx(fhex(ms["grad_norm"]), rel=max(GRAD_TOL[name], 1e-5))
    assert stats.n_micro == ms["n_micro"]
    np.testing.assert_allclose(stats.outputs.double().cpu().numpy(), a[f"{name}/{mode}/out0"], rtol=1e-4,
                               atol=1e-5)


@pytest.mark.parametrize("name", MODELS)
def test_exact_weighted_equals_full_batch(cuda, name):
    """SPEC acceptance 3 analog: exact_weighted on a ragged split == full-batch gradient (BN-free)."""
    meta = load_json("e2e.json")[name]
    a = load_npz("e2e.npz")
    mod, params = _model(meta, a, name, cuda)
    n_b = meta["n_b"]
    x, y = _xy(a, name, meta, 0, n_b, cuda)
    total, _ = mbs.mini_batch_gradient(mod, params, x, y, mbs.plan_split(n_b, meta["n_mu"]), "exact_weighted",
                                       meta["loss_kind"])
    got = to_ref(meta["spec"], {tn: total[tn] for tn in params.names()})
    full = {k: a[f"{name}/full/grad0/{k}"] for k in got}
    err = rel_l2(np.concatenate([got[k].ravel() for k in sorted(got)]),
                 np.concatenate([full[k].ravel() for k in sorted(got)]))
    if name == "convbn_ce":
        assert err > 1e-3   # BN uses micro-batch statistics: discrepancy observable (SPEC acceptance 11)
    else:
        assert err <= 1e-5


@pytest.mark.parametrize("name", MODELS)
@pytest.mark.parametrize("mode", ["paper_faithful", "exact_weighted"])
def test_train_mini_batch_post_step_weights(cuda, name, mode):
    meta = load_json("e2e.json")[name]
    a = load_npz("e2e.npz")
    mod, params = _model(meta, a, name, cuda)
    n_b = meta["n_b"]
    plan = mbs.plan_split(n_b, meta["n_mu"])
    st = _opt(meta)
    acc = mbs.GradientAccumulator(params)
    for mb in range(2):
        x, y = _xy(a, name, meta, mb * n_b, (mb + 1) * n_b, cuda)
        _, stats = mbs.train_mini_batch(mod, params, (x, y), plan, mode, meta["loss_kind"], st, accumulator=acc)
        assert stats.step_count == mb + 1
        got = to_ref(meta["spec"], {tn: params[tn] for tn in params.names()})
        keys = sorted(got)
        err = rel_l2(np.concatenate([got[k].ravel() for k in keys]),
                     np.concatenate([a[f"{name}/{mode}/p{mb + 1}/{k}"].ravel() for k in keys]))
        assert err <= 1e-5, (mb, err)


@pytest.mark.parametrize("via", ["seed", "loss_scale"])
def test_normalize_via_equivalent(cuda, via):
    meta = load_json("e2e.json")["conv_ce"]
    a = load_npz("e2e.npz")
    outs = []
    for v in ("fused", via):
        mod, params = _model(meta, a, "conv_ce", cuda)
        x, y = _xy(a, "conv_ce", meta, 0, meta["n_b"], cuda)
        total, st = mbs.mini_batch_gradient(mod, params, x, y, mbs.plan_split(meta["n_b"], meta["n_mu"]),
                                            "paper_faithful", "cross_entropy", normalize_via=v)
        outs.append((total.flat.clone(), st.losses_normalized))
    assert rel_l2(outs[0][0].double().cpu().numpy(), outs[1][0].double().cpu().numpy()) <= 1e-6
    np.testing.assert_allclose(outs[0][1], outs[1][1], rtol=1e-12)


@pytest.mark.parametrize("prefetch", [False, True])
def test_host_streamed_equals_device_resident(cuda, prefetch):
    """Streaming from host memory changes nothing: bit-identical to the HBM-resident run."""
    meta = load_json("e2e.json")["seg_bce_dice"]
    a = load_npz("e2e.npz")
    res = []
    for host in (False, True):
        mod, params = _model(meta, a, "seg_bce_dice", cuda)
        x, y = _xy(a, "seg_bce_dice", meta, 0, meta["n_b"], cuda, host=host)
        total, st = mbs.mini_batch_gradient(mod, params, x, y, mbs.plan_split(meta["n_b"], meta["n_mu"]),
                                            "exact_weighted", "bce_dice", prefetch=prefetch)
        res.append((total.flat.clone(), st.losses_raw))
    assert torch.equal(res[0][0], res[1][0])
    assert res[0][1] == res[1][1]


@pytest.mark.parametrize("host", [False, True])
def test_train_epoch_matches_reference(cuda, host):
    meta = load_json("epoch.json")
    a = load_npz("epoch.npz")
    torch.manual_seed(0)
    mod = build_torch(meta["spec"], tuple(meta["input_shape"])).to(cuda)
    names = [k[3:] for k in a if k.startswith("p0/")]
    load_ref_params(mod, meta["spec"], {n: a[f"p0/{n}"] for n in names})
    params = mbs.ParameterSet(mod)
    x = torch.from_numpy(a["x"]).float()
    y = torch.from_numpy(a["y"]).long()
    if not host:
        x, y = x.to(cuda), y.to(cuda)
    st = mbs.sgd_state(0.05, 0.9, 5e-4)
    for epoch in range(2):
        es = mbs.train_epoch(mod, params, x, y, mini_batch_size=meta["mini"], micro_batch_size=meta["micro"],
                             normalization="exact_weighted", loss_kind="cross_entropy", optimizer_state=st,
                             seed=meta["seed"], epoch_index=epoch, lr_for_step=lambda s: mbs.linear_lr(0.05, s, 10),
                             prefetch=True, keep_mini_stats=True)
        want = meta["epochs"][epoch]
        assert es.mini_sizes == want["mini_sizes"]                 # 33/16 -> [16, 16, 1]
        assert es.step_count == want["step_count"]
        assert [s.n_micro for s in es.mini_stats] == want["n_micro"]
        np.testing.assert_allclose(es.mini_losses, [fhex(v) for v in want["mini_losses"]], rtol=1e-5)
        assert es.mean_loss == pytest.approx(fhex(want["mean_loss"]), rel=1e-5)
        got = to_ref(meta["spec"], {tn: params[tn] for tn in params.names()})
        keys = sorted(got)
        err = rel_l2(np.concatenate([got[k].ravel() for k in keys]),
                     np.concatenate([a[f"e{epoch}/{k}"].ravel() for k in keys]))
        assert err <= 1e-5


def test_step_count_is_per_mini_batch(cuda):
    meta = load_json("e2e.json")["mlp_mse"]
    a = load_npz("e2e.npz")
    mod, params = _model(meta, a, "mlp_mse", cuda)
    x, y = _xy(a, "mlp_mse", meta, 0, 24, cuda)
    st = mbs.adam_state()
    es = mbs.train_epoch(mod, params, x, y, mini_batch_size=7, micro_batch_size=2, normalization="paper_faithful",
                         loss_kind="mse", optimizer_state=st, seed=1, epoch_index=0)
    assert es.step_count == 4 and es.mini_sizes == [7, 7, 7, 3]   # never per micro-batch (SPEC acceptance 6)


def test_edge_cases(cuda):
    meta = load_json("e2e.json")["mlp_mse"]
    a = load_npz("e2e.npz")
    mod, params = _model(meta, a, "mlp_mse", cuda)
    st = mbs.adam_state()
    with pytest.raises(ValueError):                               # engine.py:295-296
        mbs.train_epoch(mod, params, torch.zeros(0, 6, device=cuda), torch.zeros(0, 3, device=cuda),
                        mini_batch_size=4, micro_batch_size=2, normalization="off", loss_kind="mse",
                        optimizer_state=st, seed=0, epoch_index=0)
    x, y = _xy(a, "mlp_mse", meta, 0, 5, cuda)
    with pytest.raises(ValueError):                               # engine.py:197-198
        mbs.mini_batch_gradient(mod, params, x, y, mbs.plan_split(6, 2), "off", "mse")
    with pytest.raises(ValueError):
        mbs.mini_batch_gradient(mod, params, x, y, mbs.plan_split(5, 2), "bogus", "mse")
    with pytest.raises(ValueError):
        mbs.mini_batch_gradient(mod, params, x, y, mbs.plan_split(5, 2), "off", "mse", normalize_via="x")
    # n_mu > n_b clamps (engine.py:66-67); size-1 micro-batches are legal
    total, s = mbs.mini_batch_gradient(mod, params, x, y, mbs.plan_split(5, 8), "paper_faithful", "mse")
    assert s.n_micro == 1
    total1, s1 = mbs.mini_batch_gradient(mod, params, x, y, mbs.plan_split(5, 1), "exact_weighted", "mse")
    assert s1.n_micro == 5
    assert rel_l2(total1.flat.double().cpu().numpy(), total.flat.double().cpu().numpy()) <= 1e-6
    # N_smu = 1: identical to plain mini-batch training in every mode
    outs = [mbs.mini_batch_gradient(mod, params, x, y, mbs.plan_split(5, 5), m, "mse")[0].flat.clone()
            for m in ("paper_faithful", "exact_weighted", "off")]
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[1], outs[2])


def test_nonfinite_loss_raises_and_keeps_params(cuda):
    meta = load_json("e2e.json")["mlp_mse"]
    a = load_npz("e2e.npz")
    mod, params = _model(meta, a, "mlp_mse", cuda)
    x, y = _xy(a, "mlp_mse", meta, 0, 6, cuda)
    x[2, 0] = float("inf")
    before = params.flat.clone()
    st = mbs.sgd_state()
    # the reference raises before any update (nn.py:578-579): parameters, moments and step_count untouched
    with pytest.raises(mbs.NonFiniteError):
        mbs.train_mini_batch(mod, params, (x, y), mbs.plan_split(6, 3), "paper_faithful", "mse", st)
    assert torch.equal(params.flat, before)
    assert st.step_count == 0 and not st.velocity


def test_nonfinite_in_epoch_raises_before_that_mini_batch_step(cuda):
    """A non-finite sample in mini-batch 2 of an epoch: the exception surfaces with exactly the state the
    reference leaves (mini-batch 1 stepped, mini-batch 2 not; step_count 1)."""
    from paper_2110_12484_b200.rng import epoch_order
    meta = load_json("e2e.json")["mlp_mse"]
    a = load_npz("e2e.npz")
    mod, params = _model(meta, a, "mlp_mse", cuda)
    x, y = _xy(a, "mlp_mse", meta, 0, 12, cuda)
    order = epoch_order(12, 5, 0, True)
    x[int(order[6 + 1]), 0] = float("nan")                 # lands in the second mini-batch of 6
    w0 = params.flat.clone()
    st = mbs.sgd_state(0.01, 0.9, 0.0)
    with pytest.raises(mbs.NonFiniteError):
        mbs.train_epoch(mod, params, x, y, mini_batch_size=6, micro_batch_size=4, normalization="exact_weighted",
                        loss_kind="mse", optimizer_state=st, seed=5, epoch_index=0)
    assert st.step_count == 1
    after_first = params.flat.clone()
    # the same first step taken alone from the same start
    params.flat.copy_(w0)
    st1 = mbs.sgd_state(0.01, 0.9, 0.0)
    idx = torch.from_numpy(order[:6].astype(np.int64)).to(cuda)
    mbs.train_mini_batch(mod, params, (x[idx], y[idx]), mbs.plan_split(6, 4), "exact_weighted", "mse", st1)
    assert torch.equal(params.flat, after_first)


def test_cuda_graph_micro_step_matches_eager(cuda, monkeypatch):
    """The captured micro step (graphs.MicroStepGraph) gives the eager result: same accumulated
    gradients, loss, BN running statistics, step count; ragged tail -> a second graph."""
    import copy
    from paper_2110_12484_b200 import engine, graphs
    from paper_2110_12484_b200.workloads import WORKLOADS, build_model
    torch.manual_seed(0)
    base = build_model(WORKLOADS["c1"], ops="native").to(cuda).to(memory_format=torch.channels_last)
    g = torch.Generator().manual_seed(3)
    x = torch.randn(20, 3, 32, 32, generator=g).to(cuda).contiguous(memory_format=torch.channels_last)
    y = torch.randint(0, 10, (20,), generator=g).to(cuda)
    res = {}
    for use in (False, True):
        monkeypatch.setattr(engine, "CUDA_GRAPHS", use)
        graphs.clear()
        net = copy.deepcopy(base)
        params = mbs.ParameterSet(net)
        for _ in range(2):                                   # second pass replays the captured graphs
            total, st = mbs.mini_batch_gradient(net, params, x, y, mbs.plan_split(20, 8), "exact_weighted",
                                                "cross_entropy")
        res[use] = (np.concatenate([total[n].detach().double().cpu().numpy().ravel() for n in params.names()]),
                    st.loss, {k: v.detach().clone() for k, v in net.state_dict().items() if "running" in k})
        if use:
            assert len(graphs._CACHE) == 2                  # [8, 8, 4]: full + tail shape
    a, b = res[False], res[True]
    assert np.linalg.norm(a[0] - b[0]) / np.linalg.norm(a[0]) <= 1e-5
    assert abs(a[1] - b[1]) <= 1e-5 * abs(a[1])
    for k in a[2]:
        assert torch.allclose(a[2][k], b[2][k], rtol=1e-5, atol=1e-6), k
    graphs.clear()


@pytest.mark.parametrize("mode", ["paper_faithful", "exact_weighted", "off"])
def test_bn_one_sample_tail_matches_reference(cuda, mode):
    """9/4 -> [4, 4, 1] into a BatchNorm over a 1x1 map: the tail micro-batch has ONE value per channel.
    The reference accepts it; torch's BatchNorm raises; K5 follows the reference: gradients,
    losses and two post-step weights against the reference's own run (fixture ``bn1_tail``)."""
    from paper_2110_12484_b200 import bn as K5
    name = "bn1_tail"
    meta = load_json("e2e.json")[name]
    a = load_npz("e2e.npz")
    torch.manual_seed(0)
    mod = build_torch(meta["spec"], tuple(meta["input_shape"])).to(cuda)
    load_ref_params(mod, meta["spec"], {n: a[f"{name}/p0/{n}"] for n in meta["param_names"]})
    K5.fuse_batchnorm(mod)
    params = mbs.ParameterSet(mod)
    n_b = meta["n_b"]
    plan = mbs.plan_split(n_b, meta["n_mu"])
    assert plan.sizes == (4, 4, 1)
    x, y = _xy(a, name, meta, 0, n_b, cuda)
    total, stats = mbs.mini_batch_gradient(mod, params, x, y, plan, mode, meta["loss_kind"])
    got = to_ref(meta["spec"], {tn: total[tn] for tn in params.names()})
    keys = sorted(got)
    assert rel_l2(np.concatenate([got[k].ravel() for k in keys]),
                  np.concatenate([a[f"{name}/{mode}/grad0/{k}"].ravel() for k in keys])) <= 1e-5
    ms = meta["modes"][mode][0]
    np.testing.assert_allclose(stats.losses_raw, [fhex(v) for v in ms["losses_raw"]], rtol=1e-5)
    assert stats.loss == pytest.approx(fhex(ms["loss"]), rel=1e-5)
    # the running statistics of the first mini-batch differ only in the variance convention (documented);
    # restart from the fixture's start for the two-step trajectory
    mod2 = build_torch(meta["spec"], tuple(meta["input_shape"])).to(cuda)
    load_ref_params(mod2, meta["spec"], {n: a[f"{name}/p0/{n}"] for n in meta["param_names"]})
    K5.fuse_batchnorm(mod2)
    params2 = mbs.ParameterSet(mod2)
    st = _opt(meta)
    for mb in range(2):
        x, y = _xy(a, name, meta, mb * n_b, (mb + 1) * n_b, cuda)
        mbs.train_mini_batch(mod2, params2, (x, y), plan, mode, meta["loss_kind"], st)
        got = to_ref(meta["spec"], {tn: params2[tn] for tn in params2.names()})
        assert rel_l2(np.concatenate([got[k].ravel() for k in keys]),
                      np.concatenate([a[f"{name}/{mode}/p{mb + 1}/{k}"].ravel() for k in keys])) <= 1e-5


@pytest.mark.parametrize("name", ["conv_ce", "seg_bce_dice"])
@pytest.mark.parametrize("host", [False, True], ids=["hbm", "host"])
def test_train_epoch_metric_fn_matches_reference(cuda, name, host):
    """train_epoch(metric_fn=...) (engine.py:323-324): per-mini-batch accuracy / IoU on the mini-batch's
    concatenated micro outputs, two epochs, against the reference's own run (fixture epoch_metrics)."""
    meta = load_json("epoch_metrics.json")[name]
    a = load_npz("epoch_metrics.npz")
    torch.manual_seed(0)
    mod = build_torch(meta["spec"], tuple(meta["input_shape"])).to(cuda)
    load_ref_params(mod, meta["spec"], {k[len(name) + 4:]: a[k] for k in a.keys() if k.startswith(f"{name}/p0/")})
    params = mbs.ParameterSet(mod)
    x = torch.from_numpy(a[f"{name}/x"]).float()
    y = torch.from_numpy(a[f"{name}/y"])
    if meta["loss_kind"] != "cross_entropy":
        y = y.float()
    if host:
        x, y = x.contiguous(), y.contiguous()
    else:
        x, y = x.to(cuda), y.to(cuda)
    st = mbs.sgd_state(0.01, 0.9, 5e-4) if meta["optimizer"] == "sgd" else mbs.adam_state(0.01, 5e-4)
    if name == "conv_ce":
        metric = mbs.accuracy
    else:
        def metric(o, t):
            return mbs.iou(torch.sigmoid(o), t)
    for epoch, want in enumerate(meta["epochs"]):
        es = mbs.train_epoch(mod, params, x, y, mini_batch_size=meta["mini"], micro_batch_size=meta["micro"],
                             normalization="exact_weighted", loss_kind=meta["loss_kind"], optimizer_state=st,
                             seed=meta["seed"], epoch_index=epoch, metric_fn=metric, prefetch=True)
        assert es.mini_sizes == want["mini_sizes"] and es.step_count == want["step_count"]
        np.testing.assert_allclose(es.mini_losses, [fhex(v) for v in want["mini_losses"]], rtol=1e-5)
        # thresholded metrics of fp32 outputs: identical unless an output sits within fp32 noise of the
        # decision boundary (argmax tie / the 0.5 threshold) — none does on this data
        np.testing.assert_allclose(es.mini_metrics, want["mini_metrics"], rtol=0, atol=1e-12)
