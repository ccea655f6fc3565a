"""The measured schedule (streaming.ScheduleTracer): real CUDA events per micro-batch, in the reference's
StreamEvent / StreamSchedule shapes (streaming.py:41-53), fed to overhead_report (streaming.py:130-149)."""
import pytest
import torch

import paper_2110_12484_b200 as mbs
from paper_2110_12484_b200 import graphs, streaming
from paper_2110_12484_b200.streamer import Staging
from paper_2110_12484_b200.workloads import WORKLOADS, build_model

pytestmark = pytest.mark.gpu

EPS = 50e-6    # event timestamps are ~0.5 us resolution; cross-stream ordering is exact up to that


def _run(cuda, host: bool, tracer):
    w = WORKLOADS["c1"]
    torch.manual_seed(0)
    net = build_model(w, ops="native").to(cuda).to(memory_format=torch.channels_last)
    params = mbs.ParameterSet(net, shadow=torch.bfloat16)
    g = torch.Generator().manual_seed(4)
    x = torch.randint(0, 256, (44, 3, 32, 32), dtype=torch.uint8, generator=g)
    y = torch.randint(0, 10, (44,), generator=g)
    if host:
        x, y = x.pin_memory(), y.pin_memory()
    else:
        x, y = x.to(cuda), y.to(cuda)
    st = mbs.sgd_state(0.01, 0.9, 5e-4)
    streamer = mbs.make_streamer(x, y, 8, n_slots=3) if host else None
    es = mbs.train_epoch(net, params, x, y, mini_batch_size=20, micro_batch_size=8,
                         normalization="exact_weighted", loss_kind="cross_entropy", optimizer_state=st, seed=3,
                         epoch_index=0, prefetch=True, staging=Staging(torch.bfloat16, True),
                         autocast_dtype=torch.bfloat16, streamer=streamer, tracer=tracer)
    if streamer is not None:
        streamer.close()
    return es, params.flat.clone()


@pytest.mark.parametrize("host", [True, False], ids=["host_streamed", "hbm_resident"])
def test_tracer_schedule_shape_and_order(cuda, host, monkeypatch):
    monkeypatch.setattr(torch.backends.cudnn, "deterministic", True)
    graphs.clear()
    es0, w0 = _run(cuda, host, None)
    graphs.clear()
    tr = streaming.ScheduleTracer(cuda)
    es1, w1 = _run(cuda, host, tr)
    graphs.clear()
    # tracing changes nothing (same kernels, same order)
    assert torch.equal(w0, w1) and es0.mini_losses == es1.mini_losses
    scheds = tr.schedules()
    assert [len(s.events) for s in scheds] == [(2 + host) * n + 1 for n in (3, 3, 1)]   # 44 = 20 + 20 + 4
    prev_update_end = -1.0
    for s in scheds:
        ev = {(e.kind, e.index): e for e in s.events}
        n = sum(1 for e in s.events if e.kind == "forward")
        for k in range(n):
            f, b = ev[("forward", k)], ev[("backward", k)]
            assert f.start <= f.end <= b.end
            if host:
                t = ev[("transfer", k)]
                assert t.start < t.end <= f.start + EPS        # compute starts only after its copy landed
            if k:
                assert f.start >= ev[("backward", k - 1)].end - EPS
        u = ev[("update", -1)]
        assert u.start >= ev[("backward", n - 1)].end - EPS and u.end > u.start
        assert ev[("forward", 0)].start >= prev_update_end - EPS
        prev_update_end = u.end
        assert s.makespan > 0 and s.overlap_enabled
        if host:
            frac = streaming.overlap_fraction(s)
            assert frac is not None and 0.0 <= frac <= 1.0
    rep = streaming.overhead_report(scheds[0], scheds[1])
    assert rep.baseline_makespan == pytest.approx(scheds[1].makespan)


def test_graph_step_stages_into_its_static_input(cuda):
    """Once a micro step is captured, K2 stages the next micro-batches straight into its static input
    (no second copy of the staged bytes) — and the results equal the eager path's."""
    from paper_2110_12484_b200 import engine
    graphs.clear()
    es_g, w_g = _run(cuda, False, None)
    caps = list(graphs._CACHE.values())
    assert caps, "no captured micro step"
    graphs.clear()
    old = engine.CUDA_GRAPHS
    engine.CUDA_GRAPHS = False
    try:
        es_e, w_e = _run(cuda, False, None)
    finally:
        engine.CUDA_GRAPHS = old
    assert float((w_g - w_e).norm() / w_e.norm()) <= 1e-6
    assert es_g.mini_losses == pytest.approx(es_e.mini_losses, rel=1e-3)
    # the dest hook returns the captured buffers for the captured shapes
    w = WORKLOADS["c1"]
    torch.manual_seed(0)
    net = build_model(w, ops="native").to(cuda).to(memory_format=torch.channels_last)
    params = mbs.ParameterSet(net, shadow=torch.bfloat16)
    acc = mbs.GradientAccumulator(params)
    x = torch.randint(0, 256, (16, 3, 32, 32), dtype=torch.uint8, device=cuda)
    y = torch.randint(0, 10, (16,), device=cuda)
    net.train()
    dest = engine._graph_dest(net, acc, "cross_entropy", torch.bfloat16, True, 1.0, "fused")
    assert dest((8, 3, 32, 32), torch.bfloat16, True, (8,), torch.int64) is None
    mbs.mini_batch_gradient(net, params, x, y, mbs.plan_split(16, 8), "exact_weighted", "cross_entropy",
                            accumulator=acc, staging=Staging(torch.bfloat16, True), autocast_dtype=torch.bfloat16)
    bufs = dest((8, 3, 32, 32), torch.bfloat16, True, (8,), torch.int64)
    assert bufs is not None and bufs[0].is_contiguous(memory_format=torch.channels_last)
    graphs.clear()
