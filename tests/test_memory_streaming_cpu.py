"""memory.fit_micro_batch vs the reference's fixtures; the oracle's stream simulator vs the reference's
schedules; the product's schedule shapes / overhead report / overlap fraction (CPU)."""
import pytest

import paper_2110_12484_b200 as mbs
from oracle import streaming_sim as S
from paper_2110_12484_b200 import memory, streaming
from tests.golden_io import load_json


def test_fit_micro_batch_golden():
    for cap, res, per, want in load_json("misc.json")["fit_micro_batch"]:
        b = memory.MemoryBudget(capacity_bytes=cap, param_bytes=res, data_bytes_per_sample=per)
        if isinstance(want, int):
            assert memory.fit_micro_batch(b) == want
            assert b.fits(want) and not b.fits(want + 1)
        else:
            with pytest.raises(mbs.ModelDoesNotFitError):
                memory.fit_micro_batch(b)
    with pytest.raises(ValueError):
        memory.MemoryBudget(capacity_bytes=0, param_bytes=1, data_bytes_per_sample=1)
    assert memory.parameter_space_bytes(10, "adam") == 4 * 10 * 4


def test_simulate_stream_golden():
    """The oracle's virtual-time simulator (test infrastructure) == the reference's own schedules."""
    for case in load_json("misc.json")["simulate_stream"]:
        sizes = mbs.plan_split(case["n_b"], case["n_mu"]).sizes
        cost = S.CostModel(*case["cost"])
        makespan, events = S.simulate_stream(sizes, cost, case["bps"], overlap=case["overlap"])
        assert makespan.hex() == case["makespan"]
        assert [[e[0], e[1], e[2].hex(), e[3].hex()] for e in events] == case["events"]
        if not case["overlap"]:
            assert S.sequential_makespan(sizes, cost, case["bps"]).hex() == case["makespan"]
    with pytest.raises(ValueError):
        S.CostModel(-1.0, 0.0, 0.0)


def _sched(events):
    evs = tuple(streaming.StreamEvent(*e) for e in events)
    t0 = min(e.start for e in evs)
    return streaming.StreamSchedule(evs, max(e.end for e in evs) - t0, True)


def test_overhead_report_on_schedules():
    """streaming.py:130-149 applied to two (measured-shape) schedules; a failed baseline is reported."""
    sizes = mbs.plan_split(8, 2).sizes
    c = S.CostModel(1e-3, 1.0, 2.0, 0.5, 0.1, 0.2)
    a = _sched(S.simulate_stream(sizes, c, 100, overlap=True)[1])
    b = _sched(S.simulate_stream((8,), c, 100, overlap=False)[1])
    r = streaming.overhead_report(a, b)
    assert r.overhead_seconds == pytest.approx(a.makespan - b.makespan)
    assert r.overhead_pct == pytest.approx(100 * (a.makespan - b.makespan) / b.makespan)
    assert streaming.overhead_report(a, None).baseline_failed


def test_overlap_fraction():
    # transfer 1 hidden behind compute 0; transfer 2 ends 0.5 after compute 1 -> 0.5 of 3.0 exposed
    s = _sched([("transfer", 0, 0.0, 1.0), ("forward", 0, 1.0, 2.0), ("backward", 0, 2.0, 4.0),
                ("transfer", 1, 1.0, 2.0), ("forward", 1, 4.0, 5.0), ("backward", 1, 5.0, 7.0),
                ("transfer", 2, 6.5, 7.5), ("forward", 2, 7.5, 8.0), ("backward", 2, 8.0, 9.0),
                ("update", -1, 9.0, 9.5)])
    assert streaming.overlap_fraction(s) == pytest.approx(1.0 - 0.5 / 3.0)
    assert streaming.overlap_fraction(_sched([("forward", 0, 0.0, 1.0), ("backward", 0, 1.0, 2.0)])) is None


def test_bn_safe_micro_batch():
    from paper_2110_12484_b200.memory import bn_safe_micro_batch
    assert bn_safe_micro_batch(33, 16) == 15            # 33/16 -> [16,16,1]; 33/15 -> [15,15,3]
    assert bn_safe_micro_batch(64, 8) == 8
    assert bn_safe_micro_batch(2, 5) == 2
    assert bn_safe_micro_batch(1, 5) == 1
    for n_b in range(2, 200):
        for n_mu in (1, 2, 3, 7, 16, 48, 128):
            m = bn_safe_micro_batch(n_b, n_mu)
            assert 1 <= m <= n_mu
            assert min(mbs.plan_split(n_b, m).sizes) > 1 or m == 1


def test_auto_micro_batch_applies_the_bn_guard_to_stock_batchnorm_only():
    import torch
    from paper_2110_12484_b200 import bn
    b = memory.MemoryBudget(capacity_bytes=1000 + 16 * 10, param_bytes=1000, data_bytes_per_sample=10)
    assert memory.fit_micro_batch(b) == 16
    stock = torch.nn.Sequential(torch.nn.Conv2d(3, 4, 3), torch.nn.BatchNorm2d(4))
    assert memory.auto_micro_batch(b, 33, stock) == 15           # 33/16 -> [16,16,1]: torch BN would raise
    native = torch.nn.Sequential(torch.nn.Conv2d(3, 4, 3), torch.nn.BatchNorm2d(4))
    bn.fuse_batchnorm(native)
    assert memory.auto_micro_batch(b, 33, native) == 16          # K5 takes the 1-sample tail (reference rule)
    assert memory.auto_micro_batch(b, 8, stock) == 8             # capped at the mini-batch
    assert memory.auto_micro_batch(b, 33, None) == 16
