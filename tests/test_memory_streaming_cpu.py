"""memory.fit_micro_batch and streaming.simulate_stream vs the reference's fixtures (CPU)."""
import pytest

import paper_2110_12484_b200 as mbs
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
    for case in load_json("misc.json")["simulate_stream"]:
        plan = mbs.plan_split(case["n_b"], case["n_mu"])
        cost = streaming.CostModel(*case["cost"])
        s = streaming.simulate_stream(plan, cost, case["bps"], overlap=case["overlap"])
        assert s.makespan.hex() == case["makespan"]
        assert [[e.kind, e.index, e.start.hex(), e.end.hex()] for e in s.events] == case["events"]
        if not case["overlap"]:
            assert streaming.sequential_makespan(plan, cost, case["bps"]).hex() == case["makespan"]


def test_overhead_report():
    plan = mbs.plan_split(8, 2)
    c = streaming.CostModel(1e-3, 1.0, 2.0, 0.5, 0.1, 0.2)
    a = streaming.simulate_stream(plan, c, 100, overlap=True)
    b = streaming.simulate_stream(mbs.plan_split(8, 8), c, 100, overlap=False)
    r = streaming.overhead_report(a, b)
    assert r.overhead_seconds == pytest.approx(a.makespan - b.makespan)
    assert streaming.overhead_report(a, None).baseline_failed
    m = streaming.measured_schedule([1.0, 1.0, 1.0], [30.0, 30.0, 30.0], 0.5)
    assert m.makespan == pytest.approx((1.0 + 90.0 + 0.5) / 1e3)


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
