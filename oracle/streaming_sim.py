"""Virtual-time streaming simulator — TEST INFRASTRUCTURE ONLY (see mbs_oracle.py header).

Restates the reference's ``streaming.py`` cost model and two-slot schedule
(``/root/reference/pkg/src/mbstream/streaming.py``): ``CostModel`` (19-38),
``_durations`` (56-63), ``sequential_makespan`` (66-75), ``simulate_stream``
(78-111) and ``epoch_makespan`` (152-161). The product package does not
simulate: it MEASURES its schedule with CUDA events
(``paper_2110_12484_b200.streaming.ScheduleTracer``) and emits the reference's
``StreamEvent`` / ``StreamSchedule`` shapes. This module is the ideal those
measured schedules are compared with in tests and bench.py, and is pinned to
the reference's own outputs by ``tests/test_memory_streaming_cpu.py``.
"""

from __future__ import annotations

from dataclasses import dataclass

from . import mbs_oracle as O


@dataclass(frozen=True)
class CostModel:
    """streaming.py:19-38 (non-negative fields)."""

    transfer_seconds_per_byte: float
    compute_seconds_per_sample_forward: float
    compute_seconds_per_sample_backward: float
    update_seconds: float = 0.0
    transfer_latency_seconds: float = 0.0
    compute_latency_seconds: float = 0.0

    def __post_init__(self):
        for name, value in self.__dict__.items():
            if value < 0:
                raise ValueError(f"{name} must be non-negative, got {value}")


def durations(sizes, cost: CostModel, bytes_per_sample: int):
    """streaming.py:56-63: per-micro (transfer, forward, backward) seconds."""
    tr = [cost.transfer_latency_seconds + s * bytes_per_sample * cost.transfer_seconds_per_byte for s in sizes]
    fw = [cost.compute_latency_seconds + s * cost.compute_seconds_per_sample_forward for s in sizes]
    bw = [cost.compute_latency_seconds + s * cost.compute_seconds_per_sample_backward for s in sizes]
    return tr, fw, bw


def simulate_stream(sizes, cost: CostModel, bytes_per_sample: int, overlap: bool = False):
    """streaming.py:78-111 -> (makespan, [(kind, index, start, end), ...])."""
    tr, fw, bw = durations(sizes, cost, bytes_per_sample)
    return O.simulate_stream(tr, fw, bw, cost.update_seconds, overlap)


def sequential_makespan(sizes, cost: CostModel, bytes_per_sample: int) -> float:
    """streaming.py:66-75: every transfer, forward and backward back to back, then the update."""
    tr, fw, bw = durations(sizes, cost, bytes_per_sample)
    total = 0.0
    for k in range(len(sizes)):
        total += tr[k]
        total += fw[k]
        total += bw[k]
    return total + cost.update_seconds


def epoch_makespan(plans_sizes, cost: CostModel, bytes_per_sample: int, overlap: bool = False) -> float:
    """streaming.py:152-161: the mini-batch makespans of an epoch, summed."""
    return sum(simulate_stream(s, cost, bytes_per_sample, overlap)[0] for s in plans_sizes)
