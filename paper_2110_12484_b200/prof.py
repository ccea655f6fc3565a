"""Live per-kernel timing with CUDA events on the launching stream (used by bench.py).

When enabled, every K1 / K2 / K3 launch made through the package is bracketed
by a pair of timing events recorded on the stream it is launched on, together
with its ALGORITHMIC byte count (what the reference semantics must move:
K1 (g bytes + 8) B/param for acc += s*g and (g bytes + 4) B/param for the
first micro-batch's acc = s*g — g is 4 B fp32, or 2 B for the bf16 weight
gradients of shadow-weight mode, so 12/8 or 10/6 B/param; K3 20 B/param SGD,
28 B/param Adam, +2 B/param when it also writes the bf16 shadow; K2 source +
staged bytes).
Disabled (the default) it costs one attribute test per launch.
"""

from __future__ import annotations

from collections import defaultdict

import torch


class KernelTimer:
    def __init__(self):
        self.enabled = False
        self.k5 = False            # also time the model-side K5 BatchNorm launches (bn.py)
        self.launches = 0          # every native kernel launch made through the package
        self._open = defaultdict(list)

    def reset(self):
        self._open = defaultdict(list)
        self.launches = 0

    def start(self, stream=None):
        self.launches += 1
        if not self.enabled or torch.cuda.is_current_stream_capturing():
            return None
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(stream or torch.cuda.current_stream())
        return ev

    def start_k5(self, n_launches: int, stream=None):
        """K5 calls launch ``n_launches`` kernels each; timed only when ``enabled and k5``."""
        self.launches += n_launches
        if not (self.enabled and self.k5) or torch.cuda.is_current_stream_capturing():
            return None
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(stream or torch.cuda.current_stream())
        return ev

    def stop(self, name: str, start_ev, nbytes: int, stream=None):
        if start_ev is None:
            return
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(stream or torch.cuda.current_stream())
        self._open[name].append((start_ev, ev, int(nbytes)))

    def summary(self) -> dict:
        """{name: {launches, total_ms, avg_ms, bytes_per_launch, gbs}} (synchronises)."""
        torch.cuda.synchronize()
        out = {}
        for name, recs in self._open.items():
            ms = [a.elapsed_time(b) for a, b, _ in recs]
            nb = [n for _, _, n in recs]
            tot = sum(ms)
            out[name] = {"launches": len(recs), "total_ms": tot, "avg_ms": tot / max(1, len(recs)),
                         "bytes_per_launch": sum(nb) / max(1, len(nb)),
                         "gbs": (sum(nb) / (tot / 1e3) / 1e9) if tot > 0 else 0.0}
        return out


TIMER = KernelTimer()
