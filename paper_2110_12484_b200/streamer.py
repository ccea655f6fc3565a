"""Micro-batch sources on the B200: device staging (K2) and the pinned H2D streamer.

Reference: ``_micro_batches`` (``engine.py:140-163``) yields
``ascontiguousarray(x[lo:hi])`` slices in plan order, optionally materialising
micro-batch k+1 on one worker thread while k computes; ``train_epoch`` first
gathers ``x[order[start:start+M]]`` (``engine.py:310-312``). Here:

* a DEVICE-resident source is sliced (zero-copy view) or, when a row gather,
  dtype cast or NHWC layout is needed, staged by ``mbs_stage`` (K2) into a
  fresh model-input tensor on the compute stream;
* a HOST-resident source goes through ``MicroBatchStreamer``: a ring of
  pinned slots filled by a native gather pool, ``cudaMemcpyAsync`` on a
  dedicated copy stream into per-slot device buffers, and K2 staging from the
  slot into the model input; compute waits only on the slot's ready event, so
  the copy of micro-batch k+1 overlaps the forward/backward of k.

Staged bytes are bit-identical to ``x[rows].to(dtype[, channels_last])`` and the
partition is exactly the reference's index split (tests/test_stage_gpu.py).
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .prof import TIMER

_DT_CODE = {torch.uint8: N.U8, torch.float32: N.F32, torch.float64: N.F64, torch.bfloat16: N.BF16,
            torch.float16: N.F16}


@dataclass(frozen=True)
class Staging:
    """How micro-batch inputs are presented to the model."""

    dtype: torch.dtype = torch.float32      # model input dtype (f32 / bf16 / f16)
    channels_last: bool = False             # NHWC for 4-D inputs
    target_dtype: torch.dtype | None = None  # uint8 dense targets (masks) are staged to this dtype by K2

    def out_tensor(self, n: int, sample_shape: tuple, device) -> torch.Tensor:
        shape = (n,) + tuple(sample_shape)
        if self.channels_last and len(shape) == 4:
            return torch.empty(shape, dtype=self.dtype, device=device, memory_format=torch.channels_last)
        return torch.empty(shape, dtype=self.dtype, device=device)

    def is_identity_for(self, x: torch.Tensor) -> bool:
        return x.dtype == self.dtype and not (self.channels_last and x.dim() == 4)


def _chw(sample_shape: tuple) -> tuple:
    if len(sample_shape) == 3:
        return tuple(int(d) for d in sample_shape)
    return (1, 1, int(np.prod(sample_shape)) if sample_shape else 1)


def _stream_ptr(stream=None) -> int:
    return (stream or torch.cuda.current_stream()).cuda_stream


def stage_rows(src: torch.Tensor | int, src_dtype: torch.dtype, sample_shape: tuple, rows, row0: int, n: int,
               staging: Staging, device, stream=None, out: torch.Tensor | None = None) -> torch.Tensor:
    """K2: gather ``n`` rows (device ``rows`` tensor or ``row0..``) of ``src``, cast and lay out.

    ``src`` is a device tensor or a raw device/pinned pointer holding NCHW
    samples of ``src_dtype``. ``out``: a preallocated destination of the
    staged shape, dtype and layout (e.g. a captured micro step's static input,
    so the staged bytes are not copied a second time).
    """
    if src_dtype not in (torch.uint8, torch.float32, torch.float64):
        raise ValueError(f"staging supports uint8/float32/float64 sources, got {src_dtype}")
    if staging.dtype not in (torch.float32, torch.bfloat16, torch.float16):
        raise ValueError(f"staging produces float32/bfloat16/float16, got {staging.dtype}")
    if out is None:
        out = staging.out_tensor(n, sample_shape, device)
    elif not _fits(out, staging, (n,) + tuple(sample_shape)):
        raise ValueError("stage_rows: `out` does not have the staged shape / dtype / layout")
    C, H, W = _chw(sample_shape)
    layout = N.NHWC if (staging.channels_last and len(sample_shape) == 3) else N.NCHW
    src_ptr = src if isinstance(src, int) else src.data_ptr()
    rows_ptr = rows.data_ptr() if rows is not None else None
    t0 = TIMER.start(stream)
    N.check(N.lib().mbs_stage(src_ptr, _DT_CODE[src_dtype], rows_ptr, int(row0), int(n), C, H, W, out.data_ptr(),
                              _DT_CODE[staging.dtype], layout, _stream_ptr(stream)), "mbs_stage")
    if t0 is not None:
        elems = n * C * H * W
        TIMER.stop("k2_stage", t0, elems * (torch.tensor([], dtype=src_dtype).element_size() + out.element_size()),
                   stream)
    return out


def gather_rows(src: torch.Tensor | int, dtype: torch.dtype, sample_shape: tuple, rows, row0: int, n: int, device,
                stream=None, out: torch.Tensor | None = None) -> torch.Tensor:
    """Byte-exact row gather of targets (labels, masks) into a fresh (or the given contiguous) device tensor."""
    if out is None:
        out = torch.empty((n,) + tuple(sample_shape), dtype=dtype, device=device)
    elif out.dtype != dtype or tuple(out.shape) != (n,) + tuple(sample_shape) or not out.is_contiguous():
        raise ValueError("gather_rows: `out` does not have the gathered shape / dtype")
    row_bytes = int(np.prod(sample_shape)) * out.element_size() if sample_shape else out.element_size()
    src_ptr = src if isinstance(src, int) else src.data_ptr()
    rows_ptr = rows.data_ptr() if rows is not None else None
    t0 = TIMER.start(stream)
    N.check(N.lib().mbs_gather_rows(src_ptr, rows_ptr, int(row0), int(n), row_bytes, out.data_ptr(),
                                    _stream_ptr(stream)), "mbs_gather_rows")
    TIMER.stop("k2_gather_rows", t0, 2 * n * row_bytes, stream)
    return out


def _fits(t: torch.Tensor, staging: Staging, shape: tuple) -> bool:
    if t.dtype != staging.dtype or tuple(t.shape) != tuple(shape):
        return False
    if staging.channels_last and len(shape) == 4:
        return t.is_contiguous(memory_format=torch.channels_last)
    return t.is_contiguous()


def _target_staging(staging: Staging | None, y: torch.Tensor) -> Staging | None:
    """How dense uint8 targets (segmentation masks) are staged for the loss (K2, NCHW), or None to copy bytes."""
    if staging is None or staging.target_dtype is None or y.dim() < 2 or y.dtype != torch.uint8:
        return None
    return Staging(dtype=staging.target_dtype, channels_last=False)


def _dest(dest, n, sample_shape, staging, y_shape, y_dtype):
    """The consumer's preallocated (x, y) buffers for a micro-batch of n rows, or None."""
    if dest is None:
        return None
    return dest((n,) + tuple(sample_shape), staging.dtype, staging.channels_last and len(sample_shape) == 3,
                (n,) + tuple(y_shape), y_dtype)


def device_micro_batches(x: torch.Tensor, y: torch.Tensor, jobs, staging: Staging | None, *, dest=None,
                         tracer=None):
    """Device-resident source: yields (xk, yk) for each (rows, row0, n) job.

    ``dest(x_shape, x_dtype, channels_last, y_shape, y_dtype) -> (x_buf, y_buf) | None`` lets the consumer
    name where a staged micro-batch goes (a captured micro step's static buffers); ``tracer`` marks the
    point each micro-batch's data is ready (``streaming.ScheduleTracer``)."""
    dev = x.device
    st = staging or Staging(dtype=x.dtype if x.is_floating_point() and x.dtype != torch.float64
                            else torch.float32)
    ts = _target_staging(staging, y)
    y_shape = tuple(y.shape[1:])
    for rows, row0, n in jobs:
        if tracer is not None:
            tracer.data_ready()
        if rows is None and (staging is None or staging.is_identity_for(x)):
            xk = x[row0:row0 + n]
            yk = y[row0:row0 + n] if ts is None else stage_rows(y, y.dtype, y_shape, None, row0, n, ts, dev)
        else:
            buf = _dest(dest, n, tuple(x.shape[1:]), st, y_shape, ts.dtype if ts is not None else y.dtype)
            xk = stage_rows(x, x.dtype, tuple(x.shape[1:]), rows, row0, n, st, dev,
                            out=buf[0] if buf is not None else None)
            if ts is not None:
                yk = stage_rows(y, y.dtype, y_shape, rows, row0, n, ts, dev, out=buf[1] if buf is not None else None)
            elif rows is not None:
                yk = gather_rows(y, y.dtype, y_shape, rows, row0, n, dev, out=buf[1] if buf is not None else None)
            else:
                yk = y[row0:row0 + n]
        yield xk, yk


def _align(n: int, a: int = 256) -> int:
    return (n + a - 1) // a * a


class MicroBatchStreamer:
    """Pinned-ring host->device streamer (native worker + copy stream) with K2 staging.

    ``n_slots`` is the number of micro-batches in flight (2 = the reference's
    double buffering, ``streaming.py:96-101``; 3 = triple buffering).
    """

    def __init__(self, x_row_bytes: int, y_row_bytes: int, max_rows: int, *, n_slots: int = 3,
                 n_threads: int | None = None, device=None):
        if not torch.cuda.is_available():
            raise RuntimeError("MicroBatchStreamer needs a CUDA device (no CPU fallback)")
        self.device = torch.device(device or "cuda")
        self.n_slots = int(n_slots)
        self.max_rows = int(max_rows)
        self.x_row_bytes, self.y_row_bytes = int(x_row_bytes), int(y_row_bytes)
        self.y_off = _align(self.max_rows * self.x_row_bytes)
        self.slot_bytes = self.y_off + _align(self.max_rows * self.y_row_bytes)
        self.copy_stream = torch.cuda.Stream(self.device)
        threads = n_threads or max(1, min(16, (os.cpu_count() or 2) // 2))
        h = ctypes.c_void_p()
        N.check(N.lib().mbs_streamer_create(self.n_slots, self.slot_bytes, threads, self.copy_stream.cuda_stream,
                                            ctypes.byref(h)), "mbs_streamer_create")
        self._h = h
        self.dev_slots = [torch.empty(self.slot_bytes, dtype=torch.uint8, device=self.device)
                          for _ in range(self.n_slots)]
        self.jobs_issued: list = []   # (job_seq, n_rows) not yet harvested
        self.slot_job = [-1] * self.n_slots
        self._harvested: list = []    # (gather_ms, copy_ms, blocked_ms, bytes) of older jobs

    def close(self):
        if getattr(self, "_h", None):
            torch.cuda.synchronize(self.device)
            N.lib().mbs_streamer_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _submit(self, slot: int, x: torch.Tensor, y: torch.Tensor, rows: np.ndarray | None, row0: int, n: int):
        if n > self.max_rows:
            raise ValueError(f"micro-batch of {n} rows exceeds the streamer's max_rows={self.max_rows}")
        parts = (N.Part * 2)()
        base = self.dev_slots[slot].data_ptr()
        pinned = bool(x.is_pinned())
        parts[0] = N.Part(x.data_ptr(), self.x_row_bytes, base, int(pinned))
        parts[1] = N.Part(y.data_ptr(), self.y_row_bytes, base + self.y_off, int(bool(y.is_pinned())))
        rows_ptr = None
        if rows is not None:
            rows = np.ascontiguousarray(rows, dtype=np.int64)
            rows_ptr = rows.ctypes.data
        job = ctypes.c_int64(-1)
        N.check(N.lib().mbs_streamer_submit(self._h, slot, parts, 2, rows_ptr, int(row0), int(n),
                                            ctypes.byref(job)), "mbs_streamer_submit")
        self.jobs_issued.append((job.value, n))
        self.slot_job[slot] = job.value
        if len(self.jobs_issued) > 128:       # harvest long-finished jobs before the native ring (256) wraps
            old, self.jobs_issued = self.jobs_issued[:64], self.jobs_issued[64:]
            self._harvested.extend(self._read_timings(old))

    def timeline(self, job: int, origin: torch.cuda.Event) -> tuple:
        """(copy start, copy end) of job ``job``, seconds after ``origin`` (copy-stream events)."""
        from .streaming import streamer_timeline
        return streamer_timeline(self._h, job, origin)

    def stream(self, x: torch.Tensor, y: torch.Tensor, jobs, staging: Staging | None, *, prefetch: bool = True,
               dest=None, tracer=None):
        """Yield (xk, yk) device tensors for each (rows, row0, n) job over host tensors x, y
        (``dest`` / ``tracer``: see ``device_micro_batches``)."""
        if x.device.type != "cpu" or y.device.type != "cpu":
            raise ValueError("MicroBatchStreamer streams host-resident tensors")
        if not (x.is_contiguous() and y.is_contiguous()):
            raise ValueError("host source tensors must be contiguous")
        if x.element_size() * int(np.prod(x.shape[1:])) != self.x_row_bytes or \
                y.element_size() * int(np.prod(y.shape[1:])) != self.y_row_bytes:
            raise ValueError("row sizes differ from the streamer's configuration")
        jobs = list(jobs)
        staging = staging or Staging(dtype=x.dtype if x.dtype in (torch.float32,) else torch.float32)
        sample_shape, y_shape = tuple(x.shape[1:]), tuple(y.shape[1:])
        ts = _target_staging(staging, y)
        depth = self.n_slots if prefetch else 1
        nxt = 0
        while nxt < min(depth, len(jobs)):
            self._submit(nxt % self.n_slots, x, y, *jobs[nxt])
            nxt += 1
        cs = torch.cuda.current_stream(self.device)
        for k, (rows, row0, n) in enumerate(jobs):
            slot = k % self.n_slots
            if not prefetch and nxt == k:
                self._submit(slot, x, y, *jobs[k])
                nxt += 1
            N.check(N.lib().mbs_streamer_wait(self._h, slot, cs.cuda_stream), "mbs_streamer_wait")
            if tracer is not None:
                tracer.data_ready(self.slot_job[slot], self, cs)
            base = self.dev_slots[slot].data_ptr()
            buf = _dest(dest, n, sample_shape, staging, y_shape, ts.dtype if ts is not None else y.dtype)
            xk = stage_rows(base, x.dtype, sample_shape, None, 0, n, staging, self.device, cs,
                            out=buf[0] if buf is not None else None)
            if ts is not None:
                yk = stage_rows(base + self.y_off, y.dtype, y_shape, None, 0, n, ts, self.device, cs,
                                out=buf[1] if buf is not None else None)
            else:
                yk = gather_rows(base + self.y_off, y.dtype, y_shape, None, 0, n, self.device, cs,
                                 out=buf[1] if buf is not None else None)
            N.check(N.lib().mbs_streamer_release(self._h, slot, cs.cuda_stream), "mbs_streamer_release")
            if prefetch and nxt < len(jobs):
                self._submit(nxt % self.n_slots, x, y, *jobs[nxt])
                nxt += 1
            yield xk, yk

    def timings(self, flush: bool = True) -> list:
        """Per-job (gather_ms, copy_ms, blocked_ms, bytes) for the jobs issued so far (synchronises)."""
        out = self._harvested + self._read_timings(self.jobs_issued)
        if flush:
            self.jobs_issued = []
            self._harvested = []
        return out

    def _read_timings(self, jobs) -> list:
        out = []
        for seq, _n in jobs:
            g, c, b = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
            nb = ctypes.c_int64()
            st = N.lib().mbs_streamer_timing(self._h, seq, ctypes.byref(g), ctypes.byref(c), ctypes.byref(b),
                                             ctypes.byref(nb))
            if st == N.OK:
                out.append((g.value, c.value, b.value, nb.value))
        return out
