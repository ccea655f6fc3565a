"""ctypes binding of ``libmbs_native.so`` — the C-ABI declared in ``include/mbs.h``.

The product path has exactly one implementation: the sm_100a kernels in this
library. There is no CPU or PyTorch fallback; if the library is missing or a
GPU call is made without CUDA, the call raises.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_double, c_int, c_int64, c_void_p

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MBS_NATIVE_LIB") or os.path.join(_HERE, "libmbs_native.so")  # override: kernel A/B runs

# status codes (include/mbs.h)
OK, EINVAL, EOVERFLOW, EKEY, ECUDA, ENONFINITE = range(6)
NORM_MODES = {"paper_faithful": 0, "exact_weighted": 1, "off": 2}
U8, F32, BF16, F16, F64 = range(5)
NCHW, NHWC = 0, 1
MAX_PARTS = 4
PEER_HANDLE_BYTES = 128


class Part(ctypes.Structure):
    """``mbs_part_t``."""

    _fields_ = [("src", c_void_p), ("row_bytes", c_int64), ("dst", c_void_p), ("src_pinned", c_int)]


_lib = None

_SIGS = {
    "mbs_status_string": (ctypes.c_char_p, [c_int]),
    "mbs_last_error": (ctypes.c_char_p, []),
    "mbs_version": (c_int, []),
    "mbs_plan_split": (c_int, [c_int64, c_int64, POINTER(c_int64), POINTER(c_int64), POINTER(c_int64), c_int64]),
    "mbs_normalization_factor": (c_int, [c_int64, c_int64, c_int64, c_int, POINTER(c_double)]),
    "mbs_accum_create": (c_int, [c_void_p, c_int64, c_int64, POINTER(c_int64), POINTER(c_int64), c_int64,
                                 POINTER(c_void_p)]),
    "mbs_accum_destroy": (c_int, [c_void_p]),
    "mbs_accum_begin": (c_int, [c_void_p, c_int64]),
    "mbs_accum_zero": (c_int, [c_void_p, c_void_p]),
    "mbs_accum_add": (c_int, [c_void_p, POINTER(c_void_p), c_int64, c_int64, c_double, c_void_p, c_double, c_double,
                              c_int, c_void_p]),
    "mbs_accum_add_typed": (c_int, [c_void_p, POINTER(c_void_p), c_void_p, c_int64, c_int64, c_double, c_void_p,
                                    c_double, c_double, c_int, c_void_p]),
    "mbs_accum_add_flat": (c_int, [c_void_p, c_void_p, c_double, c_void_p, c_double, c_double, c_int, c_void_p]),
    "mbs_accum_norm": (c_int, [c_void_p, c_void_p]),
    "mbs_accum_finalize": (c_int, [c_void_p, c_int64, c_void_p, c_void_p]),
    "mbs_accum_seen": (c_int, [c_void_p, POINTER(c_int64), POINTER(c_int64)]),
    "mbs_sgd_step": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_double, c_double, c_double, c_void_p,
                             c_void_p, c_void_p]),
    "mbs_adam_step": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_double, c_double, c_double,
                              c_double, c_double, c_int64, c_void_p, c_void_p, c_void_p]),
    "mbs_stage": (c_int, [c_void_p, c_int, c_void_p, c_int64, c_int64, c_int64, c_int64, c_int64, c_void_p, c_int,
                          c_int, c_void_p]),
    "mbs_gather_rows": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_int64, c_void_p, c_void_p]),
    "mbs_streamer_create": (c_int, [c_int, c_int64, c_int, c_void_p, POINTER(c_void_p)]),
    "mbs_streamer_destroy": (c_int, [c_void_p]),
    "mbs_streamer_submit": (c_int, [c_void_p, c_int, POINTER(Part), c_int, c_void_p, c_int64, c_int64,
                                    POINTER(c_int64)]),
    "mbs_streamer_wait": (c_int, [c_void_p, c_int, c_void_p]),
    "mbs_streamer_release": (c_int, [c_void_p, c_int, c_void_p]),
    "mbs_streamer_timing": (c_int, [c_void_p, c_int64, POINTER(c_double), POINTER(c_double), POINTER(c_double),
                                    POINTER(c_int64)]),
    "mbs_streamer_timeline": (c_int, [c_void_p, c_int64, c_void_p, POINTER(c_double), POINTER(c_double)]),
    "mbs_host_gather": (c_int, [c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_int]),
    "mbs_peer_create": (c_int, [c_int, c_int, c_int64, POINTER(c_void_p)]),
    "mbs_peer_handle": (c_int, [c_void_p, c_void_p]),
    "mbs_peer_open": (c_int, [c_void_p, c_void_p]),
    "mbs_peer_destroy": (c_int, [c_void_p]),
    "mbs_peer_status": (c_int, [c_void_p, POINTER(c_int)]),
    "mbs_accum_add_allreduce": (c_int, [c_void_p, c_void_p, POINTER(c_void_p), c_double, c_void_p, c_double,
                                        c_double, c_double, c_void_p]),
    "mbs_bn_workspace_bytes": (c_int, [c_int64, c_int64, c_int, POINTER(c_int64)]),
    "mbs_bn_forward": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_int64, c_int64, c_void_p, c_void_p, c_void_p,
                               c_void_p, c_void_p, c_double, c_double, c_int, c_void_p, c_void_p, c_void_p,
                               c_void_p]),
    "mbs_bn_backward": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int64, c_int64,
                                c_void_p,
                                c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_void_p, c_void_p, c_void_p]),
    "mbs_maxpool_forward": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_int64, c_int64, c_int64, c_int64, c_int,
                                    c_int, c_int, c_void_p, c_int64, c_int64, c_void_p]),
    "mbs_maxpool_backward": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int64, c_int64, c_int64, c_int64,
                                     c_int, c_int, c_int, c_void_p, c_int64, c_int64, c_void_p]),
    "mbs_copy_channels": (c_int, [c_void_p, c_int64, c_int64, c_void_p, c_int64, c_int64, c_int64, c_int64, c_void_p,
                                  c_void_p, c_int64, c_int, c_void_p]),
    "mbs_im2col": (c_int, [c_void_p, c_void_p, c_int, c_int64, c_int64, c_int64, c_int64, c_int, c_int, c_int, c_int64,
                           c_void_p]),
}

EXPORTS = tuple(_SIGS)


def lib():
    """Load (once) and return the native library; raise loudly when it is absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(or `make -C paper_2110_12484_b200/csrc`). There is no CPU fallback.")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(status: int, what: str = "") -> None:
    """Map an ``MBS_*`` status to the reference's exception types (errors.py)."""
    if status == OK:
        return
    msg = lib().mbs_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if status == EINVAL:
        raise ValueError(text)
    if status == EOVERFLOW:
        raise errors.AccumulatorOverflowError(text)
    if status == EKEY:
        raise errors.GradientKeyMismatchError(text)
    if status == ENONFINITE:
        raise errors.NonFiniteError(-1, text)
    raise RuntimeError(f"CUDA error in {what}: {msg}")


def i64_array(values):
    arr = (c_int64 * len(values))(*values)
    return arr
