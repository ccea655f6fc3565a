"""SPEC data-cli datasets: synthetic classification / segmentation and the IDX loader.

The reference declares this module but does not ship it (no data/config/CSV module);
its contract is the SPEC. Everything here is host-side data plumbing: it produces host tensors that the
micro-batch streamer / K2 staging then move to HBM. Generated datasets are a pure function of
(spec, seed): every random draw comes from a named Philox substream (``rng.named_stream``), so changing
one component's stream never perturbs another.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass, field

import numpy as np

from .errors import ConfigError, IdxFormatError
from .rng import named_stream

DATASET_KINDS = ("synthetic_classification", "synthetic_segmentation", "idx_images")


@dataclass(frozen=True)
class DatasetSpec:
    """SPEC.md:477-481."""

    kind: str
    n_samples: int = 0
    input_shape: tuple = ()
    n_classes: int = 0                 # classification
    mask_shape: tuple = ()             # segmentation
    seed: int = 0
    path: str = ""                     # idx_images: the image file
    labels_path: str = ""              # idx_images: the label file (optional)
    separation: float = 3.0            # classification: distance scale of the class means (in noise units)
    extra: dict = field(default_factory=dict, compare=False, hash=False)

    def validate(self) -> None:
        if self.kind not in DATASET_KINDS:
            raise ConfigError(f"dataset.kind must be one of {DATASET_KINDS}, got {self.kind!r}")
        if self.kind == "idx_images":
            if not self.path:
                raise ConfigError("dataset.path is required for idx_images")
            return
        if self.n_samples < 1 or not self.input_shape or any(int(d) < 1 for d in self.input_shape):
            raise ConfigError(f"degenerate dataset shape: n_samples={self.n_samples}, input_shape={self.input_shape}")
        if self.seed < 0 or self.seed >= 2 ** 64:
            raise ConfigError("dataset.seed must be a 64-bit unsigned integer")
        if self.kind == "synthetic_classification" and self.n_classes < 2:
            raise ConfigError("synthetic_classification needs n_classes >= 2")
        if self.kind == "synthetic_segmentation":
            if len(self.input_shape) != 3:
                raise ConfigError("synthetic_segmentation needs input_shape (C, H, W)")
            ms = tuple(self.mask_shape) or (1,) + tuple(self.input_shape[1:])
            if tuple(ms[-2:]) != tuple(self.input_shape[1:]):
                raise ConfigError(f"mask_shape {ms} must match the input's spatial shape {self.input_shape[1:]}")


def balanced_labels(n: int, k: int, rng: np.random.Generator) -> np.ndarray:
    """Labels 0..k-1 whose counts differ by at most one, in a seeded random order."""
    return rng.permutation(np.arange(n) % k).astype(np.int64)


def gen_synthetic_classification(spec: DatasetSpec) -> tuple:
    """Gaussian class clusters: x ~ mean[y] + spread[y] * N(0, 1), float32; y int64.

    Means ~ separation * N(0, 1) per feature, spreads ~ U(0.5, 1.0) per class — both seed-deterministic.
    """
    spec.validate()
    if spec.kind != "synthetic_classification":
        raise ConfigError(f"not a classification spec: {spec.kind}")
    shape, k, n = tuple(int(d) for d in spec.input_shape), int(spec.n_classes), int(spec.n_samples)
    means = named_stream(spec.seed, "dataset/classification/means").standard_normal((k,) + shape) * spec.separation
    spreads = named_stream(spec.seed, "dataset/classification/spreads").uniform(0.5, 1.0, size=k)
    y = balanced_labels(n, k, named_stream(spec.seed, "dataset/classification/labels"))
    noise = named_stream(spec.seed, "dataset/classification/noise").standard_normal((n,) + shape)
    x = means[y] + spreads[y].reshape((n,) + (1,) * len(shape)) * noise
    return x.astype(np.float32), y


def gen_synthetic_segmentation(spec: DatasetSpec) -> tuple:
    """Images of one seeded random rectangle or disk each, with the exact ground-truth mask.

    image = 0.2 + 0.6 * mask + 0.05 * N(0, 1) per channel (float32); mask = the painted shape (uint8 {0, 1}).
    ``spec.extra["coverage"]`` = "empty" / "full" forces all-background / all-foreground samples.
    """
    spec.validate()
    if spec.kind != "synthetic_segmentation":
        raise ConfigError(f"not a segmentation spec: {spec.kind}")
    c, h, w = (int(d) for d in spec.input_shape)
    n = int(spec.n_samples)
    g = named_stream(spec.seed, "dataset/segmentation/shapes")
    kind = g.integers(0, 2, size=n)                       # 0 rectangle, 1 disk
    cy, cx = g.uniform(0, h, size=n), g.uniform(0, w, size=n)
    ry, rx = g.uniform(0.1, 0.4, size=n) * h, g.uniform(0.1, 0.4, size=n) * w
    yy, xx = np.meshgrid(np.arange(h) + 0.5, np.arange(w) + 0.5, indexing="ij")
    rect = (np.abs(yy[None] - cy[:, None, None]) <= ry[:, None, None]) & \
           (np.abs(xx[None] - cx[:, None, None]) <= rx[:, None, None])
    r = np.minimum(ry, rx)
    disk = (yy[None] - cy[:, None, None]) ** 2 + (xx[None] - cx[:, None, None]) ** 2 <= (r ** 2)[:, None, None]
    mask = np.where(kind[:, None, None] == 0, rect, disk)
    cov = spec.extra.get("coverage") if spec.extra else None
    if cov == "empty":
        mask[:] = False
    elif cov == "full":
        mask[:] = True
    noise = named_stream(spec.seed, "dataset/segmentation/noise").standard_normal((n, c, h, w))
    x = 0.2 + 0.6 * mask[:, None].astype(np.float64) + 0.05 * noise
    return x.astype(np.float32), mask[:, None].astype(np.uint8)


_IDX_TYPES = {0x08: (np.uint8, 1), 0x09: (np.int8, 1), 0x0B: (np.dtype(">i2"), 2), 0x0C: (np.dtype(">i4"), 4),
              0x0D: (np.dtype(">f4"), 4), 0x0E: (np.dtype(">f8"), 8)}


def _read_idx(path: str, want_ndim: int) -> np.ndarray:
    with open(path, "rb") as f:
        data = f.read()
    if len(data) < 4:
        raise IdxFormatError(f"{path}: truncated header at offset 0: expected 4 bytes, got {len(data)}")
    zero, dtype_code, ndim = struct.unpack(">HBB", data[:4])
    magic = struct.unpack(">I", data[:4])[0]
    if zero != 0 or dtype_code not in _IDX_TYPES or ndim != want_ndim:
        raise IdxFormatError(f"{path}: bad magic 0x{magic:08x} at offset 0 (expected 0x{0x0800 | want_ndim:08x} "
                             f"for {want_ndim}-d unsigned-byte data)")
    hdr = 4 + 4 * ndim
    if len(data) < hdr:
        raise IdxFormatError(f"{path}: truncated header at offset 4: expected {hdr} bytes, got {len(data)}")
    dims = struct.unpack(">" + "I" * ndim, data[4:hdr])
    dt, size = _IDX_TYPES[dtype_code]
    need = hdr + size * int(np.prod(dims, dtype=np.int64))
    if len(data) < need:
        raise IdxFormatError(f"{path}: truncated payload at offset {hdr}: expected {need} bytes, got {len(data)}")
    return np.frombuffer(data, dtype=dt, count=int(np.prod(dims, dtype=np.int64)), offset=hdr).reshape(dims)


def load_idx_images(path: str, labels_path: str = "") -> tuple:
    """IDX images (magic 0x00000803, big-endian dims) scaled to [0, 1] float32 as (n, 1, H, W), and the IDX
    labels (0x00000801) if given. Errors: bad magic / truncation (naming the byte offset
    and the expected vs actual byte counts) and an image/label count mismatch — all ``IdxFormatError``."""
    img = _read_idx(path, 3)
    x = (img.astype(np.float32) / 255.0)[:, None]
    if not labels_path:
        return x, None
    lab = _read_idx(labels_path, 1).astype(np.int64)
    if lab.shape[0] != img.shape[0]:
        raise IdxFormatError(f"{labels_path}: {lab.shape[0]} labels for {img.shape[0]} images")
    return x, lab


def write_idx(path: str, array: np.ndarray) -> None:
    """Write an unsigned-byte IDX file (test fixtures and user conversions)."""
    a = np.ascontiguousarray(array, dtype=np.uint8)
    with open(path, "wb") as f:
        f.write(struct.pack(">HBB", 0, 0x08, a.ndim))
        f.write(struct.pack(">" + "I" * a.ndim, *a.shape))
        f.write(a.tobytes())


def make_dataset(spec: DatasetSpec) -> tuple:
    """(x, y) host arrays for a spec: classification (float32, int64), segmentation (float32, uint8 mask),
    IDX images (float32 in [0, 1], int64 labels)."""
    spec.validate()
    if spec.kind == "synthetic_classification":
        return gen_synthetic_classification(spec)
    if spec.kind == "synthetic_segmentation":
        return gen_synthetic_segmentation(spec)
    return load_idx_images(spec.path, spec.labels_path)
