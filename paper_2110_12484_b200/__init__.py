"""B200-native Micro-Batch Streaming (arXiv 2110.12484).

Drop-in for the reference package ``mbstream``'s hot path (engine / optim /
tensor / memory / streaming APIs, same names and exception types), running
on hand-written sm_100a kernels behind the C-ABI ``libmbs_native.so``
(``include/mbs.h``): K1 fused normalise+accumulate+grad-norm, K2 staging,
K3 fused optimizer step, plus the pinned H2D micro-batch streamer; K5 runs the
model's micro-batch BatchNorm (+ReLU/+skip add) when a model is passed through
``bn.fuse_batchnorm``.
"""

from . import _native, bn, pool, refspec, stem
from .engine import (NORMALIZATION_MODES, EpochStats, GradientAccumulator, MicroBatchPlan, MiniBatchStats,
                     accumulate, make_streamer, mini_batch_gradient, normalization_factor, normalize_loss,
                     plan_split, train_epoch, train_mini_batch)
from .errors import (AccumulatorOverflowError, ConfigError, GradientKeyMismatchError, IdxFormatError,
                     ModelDoesNotFitError, NonFiniteError, ShapeCompositionError, TapeConsumedError)
from .losses import LossValue, accuracy, compute_loss, dice_coefficient, iou
from .optim import OptimizerState, adam_state, adam_step, apply_update, linear_lr, sgd_state, sgd_step
from .rng import epoch_order, named_stream, stream_key
from .streamer import MicroBatchStreamer, Staging
from .tensor import GradientSet, ParameterSet, ParamLayout

__all__ = [
    "NORMALIZATION_MODES", "EpochStats", "GradientAccumulator", "MicroBatchPlan", "MiniBatchStats", "accumulate",
    "make_streamer", "mini_batch_gradient", "normalization_factor", "normalize_loss", "plan_split", "train_epoch",
    "train_mini_batch", "AccumulatorOverflowError", "ConfigError", "GradientKeyMismatchError", "IdxFormatError",
    "ModelDoesNotFitError", "NonFiniteError", "ShapeCompositionError", "TapeConsumedError", "LossValue",
    "accuracy", "compute_loss", "dice_coefficient", "iou", "OptimizerState", "adam_state", "adam_step",
    "apply_update", "linear_lr", "sgd_state", "sgd_step", "epoch_order", "named_stream", "stream_key",
    "MicroBatchStreamer", "Staging", "GradientSet", "ParameterSet", "ParamLayout",
]
