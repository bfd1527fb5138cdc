"""Confusion counts on the device.

`accumulate(counts, predicted, truth)` mirrors the reference's
`evaluate.accumulate` (evaluate.py:87-106): pixels whose ground-truth gray
level is 85 (outside ROI) or 170 (unknown) are not scored, 255 is foreground,
every other level background.  `accumulate_device` scores a batch of masks
that are already on the device (e.g. a BatchTracker's mask output) against
device ground truth, one row of counts per stream, without a host round trip.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .errors import DimensionError
from .frames import SegmentationMask

__all__ = ["ConfusionCounts", "accumulate", "accumulate_device"]


@dataclass(frozen=True)
class ConfusionCounts:
    """Pooled per-pixel classification counts; merge by addition (evaluate.py:52-68)."""

    tp: int = 0
    fp: int = 0
    tn: int = 0
    fn: int = 0

    def __add__(self, other: "ConfusionCounts") -> "ConfusionCounts":
        return ConfusionCounts(self.tp + other.tp, self.fp + other.fp, self.tn + other.tn,
                               self.fn + other.fn)

    @property
    def total(self) -> int:
        return self.tp + self.fp + self.tn + self.fn


def accumulate_device(counts, masks, truths, mask_stride: int = 0, cuda_stream: int = 0) -> None:
    """counts: int64 [S, 4] device tensor (tp, fp, tn, fn), incremented in place;
    masks: uint8 device tensor with S rows of `mask_stride` bytes (default:
    the pixel count); truths: uint8 device tensor [S, pixels]."""
    import torch

    S, P = truths.shape
    stride = mask_stride or P
    if counts.shape != (S, 4) or counts.dtype != torch.int64:
        raise DimensionError("counts must be an int64 [S, 4] tensor")
    if masks.numel() < (S - 1) * stride + P or truths.dtype != torch.uint8 or masks.dtype != torch.uint8:
        raise DimensionError("masks / truths must be uint8 and cover every stream")
    rc = nat.lib().prost_confusion(ctypes.c_void_p(masks.data_ptr()), stride,
                                   ctypes.c_void_p(truths.contiguous().data_ptr()), S, P,
                                   ctypes.c_void_p(counts.data_ptr()), ctypes.c_void_p(cuda_stream))
    nat.check(rc, None, "confusion")


def accumulate(counts: ConfusionCounts, predicted: SegmentationMask, truth, device: int = 0) -> ConfusionCounts:
    """Score one frame against its annotation and merge into `counts`
    (evaluate.py:87-106); `truth` has .width, .height and uint8 .labels."""
    import torch

    if (predicted.width, predicted.height) != (truth.width, truth.height):
        raise DimensionError(f"mask {predicted.width}x{predicted.height} does not match "
                             f"ground truth {truth.width}x{truth.height}")
    dev = f"cuda:{device}"
    m = torch.from_numpy(np.ascontiguousarray(predicted.labels, dtype=np.uint8)).to(dev)
    g = torch.from_numpy(np.ascontiguousarray(truth.labels, dtype=np.uint8)).to(dev)[None]
    c = torch.zeros((1, 4), dtype=torch.int64, device=dev)
    accumulate_device(c, m, g)
    tp, fp, tn, fn = (int(v) for v in c.cpu().numpy()[0])
    return counts + ConfusionCounts(tp, fp, tn, fn)
