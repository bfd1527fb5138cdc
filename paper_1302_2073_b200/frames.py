"""Frame and mask containers, mirroring pipeline.py:37-96 and jobs.py:142-151."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import DimensionError

__all__ = ["FrameBuffer", "SegmentationMask", "FrameRecord"]


@dataclass
class FrameBuffer:
    """A vectorized 1- or 3-channel image on [0, 1], channel-planar (pipeline.py:37-74)."""

    width: int
    height: int
    channels: int
    data: np.ndarray

    def __post_init__(self):
        if self.channels not in (1, 3):
            raise DimensionError(f"channels must be 1 or 3, got {self.channels}")
        if self.width < 1 or self.height < 1:
            raise DimensionError(f"bad dimensions {self.width}x{self.height}")
        expected = self.width * self.height * self.channels
        if self.data.shape != (expected,):
            raise DimensionError(
                f"data length {self.data.shape} does not match "
                f"{self.width}x{self.height}x{self.channels}"
            )

    @property
    def pixels(self) -> int:
        return self.width * self.height

    def planes(self) -> np.ndarray:
        return self.data.reshape(self.channels, self.height, self.width)

    def to_gray(self) -> "FrameBuffer":
        """Average the planes (pipeline.py:69-74)."""
        if self.channels == 1:
            return self
        gray = self.planes().mean(axis=0)
        return FrameBuffer(self.width, self.height, 1, gray.reshape(-1))


@dataclass
class SegmentationMask:
    """Per-pixel labels: 0 background, 1 foreground, row-major (pipeline.py:77-96)."""

    width: int
    height: int
    labels: np.ndarray

    def __post_init__(self):
        if self.labels.shape != (self.width * self.height,):
            raise DimensionError(
                f"labels length {self.labels.shape} does not match {self.width}x{self.height}"
            )

    def grid(self) -> np.ndarray:
        return self.labels.reshape(self.height, self.width)

    def foreground_fraction(self) -> float:
        return float(np.mean(self.labels != 0))


@dataclass
class FrameRecord:
    """What one pushed frame produced, at model resolution (jobs.py:142-151)."""

    frame_index: int
    mask: SegmentationMask
    raw_mask: SegmentationMask
    residual: np.ndarray
    fit_cost: float
    step: float
