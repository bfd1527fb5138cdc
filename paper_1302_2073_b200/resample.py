"""Resampling shell on the device.

`resample` is the reference's bilinear, half-pixel-centred per-plane frame
resampling (pipeline.py:164-193) and `upsample_mask` its nearest-neighbour
label upsampling (pipeline.py:245-258), both as sm_100a kernels behind the
C-ABI (`prost_resample`, `prost_upsample_mask`).  They compute in fp64 with
the reference's operation order, so the results equal numpy's bit for bit.
Identity sizes return the input unchanged, as the reference does.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as nat
from .errors import DimensionError
from .frames import FrameBuffer, SegmentationMask

__all__ = ["resample", "resample_device", "upsample_mask"]

_CODES = {np.dtype(np.float32): nat.F32, np.dtype(np.float64): nat.F64, np.dtype(np.uint8): nat.U8}


def resample_device(src, channels: int, width: int, height: int, out_w: int, out_h: int,
                    out_dtype=None, cuda_stream: int = 0):
    """Bilinear resampling of a channel-planar device tensor (float32, float64
    or uint8 / 255) into a new float device tensor of C * out_w * out_h values."""
    import torch

    if out_w < 1 or out_h < 1:
        raise DimensionError(f"bad target dimensions {out_w}x{out_h}")
    if src.numel() != channels * width * height:
        raise DimensionError(f"frame holds {src.numel()} values, expected "
                             f"{channels} x {width} x {height}")
    code = {torch.float32: nat.F32, torch.float64: nat.F64, torch.uint8: nat.U8}[src.dtype]
    out_dtype = out_dtype or (torch.float64 if src.dtype == torch.float64 else torch.float32)
    dst = torch.empty(channels * out_w * out_h, dtype=out_dtype, device=src.device)
    rc = nat.lib().prost_resample(
        ctypes.c_void_p(src.contiguous().data_ptr()), code, channels, width, height,
        ctypes.c_void_p(dst.data_ptr()), nat.F64 if out_dtype == torch.float64 else nat.F32,
        out_w, out_h, ctypes.c_void_p(cuda_stream))
    nat.check(rc, None, "resample")
    return dst


def resample(frame: FrameBuffer, out_w: int, out_h: int, device: int = 0) -> FrameBuffer:
    """pipeline.py:164-193 on the device; returns a host FrameBuffer (f8 data)."""
    import torch

    if out_w < 1 or out_h < 1:
        raise DimensionError(f"bad target dimensions {out_w}x{out_h}")
    if (out_w, out_h) == (frame.width, frame.height):
        return frame
    src = torch.from_numpy(np.ascontiguousarray(frame.data)).to(f"cuda:{device}")
    out = resample_device(src, frame.channels, frame.width, frame.height, out_w, out_h,
                          out_dtype=torch.float64)
    return FrameBuffer(out_w, out_h, frame.channels, out.cpu().numpy())


def upsample_mask(mask: SegmentationMask, out_w: int, out_h: int, device: int = 0) -> SegmentationMask:
    """pipeline.py:245-258 on the device."""
    import torch

    if out_w < 1 or out_h < 1:
        raise DimensionError(f"bad target dimensions {out_w}x{out_h}")
    if (out_w, out_h) == (mask.width, mask.height):
        return mask
    src = torch.from_numpy(np.ascontiguousarray(mask.labels, dtype=np.uint8)).to(f"cuda:{device}")
    dst = torch.empty(out_w * out_h, dtype=torch.uint8, device=src.device)
    rc = nat.lib().prost_upsample_mask(ctypes.c_void_p(src.data_ptr()), mask.width, mask.height,
                                       ctypes.c_void_p(dst.data_ptr()), out_w, out_h,
                                       ctypes.c_void_p(0))
    nat.check(rc, None, "upsample_mask")
    return SegmentationMask(out_w, out_h, dst.cpu().numpy())
