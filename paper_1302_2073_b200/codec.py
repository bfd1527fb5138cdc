"""Binary netpbm (P5 / P6) decode with the pixel unpack on the device
(reference frameio.py:92-137).

The header is parsed on the host exactly as the reference does (same checks,
same CodecError messages); the interleaved payload is uploaded as bytes and
unpacked to channel-planar intensities on [0, 1] by `prost_unpack_pnm`
(x / 255 in fp64, bit-identical to the reference's numpy decode).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as nat
from .errors import CodecError
from .frames import FrameBuffer

__all__ = ["parse_pnm_header", "decode_pnm", "decode_pnm_device"]


def parse_pnm_header(blob: bytes, path="<bytes>"):
    """(magic, width, height, payload offset) of a binary netpbm file (frameio.py:92-117)."""
    magic = blob[:2]
    if magic not in (b"P5", b"P6"):
        raise CodecError(f"{path}: unsupported magic number {magic!r}")
    pos = 2
    fields = []
    while len(fields) < 3:
        while pos < len(blob) and blob[pos:pos + 1].isspace():
            pos += 1
        start = pos
        while pos < len(blob) and not blob[pos:pos + 1].isspace():
            pos += 1
        if start == pos:
            raise CodecError(f"{path}: truncated header")
        try:
            fields.append(int(blob[start:pos]))
        except ValueError as exc:
            raise CodecError(f"{path}: malformed header field {blob[start:pos]!r}") from exc
    width, height, maxval = fields
    if maxval != 255:
        raise CodecError(f"{path}: only maxval 255 is supported, got {maxval}")
    if width < 1 or height < 1:
        raise CodecError(f"{path}: bad dimensions {width}x{height}")
    return magic, width, height, pos + 1  # one whitespace byte before the payload


def decode_pnm_device(blob: bytes, path="<bytes>", device: int = 0, dtype=None, cuda_stream: int = 0):
    """(planar device tensor on [0, 1], width, height, channels)."""
    import torch

    magic, width, height, offset = parse_pnm_header(blob, path)
    channels = 1 if magic == b"P5" else 3
    count = width * height * channels
    payload = blob[offset:offset + count]
    if len(payload) < count:
        raise CodecError(f"{path}: truncated payload ({len(payload)} of {count} bytes)")
    raw = torch.frombuffer(bytearray(payload), dtype=torch.uint8).to(f"cuda:{device}")
    dtype = dtype or torch.float64
    out = torch.empty(count, dtype=dtype, device=raw.device)
    rc = nat.lib().prost_unpack_pnm(ctypes.c_void_p(raw.data_ptr()), channels, width * height,
                                    ctypes.c_void_p(out.data_ptr()),
                                    nat.F64 if dtype == torch.float64 else nat.F32,
                                    ctypes.c_void_p(cuda_stream))
    nat.check(rc, None, "unpack_pnm")
    return out, width, height, channels


def decode_pnm(blob: bytes, path="<bytes>", device: int = 0) -> FrameBuffer:
    """frameio.py:120-137: a host FrameBuffer (f8), decoded on the device."""
    out, width, height, channels = decode_pnm_device(blob, path, device)
    return FrameBuffer(width, height, channels, out.cpu().numpy())
