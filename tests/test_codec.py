"""Binary netpbm decode (reference frameio.py:92-137),
pinned to the reference's decode_pnm on P5 / P6 bytes with varied header
whitespace (tests/golden/pnm_vectors.npz, made by tests/golden/make_golden.py).

CPU: header parsing and its CodecErrors.  GPU: the device unpack equals the
reference's decode bit for bit."""

from pathlib import Path

import numpy as np
import pytest

import paper_1302_2073_b200 as pkg
from paper_1302_2073_b200.codec import parse_pnm_header

GOLD = Path(__file__).resolve().parent / "golden" / "pnm_vectors.npz"


def _cases():
    z = np.load(GOLD)
    i = 0
    while f"dims{i}" in z:
        yield z[f"blob{i}"].tobytes(), z[f"data{i}"], z[f"dims{i}"]
        i += 1


def test_header_parsing():
    for blob, data, (w, h, c) in _cases():
        magic, width, height, off = parse_pnm_header(blob)
        assert (width, height) == (w, h) and magic == (b"P5" if c == 1 else b"P6")
        assert len(blob) - off >= w * h * c
    for bad, msg in ((b"P3\n1 1\n255\n\x00", "unsupported magic"), (b"P5\n4 4\n", "truncated header"),
                     (b"P5\n4 x\n255\n", "malformed header"), (b"P5\n4 4\n65535\n", "maxval"),
                     (b"P5\n0 4\n255\n", "bad dimensions")):
        with pytest.raises(pkg.CodecError, match=msg):
            parse_pnm_header(bad)


@pytest.mark.gpu
def test_device_decode_matches_reference():
    from paper_1302_2073_b200.codec import decode_pnm

    for blob, data, (w, h, c) in _cases():
        fb = decode_pnm(blob)
        assert (fb.width, fb.height, fb.channels) == (w, h, c)
        np.testing.assert_array_equal(fb.data, data)
    with pytest.raises(pkg.CodecError, match="truncated payload"):
        decode_pnm(b"P5\n4 4\n255\n" + bytes(3))
