"""PROSTSNAP1 snapshots of a tracker state.

Byte-compatible with the reference (tracker.py:42, 159-285): the same magic,
header, parameter hash, little-endian f8 arrays and optional preprocessing
block, so a snapshot written by either implementation restores in the other
(`StreamTracker.restore_bytes` / `/sessions/from-snapshot` in the reference).
The device state is fp32 by default; a snapshot of it carries the fp32 values
widened to f8 (exact), and a restore rounds the f8 basis to the handle's
precision.  Like the reference, the format does not carry the QR counter: a
restored basis starts a fresh 1000-step period (manifold.py:49-78 default).
"""

from __future__ import annotations

import hashlib
import struct

import numpy as np

from .errors import SnapshotError
from .params import ProstParams

__all__ = ["SNAPSHOT_MAGIC", "params_hash", "pack_snapshot", "unpack_snapshot", "save_snapshot",
           "load_snapshot"]

SNAPSHOT_MAGIC = b"PROSTSNAP1"  # tracker.py:42


def params_hash(params: ProstParams) -> int:
    """Stable 64-bit digest of the resolved parameter set (tracker.py:159-181):
    sha256 of the '|'-joined reprs, first 8 bytes little-endian."""
    canonical = "|".join(repr(v) for v in (
        params.k, params.cfg.p, params.cfg.mu, params.delta, params.omega, params.t_init,
        params.t_min, params.tau, params.cg.max_iters, params.cg.grad_tol,
        params.cg.initial_step, params.cg.shrink, params.cg.sufficient_decrease,
        params.cg.max_backtracks))
    return struct.unpack("<Q", hashlib.sha256(canonical.encode()).digest()[:8])[0]


def pack_snapshot(state, params: ProstParams) -> bytes:
    """tracker.py:184-214: header, basis (row-major m x k), y, weights, preproc."""
    U = np.asarray(state.basis.data)
    m, k = U.shape
    pre = state.preproc
    parts = [
        SNAPSHOT_MAGIC,
        struct.pack("<IIQQB", m, k, int(state.frame_index), params_hash(params),
                    1 if pre is not None else 0),
        U.astype("<f8").tobytes(order="C"),
        np.asarray(state.y).astype("<f8").tobytes(),
        np.asarray(state.weights).astype("<f8").tobytes(),
    ]
    if pre is not None:
        parts.append(struct.pack("<IBQddQd", pre.mean.size, 1 if pre.frozen else 0,
                                 int(pre.frames_seen), float(pre.value_sum),
                                 float(pre.value_sumsq), int(pre.value_count), float(pre.std)))
        parts.append(np.asarray(pre.mean).astype("<f8").tobytes())
    return b"".join(parts)


def unpack_snapshot(blob: bytes, params: ProstParams, source: str = "<bytes>"):
    """tracker.py:230-285: (U, y, weights, frame_index, preproc or None); raises
    SnapshotError on a foreign, truncated or differently-parameterized blob."""
    from .tracker import PreprocSnapshot

    if not blob.startswith(SNAPSHOT_MAGIC):
        raise SnapshotError(f"{source}: not a tracker snapshot")
    offset = len(SNAPSHOT_MAGIC)

    def take(fmt):
        nonlocal offset
        size = struct.calcsize(fmt)
        if offset + size > len(blob):
            raise SnapshotError(f"{source}: truncated snapshot")
        vals = struct.unpack_from(fmt, blob, offset)
        offset += size
        return vals

    def take_array(count):
        nonlocal offset
        size = count * 8
        if offset + size > len(blob):
            raise SnapshotError(f"{source}: truncated snapshot")
        arr = np.frombuffer(blob, dtype="<f8", count=count, offset=offset).copy()
        offset += size
        return arr

    m, k, frame_index, stored_hash, has_pre = take("<IIQQB")
    if stored_hash != params_hash(params):
        raise SnapshotError(f"{source}: snapshot was written with different parameters")
    if k != params.k:
        raise SnapshotError(f"{source}: snapshot k={k} does not match params k={params.k}")
    U = take_array(m * k).reshape(m, k)
    y = take_array(k)
    weights = take_array(m)
    pre = None
    if has_pre:
        length, frozen, seen, vsum, vsumsq, vcount, std = take("<IBQddQd")
        pre = PreprocSnapshot(mean=take_array(length), frames_seen=seen, frozen=bool(frozen),
                              std=std, value_sum=vsum, value_sumsq=vsumsq, value_count=vcount)
    return U, y, weights, frame_index, pre


def save_snapshot(state, params: ProstParams, path) -> None:
    with open(path, "wb") as fh:
        fh.write(pack_snapshot(state, params))


def load_snapshot(path, params: ProstParams):
    with open(path, "rb") as fh:
        blob = fh.read()
    return unpack_snapshot(blob, params, source=str(path))
