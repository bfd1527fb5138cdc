"""Device-backed trackers with the reference's Python API.

`StreamTracker(RunConfig).push(FrameBuffer) -> FrameRecord` and
`background_frame()` mirror `jobs.py:154-239`; `process_frame(state, x,
params)` mirrors `tracker.py:121-156`; `BatchTracker` runs many independent
streams in every launch (the batched form `BASELINE.json` measures).  All
per-frame arithmetic runs in the CUDA library behind the C-ABI
(include/prost_b200.h); the host only draws the initial basis with the same
numpy calls as the reference (manifold.py:100-113), so U0 is bit-identical.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _native as nat
from .errors import ConfigError, DimensionError, SequenceError
from .frames import FrameBuffer, FrameRecord, SegmentationMask
from .params import DEFAULT_I_INIT, ProstParams, RunConfig, step_size, to_native

__all__ = [
    "ORTHONORMALITY_TOL",
    "SubspaceBasis",
    "TrackerState",
    "FitResult",
    "PreprocSnapshot",
    "random_orthonormal",
    "bootstrap",
    "process_frame",
    "StreamTracker",
    "BatchTracker",
]

ORTHONORMALITY_TOL = 1e-8  # manifold.py:36
PRECISIONS = {"fp32": 0, "fp64": nat.FLAG_FP64}


def _drift(data: np.ndarray) -> float:
    return float(np.linalg.norm(data.T @ data - np.eye(data.shape[1])))


@dataclass
class SubspaceBasis:
    """m x k matrix with orthonormal columns (manifold.py:49-78).

    `check=False` skips the drift validation for bases read back from an fp32
    device state, whose drift sits at fp32 rounding (~1e-7), above the
    reference's fp64 tolerance.
    """

    data: np.ndarray
    steps_since_qr: int = field(default=0, compare=False)
    check: bool = field(default=True, compare=False, repr=False)

    def __post_init__(self):
        if self.data.ndim != 2:
            raise DimensionError(f"basis must be a matrix, got shape {self.data.shape}")
        m, k = self.data.shape
        if not 1 <= k < m:
            raise DimensionError(f"need 1 <= k < m, got m={m}, k={k}")
        if self.check:
            drift = _drift(self.data)
            if drift > ORTHONORMALITY_TOL:
                raise DimensionError(
                    f"columns are not orthonormal (drift {drift:.3e} > {ORTHONORMALITY_TOL})"
                )

    @property
    def m(self) -> int:
        return self.data.shape[0]

    @property
    def k(self) -> int:
        return self.data.shape[1]


@dataclass
class PreprocSnapshot:
    """Host copy of the running statistics (pipeline.py:99-118 fields)."""

    mean: np.ndarray
    frames_seen: int = 0
    frozen: bool = False
    std: float = 0.0
    value_sum: float = 0.0
    value_sumsq: float = 0.0
    value_count: int = 0


@dataclass
class TrackerState:
    """Everything the loop carries between frames (tracker.py:79-87)."""

    basis: SubspaceBasis
    y: np.ndarray
    weights: np.ndarray
    frame_index: int = 0
    preproc: Optional[PreprocSnapshot] = None


@dataclass
class FitResult:
    """fit.py:50-63: the fitted coordinates, the residual x - U y at them
    (before the geodesic step; the residual against the updated basis is the
    second return value of `process_frame`), the cost and the counters."""

    y: np.ndarray
    residual: Optional[np.ndarray]
    cost: float
    iterations: int
    cost_evals: int
    grad_evals: int


def random_orthonormal(m: int, k: int, seed: int) -> SubspaceBasis:
    """Uniformly random k-dim subspace: Gaussian draw, thin QR, sign fix
    (manifold.py:100-113), drawn with the same numpy calls so it is
    bit-identical to the reference's bootstrap basis."""
    if not 1 <= k < m:
        raise DimensionError(f"need 1 <= k < m, got m={m}, k={k}")
    rng = np.random.default_rng(seed)
    gauss = rng.standard_normal((m, k))
    q, r = np.linalg.qr(gauss)
    q = q * np.where(np.diag(r) < 0.0, -1.0, 1.0)
    return SubspaceBasis(q)


def rewrap_fp64(state: TrackerState) -> TrackerState:
    """Export form of an fp32 device state for the reference's types.

    The fp32 basis drifts from orthonormality by ~1e-7 after some frames, and
    the reference's `SubspaceBasis` rejects drift > 1e-8 (manifold.py:66-70),
    so an exported basis is re-orthonormalized on the host in fp64 with the
    reference's own QR + sign fix (manifold.py:111-112, 192-196): U = Q R,
    diag(R) > 0.  The coordinates become R y so that the reconstruction U y
    (the background, jobs.py:231-239) is unchanged.  The subspace, weights,
    frame index and running statistics are carried over as they are."""
    U = np.asarray(state.basis.data, dtype=np.float64)
    q, r = np.linalg.qr(U)
    sign = np.where(np.diag(r) < 0.0, -1.0, 1.0)
    q = q * sign
    r = sign[:, None] * r
    y = r @ np.asarray(state.y, dtype=np.float64)
    return TrackerState(SubspaceBasis(q, steps_since_qr=0), y, state.weights, state.frame_index,
                        state.preproc)


def bootstrap(m: int, params: ProstParams, seed: int) -> TrackerState:
    """Fresh state: random orthonormal basis, zero coordinates, unit weights
    (tracker.py:106-118)."""
    basis = random_orthonormal(m, params.k, seed)
    return TrackerState(basis=basis, y=np.zeros(params.k), weights=np.ones(m), frame_index=0)


# ---------------------------------------------------------------------------
# native handle


def _is_torch(a) -> bool:
    return type(a).__module__.startswith("torch")


def _buffer(a, writable=False):
    """(pointer, dtype code, on_device, element count) of a numpy array or torch tensor."""
    if _is_torch(a):
        import torch

        if not a.is_contiguous():
            raise DimensionError("tensor must be contiguous")
        code = {torch.float32: nat.F32, torch.float64: nat.F64, torch.uint8: nat.U8}.get(a.dtype)
        if code is None:
            raise ConfigError(f"unsupported tensor dtype {a.dtype}")
        return ctypes.c_void_p(a.data_ptr()), code, 1 if a.is_cuda else 0, a.numel()
    if not isinstance(a, np.ndarray):
        raise ConfigError(f"expected a numpy array or torch tensor, got {type(a)}")
    if not a.flags.c_contiguous or (writable and not a.flags.writeable):
        raise DimensionError("array must be C-contiguous (and writable for outputs)")
    code = {np.dtype(np.float32): nat.F32, np.dtype(np.float64): nat.F64,
            np.dtype(np.uint8): nat.U8}.get(a.dtype)
    if code is None:
        raise ConfigError(f"unsupported array dtype {a.dtype}")
    return ctypes.c_void_p(a.ctypes.data), code, 0, a.size


class FitInfoBuffer:
    """Pinned host array of n `prost_fit_info` records for asynchronous
    delivery (`push(..., fit_out=buf)`); read it after the push is joined."""

    def __init__(self, n: int):
        import torch

        self.n = n
        self._t = torch.empty(n * ctypes.sizeof(nat.FitInfo), dtype=torch.uint8).pin_memory()
        self.ptr = self._t.data_ptr()
        self.nbytes = n * ctypes.sizeof(nat.FitInfo)

    def records(self):
        arr = (nat.FitInfo * self.n).from_address(self.ptr)
        return [arr[i] for i in range(self.n)]

    def fit_costs(self) -> np.ndarray:
        return np.array([r.fit_cost for r in self.records()])


class NativeTracker:
    """Owns one C-ABI handle: n_streams trackers sharing a parameter set."""

    def __init__(self, params: ProstParams, width: int, height: int, channels: int,
                 n_streams: int = 1, i_init: int = DEFAULT_I_INIT, pipeline: bool = True,
                 precision: str = "fp32", device: int = 0, latency: bool = False):
        if precision not in PRECISIONS:
            raise ConfigError(f"precision must be one of {sorted(PRECISIONS)}, got {precision!r}")
        self._lib = nat.lib()
        self.params = params
        self.width, self.height, self.channels = width, height, channels
        self.n_streams = n_streams
        self.precision = precision
        self.pipeline = pipeline
        self.m = width * height * channels
        self.pixels = width * height
        flags = (PRECISIONS[precision] | (nat.FLAG_PIPELINE if pipeline else 0)
                 | (nat.FLAG_LATENCY if latency else 0))
        h = ctypes.c_void_p()
        native = to_native(params, width, height, channels, i_init)
        rc = self._lib.prost_create(ctypes.byref(native), n_streams, flags, device, ctypes.byref(h))
        self._h = h
        if rc != nat.PROST_OK:
            msg = nat.last_error(h) if h.value else ""
            self.close()
            raise nat.error_class(rc)(msg or f"prost_create failed with status {rc}")
        self._fit = (nat.FitInfo * n_streams)()

    def close(self) -> None:
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._lib.prost_destroy(h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc: int, what: str) -> None:
        nat.check(rc, self._h, what)

    # -- state ---------------------------------------------------------------
    def set_core_state(self, stream: int, U=None, y=None, weights=None, frame_index: int = 0,
                       steps_since_qr: int = 0) -> None:
        U = None if U is None else np.ascontiguousarray(U, dtype=np.float64)
        y = None if y is None else np.ascontiguousarray(y, dtype=np.float64)
        w = None if weights is None else np.ascontiguousarray(weights, dtype=np.float64)
        if U is not None and U.shape != (self.m, self.params.k):
            raise DimensionError(f"basis must have shape ({self.m}, {self.params.k}), got {U.shape}")
        if y is not None and y.shape != (self.params.k,):
            raise DimensionError(f"coordinates must have shape ({self.params.k},), got {y.shape}")
        if w is not None and w.shape != (self.m,):
            raise DimensionError(f"weights must have shape ({self.m},), got {w.shape}")
        self._check(self._lib.prost_set_core_state(self._h, stream, nat.dptr(U), nat.dptr(y),
                                                   nat.dptr(w), frame_index, steps_since_qr),
                    "set_core_state")

    def get_core_state(self, stream: int = 0):
        U = np.empty((self.m, self.params.k))
        y = np.empty(self.params.k)
        w = np.empty(self.m)
        fi = ctypes.c_int64()
        sq = ctypes.c_int64()
        self._check(self._lib.prost_get_core_state(self._h, stream, nat.dptr(U), nat.dptr(y),
                                                   nat.dptr(w), ctypes.byref(fi), ctypes.byref(sq)),
                    "get_core_state")
        return U, y, w, fi.value, sq.value

    def set_preproc(self, stream: int, snap: PreprocSnapshot) -> None:
        mean = np.ascontiguousarray(snap.mean, dtype=np.float64)
        sc = np.array([snap.value_sum, snap.value_sumsq, snap.value_count, snap.frames_seen,
                       1.0 if snap.frozen else 0.0, snap.std], dtype=np.float64)
        self._check(self._lib.prost_set_preproc(self._h, stream, nat.dptr(mean), nat.dptr(sc)),
                    "set_preproc")

    def get_preproc(self, stream: int = 0) -> PreprocSnapshot:
        mean = np.empty(self.m)
        sc = np.empty(6)
        self._check(self._lib.prost_get_preproc(self._h, stream, nat.dptr(mean), nat.dptr(sc)),
                    "get_preproc")
        return PreprocSnapshot(mean=mean, frames_seen=int(sc[3]), frozen=bool(sc[4]),
                               std=float(sc[5]), value_sum=float(sc[0]),
                               value_sumsq=float(sc[1]), value_count=int(sc[2]))

    # -- frames --------------------------------------------------------------
    def push(self, frames, background=None, residual=None, mask=None, raw_mask=None,
             fit: bool = True, cuda_stream: int = 0, fit_residual=None, fit_out=None):
        """Enqueue one frame per stream.  Outputs are numpy arrays or torch
        tensors (host or device) to fill.  With fit=True the call waits and
        returns the per-stream `prost_fit_info` array.  `fit_residual` receives
        x - U y after the fit, before the geodesic step (FitResult.residual).
        `fit_out` (a `FitInfoBuffer`) receives the per-stream FitInfo without
        synchronizing: it is valid after `join` / `synchronize`, and host-I/O
        pushes stay pipelined."""
        fp, fdt, fdev, out = self._frame_and_outputs(frames, background, residual, mask,
                                                     raw_mask, fit and fit_out is None, fit_residual)
        if fit_out is not None:
            out.fit = ctypes.cast(ctypes.c_void_p(fit_out.ptr), ctypes.POINTER(nat.FitInfo))
            out.fit_async = 1
        rc = self._lib.prost_push(self._h, fp, fdt, fdev, ctypes.byref(out),
                                  ctypes.c_void_p(cuda_stream))
        self._check(rc, "push")
        return self._fit if fit else None

    def push_many(self, frames, background=None, residual=None, mask=None, raw_mask=None,
                  fit: bool = False, cuda_stream: int = 0, fit_residual=None, fit_out=None):
        """F consecutive frames of every stream in one call — frames
        [F, n_streams, m], outputs [F, n_streams, ...] — with each stream's
        slice kept on chip across its F frames (prost_push_many).  The results
        equal F calls of `push`.  With fit=True the call waits and returns the
        F * n_streams `prost_fit_info` records (frame-major)."""
        nf = int(frames.shape[0])
        fp, fdt, fdev, out = self._frame_and_outputs(frames, background, residual, mask,
                                                     raw_mask, False, fit_residual, nframes=nf)
        fit_arr = None
        if fit_out is not None:
            out.fit = ctypes.cast(ctypes.c_void_p(fit_out.ptr), ctypes.POINTER(nat.FitInfo))
            out.fit_async = 1
        elif fit:
            fit_arr = (nat.FitInfo * (nf * self.n_streams))()
            out.fit = ctypes.cast(fit_arr, ctypes.POINTER(nat.FitInfo))
        rc = self._lib.prost_push_many(self._h, fp, nf, fdt, fdev, ctypes.byref(out),
                                       ctypes.c_void_p(cuda_stream))
        self._check(rc, "push_many")
        return fit_arr

    def _frame_and_outputs(self, frames, background, residual, mask, raw_mask, fit,
                           fit_residual=None, nframes: int = 1):
        fp, fdt, fdev, fcount = _buffer(frames)
        if fcount != nframes * self.n_streams * self.m:
            raise DimensionError(
                f"frames hold {fcount} values, expected {nframes} x {self.n_streams} x {self.m}")
        out = nat.Outputs()
        dev_flags = set()
        dtype = None
        for name, arr, count in (("background", background, self.m), ("residual", residual, self.m),
                                 ("fit_residual", fit_residual, self.m),
                                 ("mask", mask, self.pixels), ("raw_mask", raw_mask, self.pixels)):
            if arr is None:
                continue
            p, dt, dev, cnt = _buffer(arr, writable=True)
            if cnt != nframes * self.n_streams * count:
                raise DimensionError(f"{name} holds {cnt} values, expected "
                                     f"{nframes} x {self.n_streams} x {count}")
            if name in ("mask", "raw_mask"):
                if dt != nat.U8:
                    raise ConfigError(f"{name} must be uint8")
            else:
                if dt == nat.U8:
                    raise ConfigError(f"{name} must be float32 or float64")
                if dtype is not None and dt != dtype:
                    raise ConfigError("background and residual must share a dtype")
                dtype = dt
            dev_flags.add(dev)
            setattr(out, name, p)
        if len(dev_flags) > 1:
            raise ConfigError("outputs must all be host or all be device arrays")
        out.dtype = nat.F32 if dtype is None else dtype
        out.on_device = dev_flags.pop() if dev_flags else 0
        if fit:
            out.fit = ctypes.cast(self._fit, ctypes.POINTER(nat.FitInfo))
        return fp, fdt, fdev, out

    # -- exchange (pixel-sharded) mode, include/prost_b200.h --------------
    def set_exchange(self, n_real_global: int) -> None:
        self._check(self._lib.prost_set_exchange(self._h, int(n_real_global)), "set_exchange")

    def exchange_buffer(self):
        """(device pointer, element count) of the float64 exchange buffer."""
        ptr, cnt = ctypes.c_void_p(), ctypes.c_int64()
        self._check(self._lib.prost_xbuffer(self._h, ctypes.byref(ptr), ctypes.byref(cnt)),
                    "xbuffer")
        return ptr.value, cnt.value

    def xbegin(self, frames, background=None, residual=None, mask=None, raw_mask=None,
               fit: bool = False, cuda_stream: int = 0) -> None:
        fp, fdt, fdev, out = self._frame_and_outputs(frames, background, residual, mask,
                                                     raw_mask, fit)
        self._xout = out  # the handle keeps pointers into it until xfinish
        self._xfit = fit
        self._check(self._lib.prost_xbegin(self._h, fp, fdt, fdev, ctypes.byref(out),
                                           ctypes.c_void_p(cuda_stream)), "xbegin")

    def xnext(self, cuda_stream: int = 0) -> bool:
        x = ctypes.c_int32()
        self._check(self._lib.prost_xnext(self._h, ctypes.byref(x), ctypes.c_void_p(cuda_stream)),
                    "xnext")
        return bool(x.value)

    def xapply(self, cuda_stream: int = 0) -> None:
        self._check(self._lib.prost_xapply(self._h, ctypes.c_void_p(cuda_stream)), "xapply")

    def xedges(self, top, bottom, cuda_stream: int = 0) -> None:
        self._check(self._lib.prost_xedges(self._h, ctypes.c_void_p(top), ctypes.c_void_p(bottom),
                                           ctypes.c_void_p(cuda_stream)), "xedges")

    def xpeer_handle(self, world: int) -> bytes:
        """IPC handle (64 bytes) of this rank's exchange region, sized for `world` ranks."""
        buf = ctypes.create_string_buffer(nat.IPC_HANDLE_BYTES)
        self._check(self._lib.prost_xpeer_handle(self._h, int(world), buf), "xpeer_handle")
        return buf.raw

    def xpeer_open(self, rank: int, world: int, handles) -> None:
        """Map every rank's exchange region (`handles`: the world's IPC handles in
        rank order); prost_push then runs the frame with in-kernel exchanges."""
        blob = b"".join(bytes(hd) for hd in handles)
        if len(blob) != world * nat.IPC_HANDLE_BYTES:
            raise DimensionError(f"{len(blob)} handle bytes for {world} ranks")
        buf = ctypes.create_string_buffer(blob, len(blob))
        self._check(self._lib.prost_xpeer_open(self._h, int(rank), int(world), buf), "xpeer_open")

    def xfinish(self, halo_top=None, halo_bottom=None, cuda_stream: int = 0):
        self._check(self._lib.prost_xfinish(self._h, ctypes.c_void_p(halo_top),
                                            ctypes.c_void_p(halo_bottom),
                                            ctypes.c_void_p(cuda_stream)), "xfinish")
        return self._fit if self._xfit else None

    def background(self, out, cuda_stream: int = 0) -> None:
        p, dt, dev, cnt = _buffer(out, writable=True)
        if cnt != self.n_streams * self.m:
            raise DimensionError(f"background holds {cnt} values, expected {self.n_streams} x {self.m}")
        self._check(self._lib.prost_background(self._h, p, dt, dev, ctypes.c_void_p(cuda_stream)),
                    "background")

    def synchronize(self) -> None:
        self._check(self._lib.prost_synchronize(self._h), "synchronize")

    def join(self, cuda_stream: int = 0) -> None:
        """Make `cuda_stream` wait for pipelined host-I/O pushes in flight."""
        self._check(self._lib.prost_join(self._h, ctypes.c_void_p(cuda_stream)), "join")

    def query(self, what: int) -> int:
        v = ctypes.c_int64()
        self._check(self._lib.prost_query(self._h, what, ctypes.byref(v)), "query")
        return v.value

    def profile(self, enable: bool = True) -> None:
        """Time every launch with CUDA events (per phase); read with profile_read."""
        self._check(self._lib.prost_profile(self._h, 1 if enable else 0), "profile")

    def profile_read(self) -> dict:
        """{phase: (milliseconds, launches)} accumulated since the last read."""
        n = len(nat.PHASES)
        ms = np.zeros(n)
        cnt = (ctypes.c_int64 * n)()
        self._check(self._lib.prost_profile_read(self._h, nat.dptr(ms), cnt, n), "profile_read")
        return {name: (float(ms[i]), int(cnt[i])) for i, name in enumerate(nat.PHASES)}

    def resident_counters(self) -> dict:
        """Per-CTA mean timings (us) of the last profiled resident launch."""
        n = 16
        out = (ctypes.c_int64 * n)()
        self._check(self._lib.prost_resident_counters(self._h, out, n), "resident_counters")
        names = ("kernel_us", "barrier_us", "slots_us", "logic_us", "load_us")
        d = {nm: out[i] / 1e3 for i, nm in enumerate(names)}
        d.update(team_sums=int(out[5]), rounds=int(out[6]), slowest_kernel_us=out[n - 1] / 1e3)
        for i, nm in ((7, "phase_stats_us"), (8, "phase_pass0_us"), (9, "phase_iter_us"),
                      (10, "phase_geo_us"), (12, "iter_sweep_own_us"), (13, "iter_sweep_all_us"),
                      (14, "logic_iter_us")):
            d[nm] = out[i] / 1e3
        return d

    def set_wave(self, streams: int) -> None:
        self._check(self._lib.prost_set_wave(self._h, streams), "set_wave")

    @property
    def launches(self) -> int:
        return self.query(nat.Q_LAUNCHES)


# ---------------------------------------------------------------------------
# functional seam: process_frame (tracker.py:121-156)

_CORE_CACHE: dict = {}


def _core_handle(m: int, params: ProstParams, precision: str, device: int) -> NativeTracker:
    # the kernel-path switches are read at handle creation: key on them too
    key = (m, params, precision, device, os.environ.get("PROST_RESIDENT"),
           os.environ.get("PROST_NO_RESIDENT"), os.environ.get("PROST_KERNEL"))
    h = _CORE_CACHE.get(key)
    if h is None:
        if len(_CORE_CACHE) > 8:
            for old in list(_CORE_CACHE.values()):
                old.close()
            _CORE_CACHE.clear()
        h = NativeTracker(params, m, 1, 1, 1, i_init=1, pipeline=False, precision=precision,
                          device=device)
        _CORE_CACHE[key] = h
    return h


def process_frame(state: TrackerState, x: np.ndarray, params: ProstParams, *,
                  precision: str = "fp32", device: int = 0):
    """Advance the tracker by one preprocessed frame on the GPU.

    Same contract as the reference (tracker.py:121-156): returns
    (new state, residual of x against the updated basis, FitResult), does not
    mutate `state`, raises DimensionError on a shape mismatch and
    NonFiniteError on NaN/Inf before any state change.  Weights must take the
    values {1, omega} (every state the reference itself produces does).
    """
    basis = state.basis
    x = np.asarray(x)
    if x.shape != (basis.m,):
        raise DimensionError(f"frame must have shape ({basis.m},), got {x.shape}")
    if basis.k != params.k:
        raise DimensionError(f"basis has k={basis.k}, params k={params.k}")
    h = _core_handle(basis.m, params, precision, device)
    h.set_core_state(0, basis.data, state.y, state.weights, state.frame_index,
                     basis.steps_since_qr)
    residual = np.empty(basis.m)
    fit_res = np.empty(basis.m)
    info = h.push(np.ascontiguousarray(x, dtype=np.float64), residual=residual, fit=True,
                  fit_residual=fit_res)[0]
    U, y, w, fi, since = h.get_core_state(0)
    new_state = TrackerState(
        basis=SubspaceBasis(U, steps_since_qr=since, check=False),
        y=y, weights=w, frame_index=fi, preproc=state.preproc,
    )
    fit = FitResult(y=y.copy(), residual=fit_res, cost=info.fit_cost, iterations=info.iterations,
                    cost_evals=info.cost_evals, grad_evals=info.grad_evals)
    return new_state, residual, fit


# ---------------------------------------------------------------------------
# stateful seam: StreamTracker (jobs.py:154-239)


class StreamTracker:
    """Stateful frame-in, mask-out pipeline around one device tracker.

    Drop-in for the reference's `StreamTracker` (jobs.py:154-239): dimensions
    are fixed by the first frame, one thread pushes at a time.
    """

    def __init__(self, config: RunConfig, i_init: Optional[int] = None, *,
                 precision: str = "fp32", device: int = 0):
        self.config = config
        self.i_init = i_init if i_init is not None else (
            config.i_init if config.i_init is not None else DEFAULT_I_INIT)
        if self.i_init < 1:
            raise ConfigError(f"i_init must be >= 1, got {self.i_init}")
        self.params = config.params(self.i_init)
        self.precision = precision
        self.device = device
        self.channels: Optional[int] = None
        self._native: Optional[NativeTracker] = None
        self._frame_index = 0

    @property
    def started(self) -> bool:
        return self._native is not None

    @property
    def frame_index(self) -> int:
        return self._frame_index

    def _prepare(self, frame: FrameBuffer):
        """jobs.py:181-184: gray conversion, then bilinear resampling to the
        model resolution.  Returns (channels, data): an off-resolution frame
        is resampled on the device (resample.py, fp64 like the reference) and
        stays there — the push reads the device tensor, with no round trip
        through the host; identity sizes pass the host data through."""
        if self.config.grayscale:
            frame = frame.to_gray()
        if (frame.width, frame.height) != (self.config.target_width, self.config.target_height):
            import torch

            from .resample import resample_device

            src = torch.from_numpy(np.ascontiguousarray(frame.data)).to(f"cuda:{self.device}")
            out = resample_device(src, frame.channels, frame.width, frame.height,
                                  self.config.target_width, self.config.target_height,
                                  out_dtype=torch.float64)
            return frame.channels, out
        return frame.channels, frame.data

    def _start(self, channels: int) -> None:
        w, hgt = self.config.target_width, self.config.target_height
        self.channels = channels
        self._native = NativeTracker(self.params, w, hgt, channels, 1, i_init=self.i_init,
                                     pipeline=True, precision=self.precision, device=self.device,
                                     latency=True)
        m = w * hgt * channels
        U0 = random_orthonormal(m, self.params.k, self.config.seed).data
        self._native.set_core_state(0, U0, np.zeros(self.params.k), None, 0, 0)

    def push(self, frame: FrameBuffer) -> FrameRecord:
        """Run the full pipeline on one frame and advance the model (jobs.py:186-229)."""
        channels, data = self._prepare(frame)
        if self._native is None:
            self._start(channels)
        elif channels != self.channels:
            raise SequenceError(f"frame has {channels} channels, expected {self.channels}")
        n = self._native
        t = step_size(self._frame_index, self.params)
        mask = np.empty(n.pixels, dtype=np.uint8)
        raw = np.empty(n.pixels, dtype=np.uint8)
        residual = np.empty(n.m)
        if isinstance(data, np.ndarray):
            if data.dtype not in (np.float64, np.float32, np.uint8):
                data = data.astype(np.float64)
            data = np.ascontiguousarray(data)
        info = n.push(data, residual=residual, mask=mask, raw_mask=raw, fit=True)[0]
        self._frame_index = int(info.frame_index)
        w, hgt = self.config.target_width, self.config.target_height
        return FrameRecord(
            frame_index=self._frame_index,
            mask=SegmentationMask(w, hgt, mask),
            raw_mask=SegmentationMask(w, hgt, raw),
            residual=residual,
            fit_cost=float(info.fit_cost),
            step=t,
        )

    def background_frame(self) -> FrameBuffer:
        """Current reconstruction on the intensity scale (jobs.py:231-239)."""
        if self._native is None:
            raise ConfigError("no frames pushed yet")
        out = np.empty(self._native.m)
        self._native.background(out)
        return FrameBuffer(self.config.target_width, self.config.target_height, self.channels, out)

    @property
    def state(self) -> TrackerState:
        """Host copy of the device state (tracker.py:79-87)."""
        if self._native is None:
            raise ConfigError("no frames pushed yet")
        U, y, w, fi, since = self._native.get_core_state(0)
        return TrackerState(SubspaceBasis(U, since, check=False), y, w, fi,
                            self._native.get_preproc(0))

    @property
    def stats(self) -> PreprocSnapshot:
        if self._native is None:
            raise ConfigError("no frames pushed yet")
        return self._native.get_preproc(0)

    # -- PROSTSNAP1 snapshots (jobs.py:241-277, tracker.py:184-285) -----------
    def snapshot_bytes(self) -> bytes:
        from .snapshot import pack_snapshot

        if self._native is None:
            raise ConfigError("no frames pushed yet; nothing to snapshot")
        state = self.state
        if self.precision != "fp64":
            state = rewrap_fp64(state)
        return pack_snapshot(state, self.params)

    def save(self, path) -> None:
        with open(path, "wb") as fh:
            fh.write(self.snapshot_bytes())

    def _adopt(self, U, y, weights, frame_index, pre) -> None:
        # jobs.py:251-263: the snapshot's dimension fixes the channel count
        pixels = self.config.target_width * self.config.target_height
        channels, remainder = divmod(U.shape[0], pixels)
        if remainder or channels not in (1, 3):
            raise ConfigError(
                f"snapshot dimension {U.shape[0]} does not match "
                f"{self.config.target_width}x{self.config.target_height} frames")
        w, hgt = self.config.target_width, self.config.target_height
        self.channels = channels
        self._native = NativeTracker(self.params, w, hgt, channels, 1, i_init=self.i_init,
                                     pipeline=True, precision=self.precision, device=self.device,
                                     latency=True)
        self._native.set_core_state(0, np.ascontiguousarray(U), y, weights, int(frame_index), 0)
        if pre is None:
            pre = PreprocSnapshot(mean=np.zeros(U.shape[0]))
        self._native.set_preproc(0, pre)
        self._frame_index = int(frame_index)

    @classmethod
    def restore_bytes(cls, blob: bytes, config: RunConfig, i_init: Optional[int] = None,
                      **kw) -> "StreamTracker":
        from .snapshot import unpack_snapshot

        tracker = cls(config, i_init=i_init, **kw)
        tracker._adopt(*unpack_snapshot(blob, tracker.params))
        return tracker

    @classmethod
    def restore(cls, path, config: RunConfig, i_init: Optional[int] = None, **kw) -> "StreamTracker":
        from .snapshot import unpack_snapshot

        with open(path, "rb") as fh:
            blob = fh.read()
        tracker = cls(config, i_init=i_init, **kw)
        tracker._adopt(*unpack_snapshot(blob, tracker.params, source=str(path)))
        return tracker


# ---------------------------------------------------------------------------
# many independent streams per launch


class BatchTracker:
    """`n_streams` independent StreamTrackers advanced together, one launch
    sequence per frame for all of them.

    Stream s starts from `random_orthonormal(m, k, seeds[s])` (default: every
    stream uses `config.seed`, as separate reference trackers built from the
    same RunConfig would).  `push` takes a [n_streams, m] numpy array or torch
    tensor (host or CUDA; float32, float64 or uint8) and optional output
    buffers; it does not synchronize unless `fit=True`.
    """

    def __init__(self, config: RunConfig, n_streams: int, i_init: Optional[int] = None, *,
                 seeds: Optional[Sequence[int]] = None, precision: str = "fp32",
                 device: int = 0, init_bases: bool = True, latency: bool = False):
        self.config = config
        self.i_init = i_init if i_init is not None else (
            config.i_init if config.i_init is not None else DEFAULT_I_INIT)
        self.params = config.params(self.i_init)
        self.channels = 1 if config.grayscale else 3
        self.n_streams = n_streams
        self.native = NativeTracker(self.params, config.target_width, config.target_height,
                                    self.channels, n_streams, i_init=self.i_init, pipeline=True,
                                    precision=precision, device=device, latency=latency)
        self.m = self.native.m
        self.pixels = self.native.pixels
        seeds = list(seeds) if seeds is not None else [config.seed] * n_streams
        if len(seeds) != n_streams:
            raise ConfigError("need one seed per stream")
        if init_bases:
            cache = {}
            for s, sd in enumerate(seeds):
                if sd not in cache:
                    cache[sd] = random_orthonormal(self.m, self.params.k, sd).data
                self.native.set_core_state(s, cache[sd], np.zeros(self.params.k), None, 0, 0)

    def push(self, frames, background=None, residual=None, mask=None, raw_mask=None,
             fit: bool = False, cuda_stream: int = 0, fit_out=None):
        return self.native.push(frames, background=background, residual=residual, mask=mask,
                                raw_mask=raw_mask, fit=fit, cuda_stream=cuda_stream,
                                fit_out=fit_out)

    def push_many(self, frames, background=None, residual=None, mask=None, raw_mask=None,
                  fit: bool = False, cuda_stream: int = 0, fit_out=None):
        """F consecutive frames per stream ([F, n_streams, m]) in one launch:
        each stream's basis stays on chip across its F frames (frame
        blocking).  Same results as F calls of `push`."""
        return self.native.push_many(frames, background=background, residual=residual, mask=mask,
                                     raw_mask=raw_mask, fit=fit, cuda_stream=cuda_stream,
                                     fit_out=fit_out)

    def background_frame(self, out, cuda_stream: int = 0) -> None:
        self.native.background(out, cuda_stream=cuda_stream)

    def synchronize(self) -> None:
        self.native.synchronize()

    def join(self, cuda_stream: int = 0) -> None:
        """Order `cuda_stream` after every push so far (host-I/O pushes run on
        the handle's own streams, pipelined)."""
        self.native.join(cuda_stream)
