"""ctypes binding of the C-ABI in include/prost_b200.h.

The shared library is built in-tree (`paper_1302_2073_b200/_lib/
libprost_b200.so`, see `build.py`).  There is no fallback: if the library is
missing, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .errors import ConfigError, DeviceError, DimensionError, NonFiniteError, SequenceError

LIB_PATH = Path(os.environ.get("PROST_LIB") or
                Path(__file__).resolve().parent / "_lib" / "libprost_b200.so")

PROST_OK = 0
ERR_CONFIG, ERR_DIMENSION, ERR_NONFINITE, ERR_SEQUENCE, ERR_CUDA = 1, 2, 3, 4, 5
F32, F64, U8 = 0, 1, 2
FLAG_PIPELINE, FLAG_FP64, FLAG_LATENCY = 1, 2, 4
Q_LAUNCHES, Q_WAVE, Q_BYTES_U, Q_CHUNKS, Q_INSTANCE_K = 0, 1, 2, 3, 4
Q_RESIDENT, Q_TEAM, Q_TEAMS, Q_GROUPS, Q_QPC = 5, 6, 7, 8, 9
Q_EXCHANGES, Q_CLUSTER, Q_TMA = 10, 11, 12
IPC_HANDLE_BYTES = 64

EXPORTS = (
    "prost_abi_version", "prost_create", "prost_destroy", "prost_set_core_state",
    "prost_get_core_state", "prost_set_preproc", "prost_get_preproc", "prost_push",
    "prost_push_many",
    "prost_background", "prost_synchronize", "prost_last_error", "prost_query",
    "prost_set_wave", "prost_profile", "prost_profile_read", "prost_resident_counters",
    "prost_set_exchange", "prost_xbuffer", "prost_xbegin", "prost_xnext", "prost_xapply",
    "prost_xedges", "prost_xfinish", "prost_xpeer_handle", "prost_xpeer_open", "prost_join", "prost_resample", "prost_upsample_mask",
    "prost_confusion", "prost_unpack_pnm",
)
PHASES = ("stats", "cold", "pass0", "iter", "lsfb", "gradfb", "geo", "qr", "median", "frame")

_ERRORS = {
    ERR_CONFIG: ConfigError,
    ERR_DIMENSION: DimensionError,
    ERR_NONFINITE: NonFiniteError,
    ERR_SEQUENCE: SequenceError,
    ERR_CUDA: DeviceError,
}


class Params(ctypes.Structure):
    _fields_ = [
        ("k", ctypes.c_int32), ("width", ctypes.c_int32), ("height", ctypes.c_int32),
        ("channels", ctypes.c_int32), ("cg_max_iters", ctypes.c_int32),
        ("max_backtracks", ctypes.c_int32), ("i_init", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("p", ctypes.c_double), ("mu", ctypes.c_double), ("delta", ctypes.c_double),
        ("omega", ctypes.c_double), ("t_init", ctypes.c_double), ("t_min", ctypes.c_double),
        ("tau", ctypes.c_double), ("grad_tol", ctypes.c_double),
        ("initial_step", ctypes.c_double), ("shrink", ctypes.c_double),
        ("sufficient_decrease", ctypes.c_double),
    ]


class FitInfo(ctypes.Structure):
    _fields_ = [
        ("fit_cost", ctypes.c_double), ("step", ctypes.c_double),
        ("frame_index", ctypes.c_int64), ("iterations", ctypes.c_int32),
        ("cost_evals", ctypes.c_int32), ("grad_evals", ctypes.c_int32),
        ("status", ctypes.c_int32),
    ]


class Outputs(ctypes.Structure):
    _fields_ = [
        ("background", ctypes.c_void_p), ("residual", ctypes.c_void_p),
        ("mask", ctypes.c_void_p), ("raw_mask", ctypes.c_void_p),
        ("fit", ctypes.POINTER(FitInfo)), ("dtype", ctypes.c_int32),
        ("on_device", ctypes.c_int32), ("fit_residual", ctypes.c_void_p),
        ("fit_async", ctypes.c_int32),
    ]


_lib = None


def lib() -> ctypes.CDLL:
    """Load the native library (raises ImportError when it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
        )
    L = ctypes.CDLL(os.fspath(LIB_PATH))
    vp, i32, i64, u32 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32
    dp = ctypes.POINTER(ctypes.c_double)
    L.prost_abi_version.restype = ctypes.c_int
    L.prost_create.argtypes = [ctypes.POINTER(Params), i32, u32, i32, ctypes.POINTER(vp)]
    L.prost_destroy.argtypes = [vp]
    L.prost_destroy.restype = None
    L.prost_set_core_state.argtypes = [vp, i32, dp, dp, dp, i64, i64]
    L.prost_get_core_state.argtypes = [vp, i32, dp, dp, dp, ctypes.POINTER(i64), ctypes.POINTER(i64)]
    L.prost_set_preproc.argtypes = [vp, i32, dp, dp]
    L.prost_get_preproc.argtypes = [vp, i32, dp, dp]
    L.prost_push.argtypes = [vp, vp, i32, i32, ctypes.POINTER(Outputs), vp]
    L.prost_push_many.argtypes = [vp, vp, i32, i32, i32, ctypes.POINTER(Outputs), vp]
    L.prost_background.argtypes = [vp, vp, i32, i32, vp]
    L.prost_synchronize.argtypes = [vp]
    L.prost_last_error.argtypes = [vp, ctypes.c_char_p, i32]
    L.prost_query.argtypes = [vp, i32, ctypes.POINTER(i64)]
    L.prost_set_wave.argtypes = [vp, i32]
    L.prost_profile.argtypes = [vp, i32]
    L.prost_profile_read.argtypes = [vp, dp, ctypes.POINTER(i64), i32]
    L.prost_resident_counters.argtypes = [vp, ctypes.POINTER(i64), i32]
    L.prost_set_exchange.argtypes = [vp, i64]
    L.prost_xbuffer.argtypes = [vp, ctypes.POINTER(vp), ctypes.POINTER(i64)]
    L.prost_xbegin.argtypes = [vp, vp, i32, i32, ctypes.POINTER(Outputs), vp]
    L.prost_xnext.argtypes = [vp, ctypes.POINTER(i32), vp]
    L.prost_xapply.argtypes = [vp, vp]
    L.prost_xedges.argtypes = [vp, vp, vp, vp]
    L.prost_xfinish.argtypes = [vp, vp, vp, vp]
    L.prost_xpeer_handle.argtypes = [vp, i32, vp]
    L.prost_xpeer_open.argtypes = [vp, i32, i32, vp]
    L.prost_join.argtypes = [vp, vp]
    L.prost_resample.argtypes = [vp, i32, i32, i32, i32, vp, i32, i32, i32, vp]
    L.prost_upsample_mask.argtypes = [vp, i32, i32, vp, i32, i32, vp]
    L.prost_confusion.argtypes = [vp, i64, vp, i32, i32, vp, vp]
    L.prost_unpack_pnm.argtypes = [vp, i32, i32, vp, i32, vp]
    for name in EXPORTS:
        if name not in ("prost_destroy",):
            getattr(L, name).restype = ctypes.c_int
    if L.prost_abi_version() != 2:
        raise ImportError("libprost_b200.so ABI version mismatch")
    _lib = L
    return L


def last_error(handle) -> str:
    buf = ctypes.create_string_buffer(512)
    lib().prost_last_error(handle, buf, 512)
    return buf.value.decode(errors="replace")


def error_class(rc: int):
    return _ERRORS.get(rc, DeviceError)


def check(rc: int, handle=None, what: str = "") -> None:
    if rc == PROST_OK:
        return
    msg = last_error(handle) if handle else ""
    cls = _ERRORS.get(rc, DeviceError)
    raise cls(msg or f"{what} failed with status {rc}")


def dptr(arr) -> ctypes.POINTER(ctypes.c_double):
    """ctypes double* of a C-contiguous float64 numpy array (or NULL)."""
    if arr is None:
        return None
    return arr.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
