"""B200-native pROST per-frame tracker (arXiv 1302.2073).

Public surface mirrors the reference package's hot-path API
(`/root/reference/pkg/src/prost/__init__.py:27-30`): `RunConfig`,
`StreamTracker`, `process_frame`, `bootstrap`, `ProstParams`, `LpConfig`,
`CgOptions`, `TrackerState`, `FrameBuffer`, `SegmentationMask` and the error
classes.  The per-frame arithmetic runs in hand-written sm_100a CUDA kernels
behind the C-ABI of `include/prost_b200.h`; there is no CPU fallback.
"""

from .errors import (
    CodecError,
    ConfigError,
    DeviceError,
    DimensionError,
    NonFiniteError,
    ProstError,
    SequenceError,
    SnapshotError,
)
from .frames import FrameBuffer, FrameRecord, SegmentationMask
from .params import (
    DEFAULT_I_INIT,
    CgOptions,
    LpConfig,
    ProstParams,
    RunConfig,
    smoothing_from_threshold,
    step_size,
    tau_from_init,
)
from .tracker import (
    BatchTracker,
    FitInfoBuffer,
    FitResult,
    NativeTracker,
    StreamTracker,
    SubspaceBasis,
    TrackerState,
    bootstrap,
    process_frame,
    random_orthonormal,
)

__version__ = "0.1.0"

__all__ = [
    "CodecError", "ConfigError", "DeviceError", "DimensionError", "NonFiniteError",
    "ProstError", "SequenceError", "SnapshotError", "FrameBuffer", "FrameRecord",
    "SegmentationMask", "DEFAULT_I_INIT", "CgOptions", "LpConfig", "ProstParams", "RunConfig",
    "smoothing_from_threshold", "step_size", "tau_from_init", "BatchTracker", "FitInfoBuffer", "FitResult",
    "NativeTracker", "StreamTracker", "SubspaceBasis", "TrackerState", "bootstrap",
    "process_frame", "random_orthonormal", "__version__",
]
