"""Pixel-sharded tracking of one large stream across ranks.

A stream too large for one GPU (BASELINE config C4: 3840x2160, k=30) is split
by image rows: rank g of the process group owns rows [row0, row1) of every
channel plane, i.e. a row block of the basis U, of the frame, of the running
mean and of the labels.  Every phase of the per-frame step that ends in a
reduction (running statistics, pass 0, each CG iteration's line search and
gradient, the fallbacks, the periodic Gram) leaves its per-rank partial sums
in the handle's exchange buffer; they are summed over ranks with one
all-reduce (NCCL over NVLink on GPUs), after which every rank runs the same
scalar logic, so the row blocks stay one basis.  The 3x3 median takes the
label row above and below each block from the neighbouring ranks.  No other
data crosses ranks.

Two ways to run the exchange (`exchange=`):
  "program"  the host drives it: after each phase kernel it all-reduces the
             exchange buffer (NCCL on the kernels' stream, gloo through the
             host) and applies the phase's logic (prost_xnext / xapply) —
             every phase that *can* run exchanges, 7 per frame at C4;
  "peer"     the kernels do it (prost_xpeer_open): the last CTA of each phase
             kernel stores the stream's sums into every rank's exchange region
             over NVLink and sums all ranks' vectors itself, so a frame is one
             prost_push, only the phases that run exchange (3 per steady-state
             frame at C4), and the median's halo rows arrive by peer stores.
             Needs CUDA IPC between the ranks' devices (one node).

The reference has no multi-device path; this class is the same
`StreamTracker.push` seam (jobs.py:186-229) for one stream whose frame and
outputs are each rank's row block.
"""

from __future__ import annotations

import ctypes
from typing import Optional

import numpy as np

from .errors import ConfigError, DimensionError
from .params import DEFAULT_I_INIT, RunConfig
from .tracker import NativeTracker, random_orthonormal

__all__ = ["ShardedTracker", "row_block"]


def row_block(height: int, rank: int, world: int):
    """Rows [row0, row1) of rank `rank`: contiguous, sizes differing by at most one."""
    if not 0 <= rank < world:
        raise ConfigError(f"rank {rank} outside world size {world}")
    if height < world:
        raise DimensionError(f"{height} rows cannot be split over {world} ranks")
    return rank * height // world, (rank + 1) * height // world


class _CudaArray:
    """__cuda_array_interface__ view of a device buffer owned by the library."""

    def __init__(self, ptr: int, count: int, typestr: str, shape=None):
        self.__cuda_array_interface__ = {
            "shape": tuple(shape) if shape is not None else (count,),
            "typestr": typestr, "data": (ptr, False), "version": 3, "strides": None,
        }


class ShardedTracker:
    """One stream, rows sharded over the ranks of `group` (torch.distributed).

    `push(block)` takes this rank's row block of the frame — channel-planar,
    `channels * (row1 - row0) * width` values, device or host — and fills this
    rank's block of the background / mask outputs.  With `world == 1` it is
    the unsharded tracker.
    """

    # Test hook: issue the collectives even at world size 1 (an NCCL group of
    # one rank on one GPU runs the same all-reduce / all-gather calls, stream
    # ordering included, as a multi-GPU group — the only NCCL shape one GPU has)
    collectives_at_world1 = False

    def __init__(self, config: RunConfig, group=None, i_init: Optional[int] = None, *,
                 precision: str = "fp32", device: int = 0, seed: Optional[int] = None,
                 basis: Optional[np.ndarray] = None, exchange: str = "program"):
        import torch
        import torch.distributed as dist

        self.torch = torch
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.backend = dist.get_backend(group) if dist.is_initialized() else None
        self.config = config
        self.i_init = i_init if i_init is not None else (
            config.i_init if config.i_init is not None else DEFAULT_I_INIT)
        self.params = config.params(self.i_init)
        W, H = config.target_width, config.target_height
        C = 1 if config.grayscale else 3
        self.width, self.height, self.channels = W, H, C
        self.row0, self.row1 = row_block(H, self.rank, self.world)
        self.rows = self.row1 - self.row0
        self.device = device
        self.native = NativeTracker(self.params, W, self.rows, C, 1, i_init=self.i_init,
                                    pipeline=True, precision=precision, device=device)
        self.m_global = C * H * W
        self.native.set_exchange(self.m_global)
        # the global bootstrap basis (manifold.py:100-113), restricted to this block
        if basis is None:
            basis = random_orthonormal(self.m_global, self.params.k,
                                       config.seed if seed is None else seed).data
        self.native.set_core_state(0, self.local_rows(basis), np.zeros(self.params.k), None, 0, 0)
        ptr, cnt = self.native.exchange_buffer()
        self.xred = torch.as_tensor(_CudaArray(ptr, cnt, "<f8"), device=f"cuda:{device}")
        self.edges = torch.zeros((2, W), dtype=torch.uint8, device=f"cuda:{device}")
        self.gathered = torch.zeros((self.world, 2, W), dtype=torch.uint8, device=f"cuda:{device}")
        self.exchanges = 0  # cross-rank all-reduces issued (the exchange program)
        self.frames = 0
        if exchange not in ("program", "peer"):
            raise ConfigError(f"exchange must be 'program' or 'peer', got {exchange!r}")
        self.exchange = exchange
        if exchange == "peer":
            handle = self.native.xpeer_handle(self.world)
            handles = [handle]
            if self.world > 1:
                handles = [None] * self.world
                dist.all_gather_object(handles, handle, group=group)
            self.native.xpeer_open(self.rank, self.world, handles)

    # -- layout ---------------------------------------------------------------
    def local_rows(self, full):
        """This rank's rows of a channel-planar per-coordinate array (numpy or
        torch; leading dimension C*H*W, any trailing dimensions)."""
        P, W = self.height * self.width, self.width
        parts = [full[c * P + self.row0 * W: c * P + self.row1 * W] for c in range(self.channels)]
        if isinstance(full, np.ndarray):
            return np.ascontiguousarray(np.concatenate(parts, axis=0))
        return self.torch.cat(parts, dim=0).contiguous()

    def local_pixels(self, full):
        """This rank's rows of a per-pixel array of length H*W."""
        W = self.width
        return full[self.row0 * W: self.row1 * W]

    # -- collectives ------------------------------------------------------------
    def _on(self, cuda_stream: int):
        """Run the collectives on the CUDA stream the phase kernels use, so the
        all-reduce is ordered after the kernels that fill the exchange buffer
        and before the one that consumes it."""
        torch = self.torch
        if cuda_stream == 0:
            return torch.cuda.stream(torch.cuda.default_stream(self.device))
        return torch.cuda.stream(torch.cuda.ExternalStream(cuda_stream, device=self.device))

    def _allreduce(self, t):
        if self.world == 1 and not self.collectives_at_world1:
            return
        if self.backend == "nccl":
            self.dist.all_reduce(t, group=self.group)
        else:  # gloo: host round trip
            h = t.cpu()
            self.dist.all_reduce(h, group=self.group)
            t.copy_(h)

    def _allgather_edges(self):
        if self.world == 1 and not self.collectives_at_world1:
            return
        if self.backend == "nccl":
            self.dist.all_gather_into_tensor(self.gathered, self.edges, group=self.group)
        else:
            parts = [self.torch.zeros_like(self.edges, device="cpu") for _ in range(self.world)]
            self.dist.all_gather(parts, self.edges.cpu(), group=self.group)
            self.gathered.copy_(self.torch.stack(parts))

    # -- the frame step -----------------------------------------------------------
    def push(self, block, background=None, mask=None, raw_mask=None, residual=None,
             fit: bool = False, cuda_stream: int = 0):
        """One frame: every rank calls push with its row block at the same time."""
        nt = self.native
        if self.exchange == "peer":
            self.frames += 1
            return nt.push(block, background=background, residual=residual, mask=mask,
                           raw_mask=raw_mask, fit=fit, cuda_stream=cuda_stream)
        nt.xbegin(block, background=background, residual=residual, mask=mask, raw_mask=raw_mask,
                  fit=fit, cuda_stream=cuda_stream)
        self.frames += 1
        while nt.xnext(cuda_stream):
            with self._on(cuda_stream):
                self._allreduce(self.xred)
            self.exchanges += 1
            nt.xapply(cuda_stream)
        halo_top = halo_bot = None
        if mask is not None and (self.world > 1 or self.collectives_at_world1):
            nt.xedges(self.edges[0].data_ptr(), self.edges[1].data_ptr(), cuda_stream)
            with self._on(cuda_stream):
                self._allgather_edges()
            if self.rank > 0:
                halo_top = self.gathered[self.rank - 1, 1].data_ptr()
            if self.rank < self.world - 1:
                halo_bot = self.gathered[self.rank + 1, 0].data_ptr()
        return nt.xfinish(halo_top, halo_bot, cuda_stream)

    def peer_exchanges(self) -> int:
        """In-kernel exchanges so far (peer mode; synchronizes the device)."""
        from . import _native as nat
        return self.native.query(nat.Q_EXCHANGES)

    def get_basis_block(self) -> np.ndarray:
        return self.native.get_core_state(0)[0]
