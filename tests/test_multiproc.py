"""Multi-process host logic of the stream-sharded benchmark on CPU (gloo,
world size 2): disjoint stream shards that cover the global stream set, the
max-over-ranks timing reduction, and per-rank synthetic inputs that depend only
on the global stream index (so a stream's frames are identical whatever the
rank count)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, per_rank, out):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench

    ids = bench.shard_streams(rank, per_rank)
    frames = bench.gen_frames("C0", ids, 2)
    fake_ms = 10.0 + rank  # each rank's device time
    mx = bench.reduce_max(fake_ms, world, "cpu")
    out[rank] = (ids, float(frames[1].sum()), mx)
    dist.barrier()
    dist.destroy_process_group()


def test_stream_sharding_gloo_world2():
    import torch.multiprocessing as mp

    world, per_rank = 2, 3
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, port, per_rank, out), nprocs=world, join=True)
        res = dict(out)
    ids = sorted(i for r in range(world) for i in res[r][0])
    assert ids == list(range(world * per_rank))
    assert set(res[0][0]).isdisjoint(res[1][0])
    assert all(res[r][2] == 11.0 for r in range(world))  # max over ranks
    # the same global stream gets the same frames in a single-rank run
    import bench

    single = bench.gen_frames("C0", bench.shard_streams(0, world * per_rank), 2)
    np.testing.assert_allclose(single[1][per_rank:].sum(), res[1][1], rtol=1e-6)
