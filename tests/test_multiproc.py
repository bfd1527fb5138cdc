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


# ---------------------------------------------------------------------------
# Pixel sharding (C4) host logic on CPU: per-rank partial sums
# over row blocks, summed with an all-reduce, equal the full-frame reductions
# of the oracle; and the halo-row median (the rule k_median4 applies with
# prost_xedges / prost_xfinish) over row blocks equals the full-frame median.


def _pixel_worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    from oracle import prost_oracle as orc
    from paper_1302_2073_b200.shard import row_block

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    W, H, k = 24, 17, 5
    rng = np.random.default_rng(7)
    U = np.linalg.qr(rng.standard_normal((W * H, k)))[0]
    x = rng.standard_normal(W * H)
    y = rng.standard_normal(k)
    w = np.where(rng.random(W * H) < 0.2, 5e-5, 1.0)
    labels = (rng.random((H, W)) < 0.4).astype(np.uint8)
    r0, r1 = row_block(H, rank, world)
    sl = slice(r0 * W, r1 * W)
    # pass-0 partials of this block: cost, U^T g, ||g||^2 (fit.py:96-104)
    res = x[sl] - U[sl] @ y
    c, g = orc.lp_cost_grad(res, 0.5, 1e-4, w[sl])
    part = torch.tensor(np.concatenate([[c], U[sl].T @ g, [g @ g]]))
    dist.all_reduce(part)
    # halo exchange of the block's first and last label rows
    blk = labels[r0:r1]
    edges = torch.tensor(np.stack([blk[0], blk[-1]]))
    gathered = [torch.zeros_like(edges) for _ in range(world)]
    dist.all_gather(gathered, edges)
    above = gathered[rank - 1][1].numpy() if rank > 0 else blk[0]
    below = gathered[rank + 1][0].numpy() if rank < world - 1 else blk[-1]
    ext = np.vstack([above[None], blk, below[None]]).astype(np.int32)
    padx = np.pad(ext, ((0, 0), (1, 1)), mode="edge")
    votes = sum(padx[dy:dy + blk.shape[0], dx:dx + W] for dy in range(3) for dx in range(3))
    out[rank] = (part.numpy(), (votes >= 5).astype(np.uint8), r0, r1)
    if rank == 0:
        res_full = x - U @ y
        cf, gf = orc.lp_cost_grad(res_full, 0.5, 1e-4, w)
        out["full"] = (np.concatenate([[cf], U.T @ gf, [gf @ gf]]),
                       orc.majority3x3(labels.reshape(-1), W, H).reshape(H, W))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_pixel_sharding_gloo(world):
    import torch.multiprocessing as mp

    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_pixel_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    full_part, full_median = res["full"]
    for r in range(world):
        np.testing.assert_allclose(res[r][0], full_part, rtol=1e-12, atol=1e-12)
    med = np.vstack([res[r][1] for r in range(world)])
    np.testing.assert_array_equal(med, full_median)
