"""Pixel-sharded single stream: the exchange-mode phase
program against the unsharded tracker.

CPU: the row decomposition.  GPU: world size 1 (no collective) is bit-identical
to the unsharded streamed path; two ranks (gloo, host-side all-reduce and edge
exchange, both on cuda:0 — the ranks' kernels never wait on one another) agree
with the unsharded run within fp32 summation-order tolerances.
"""

import os
import socket

import numpy as np
import pytest

import paper_1302_2073_b200 as pkg
from paper_1302_2073_b200.shard import row_block


def test_row_block_partition():
    for H, world in ((2160, 8), (240, 2), (7, 3), (120, 1)):
        blocks = [row_block(H, r, world) for r in range(world)]
        assert blocks[0][0] == 0 and blocks[-1][1] == H
        for (a0, a1), (b0, b1) in zip(blocks, blocks[1:]):
            assert a1 == b0
        sizes = [b - a for a, b in blocks]
        assert max(sizes) - min(sizes) <= 1
    with pytest.raises(pkg.DimensionError):
        row_block(3, 0, 4)


W, H, K, F = 64, 48, 8, 10


def _frames(seed=0):
    from paper_1302_2073_b200.synth import SceneSpec, SceneStream

    return SceneStream(SceneSpec(width=W, height=H, channels=1, rank=4, noise=0.02,
                                 seed=seed)).next_frames(F).astype(np.float32)


def _cfg():
    return pkg.RunConfig(subspace_dim=K, p=0.5, mu=1e-4, cg_max_iters=2, target_width=W,
                         target_height=H, grayscale=True, i_init=4, seed=3)


def _unsharded(frames):
    import torch

    os.environ["PROST_KERNEL"] = "streamed"
    try:
        bt = pkg.BatchTracker(_cfg(), 1, seeds=[3])
    finally:
        del os.environ["PROST_KERNEL"]
    masks, bgs = [], []
    mask = torch.empty((1, W * H), dtype=torch.uint8, device="cuda")
    bg = torch.empty((1, W * H), dtype=torch.float32, device="cuda")
    for f in frames:
        bt.push(torch.from_numpy(f).cuda()[None], background=bg, mask=mask)
        masks.append(mask.cpu().numpy()[0].copy())
        bgs.append(bg.cpu().numpy()[0].copy())
    return np.array(masks), np.array(bgs), bt.native.get_core_state(0)[0]


def _sharded_run(frames, group=None, exchange="program"):
    import torch
    from paper_1302_2073_b200.shard import ShardedTracker

    st = ShardedTracker(_cfg(), group=group, exchange=exchange)
    n = st.rows * W
    mask = torch.empty(n, dtype=torch.uint8, device="cuda")
    bg = torch.empty(n, dtype=torch.float32, device="cuda")
    masks, bgs = [], []
    for f in frames:
        st.push(torch.from_numpy(st.local_rows(f)).cuda(), background=bg, mask=mask)
        masks.append(mask.cpu().numpy().copy())
        bgs.append(bg.cpu().numpy().copy())
    return np.array(masks), np.array(bgs), st.get_basis_block(), st


@pytest.mark.gpu
def test_world1_matches_unsharded_bitwise():
    frames = _frames()
    m0, b0, U0 = _unsharded(frames)
    m1, b1, U1, st = _sharded_run(frames)
    assert st.exchanges > 0
    np.testing.assert_array_equal(m1, m0)
    np.testing.assert_array_equal(b1, b0)
    np.testing.assert_array_equal(U1, U0)


@pytest.mark.gpu
def test_peer_exchange_world1_matches_unsharded_bitwise():
    """In-kernel exchange through the peer-memory region (world size 1: the
    region is this rank's own): the same results bit for bit, and only the
    phases that ran exchanged."""
    frames = _frames()
    m0, b0, U0 = _unsharded(frames)
    m1, b1, U1, st = _sharded_run(frames, exchange="peer")
    np.testing.assert_array_equal(m1, m0)
    np.testing.assert_array_equal(b1, b0)
    np.testing.assert_array_equal(U1, U0)
    _, _, _, sp = _sharded_run(frames)
    ex = st.peer_exchanges()
    assert F <= ex < sp.exchanges
    assert st.native.query(0) < sp.native.query(0)  # fewer launches: no k_xlogic


def _worker(rank, world, port, frames, out):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    m, b, U, st = _sharded_run(frames)
    np.savez(out.format(rank), m=m, b=b, U=U, row0=st.row0, row1=st.row1)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_two_ranks_match_unsharded(tmp_path):
    import torch.multiprocessing as mp

    frames = _frames()
    m0, b0, U0 = _unsharded(frames)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = str(tmp_path / "rank{}.npz")
    mp.spawn(_worker, args=(2, port, frames, out), nprocs=2, join=True)
    parts = [np.load(out.format(r)) for r in range(2)]
    m = np.concatenate([p["m"] for p in parts], axis=1)
    b = np.concatenate([p["b"] for p in parts], axis=1)
    U = np.concatenate([p["U"] for p in parts], axis=0)
    assert int(parts[0]["row1"]) == int(parts[1]["row0"])
    # same algorithm, partial sums added in another order: fp32-level agreement
    assert np.mean(m != m0) <= 1e-3
    assert np.linalg.norm(b - b0) <= 1e-4 * np.linalg.norm(b0)
    q0, _ = np.linalg.qr(U0)
    q1, _ = np.linalg.qr(U)
    s = np.linalg.svd(q0.T @ q1, compute_uv=False)
    assert np.sqrt(max(0.0, 1.0 - float(s.min()) ** 2)) <= 1e-4


@pytest.mark.gpu
@pytest.mark.parametrize("exchange", ["program", "peer"])
def test_non_finite_frame_after_the_window(exchange):
    """A non-finite frame after the statistics window is rejected and the next
    frame runs normally: the host-driven program no longer exchanges for the
    statistics phase once every stream is frozen, but still resets the frame
    status (k_stats' no-op branch) — bit for bit the unsharded tracker."""
    frames = list(_frames())
    bad = frames[7].copy()
    bad[5] = np.nan
    seq = frames[:7] + [bad] + frames[7:]
    m0, b0, U0 = _unsharded(seq)
    m1, b1, U1, st = _sharded_run(seq, exchange=exchange)
    keep = [i for i in range(len(seq)) if i != 7]
    np.testing.assert_array_equal(m1[keep], m0[keep])
    np.testing.assert_array_equal(b1[keep], b0[keep])
    np.testing.assert_array_equal(U1, U0)


def _nccl_worker(rank, port, frames, out):
    """One-rank NCCL group: the exchange program's all-reduces and the halo
    all-gather go through NCCL on a side CUDA stream (shard.py _on)."""
    import torch
    import torch.distributed as dist
    from paper_1302_2073_b200.shard import ShardedTracker

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    ShardedTracker.collectives_at_world1 = True
    st = ShardedTracker(_cfg())
    assert st.backend == "nccl"
    side = torch.cuda.Stream()
    n = st.rows * W
    mask = torch.empty(n, dtype=torch.uint8, device="cuda")
    bg = torch.empty(n, dtype=torch.float32, device="cuda")
    masks, bgs = [], []
    for f in frames:
        blk = torch.from_numpy(st.local_rows(f)).cuda()
        torch.cuda.synchronize()
        st.push(blk, background=bg, mask=mask, cuda_stream=side.cuda_stream)
        side.synchronize()
        masks.append(mask.cpu().numpy().copy())
        bgs.append(bg.cpu().numpy().copy())
    torch.cuda.synchronize()
    np.savez(out, m=np.array(masks), b=np.array(bgs), U=st.get_basis_block(), ex=st.exchanges)
    dist.destroy_process_group()


@pytest.mark.gpu
def test_nccl_exchange_program_world1_matches_unsharded_bitwise(tmp_path):
    """The NCCL branch of the exchange program (all_reduce of the exchange
    buffer, all_gather of the label edges) on a non-default CUDA stream: a
    one-rank sum is the identity, so the run is bit-identical to the unsharded
    tracker, and every phase that can run was exchanged through NCCL."""
    import torch.multiprocessing as mp

    frames = _frames()
    m0, b0, U0 = _unsharded(frames)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = str(tmp_path / "nccl.npz")
    mp.spawn(_nccl_worker, args=(port, frames, out), nprocs=1, join=True)
    r = np.load(out)
    assert int(r["ex"]) >= 3 * F
    np.testing.assert_array_equal(r["m"], m0)
    np.testing.assert_array_equal(r["b"], b0)
    np.testing.assert_array_equal(r["U"], U0)
