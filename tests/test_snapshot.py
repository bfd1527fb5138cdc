"""PROSTSNAP1 snapshots (reference tracker.py:159-285 and
jobs.py:241-277), pinned to bytes written by the reference itself
(tests/golden/snapshot_gray.npz, made by tests/golden/make_golden.py).

CPU: the format — our params hash, unpack and pack reproduce the reference's
bytes exactly; foreign / truncated / mismatched blobs raise SnapshotError.
GPU: StreamTracker.restore_bytes of the reference's snapshot continues the
stream as the reference does, and snapshot_bytes of the restored fp64 tracker
is byte-identical to the reference's.
"""

from pathlib import Path

import numpy as np
import pytest

import paper_1302_2073_b200 as pkg
from paper_1302_2073_b200.snapshot import pack_snapshot, params_hash, unpack_snapshot
from paper_1302_2073_b200.tracker import PreprocSnapshot, SubspaceBasis, TrackerState

GOLD = Path(__file__).resolve().parent / "golden" / "snapshot_gray.npz"


def _load():
    z = np.load(GOLD)
    k, p, mu, iters, i_init, seed, n_before = z["cfg"]
    cfg = pkg.RunConfig(subspace_dim=int(k), p=float(p), mu=float(mu), cg_max_iters=int(iters),
                        target_width=32, target_height=24, grayscale=True, i_init=int(i_init),
                        seed=int(seed))
    return z, cfg, int(i_init), int(n_before)


def test_format_round_trip_matches_reference_bytes():
    z, cfg, i_init, _ = _load()
    blob = z["blob"].tobytes()
    params = cfg.params(i_init)
    U, y, w, fi, pre = unpack_snapshot(blob, params)
    assert U.shape == (32 * 24, 4) and pre is not None and fi == 8
    state = TrackerState(SubspaceBasis(U, check=False), y, w, fi, pre)
    assert pack_snapshot(state, params) == blob
    assert int.from_bytes(blob[10 + 16:10 + 24], "little") == params_hash(params)


def test_format_rejections():
    z, cfg, i_init, _ = _load()
    blob = z["blob"].tobytes()
    params = cfg.params(i_init)
    with pytest.raises(pkg.SnapshotError):
        unpack_snapshot(b"NOTASNAP" + blob[10:], params)
    with pytest.raises(pkg.SnapshotError):
        unpack_snapshot(blob[:200], params)
    other = pkg.RunConfig(subspace_dim=4, p=0.5, mu=2e-4, cg_max_iters=2, target_width=32,
                          target_height=24, grayscale=True, i_init=i_init, seed=4).params(i_init)
    with pytest.raises(pkg.SnapshotError):
        unpack_snapshot(blob, other)


@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_restore_continues_like_reference(precision):
    z, cfg, i_init, n_before = _load()
    blob = z["blob"].tobytes()
    tr = pkg.StreamTracker.restore_bytes(blob, cfg, precision=precision)
    assert tr.frame_index == n_before and tr.started
    if precision == "fp64":
        assert tr.snapshot_bytes() == blob
    frames = z["frames"][n_before:]
    worst_mask, worst_bg = 0.0, 0.0
    for i, v in enumerate(frames):
        rec = tr.push(pkg.FrameBuffer(32, 24, 1, v))
        bg = tr.background_frame().data
        worst_mask = max(worst_mask, float(np.mean(rec.mask.labels != z["mask"][i])))
        worst_bg = max(worst_bg, float(np.linalg.norm(bg - z["background"][i]) /
                                       np.linalg.norm(z["background"][i])))
    if precision == "fp64":
        assert worst_mask == 0.0 and worst_bg <= 1e-9
    else:
        assert worst_mask <= 1e-3 and worst_bg <= 1e-4


@pytest.mark.gpu
def test_fp32_export_is_accepted_by_reference_types():
    """A snapshot of an fp32 tracker after 220 frames: its basis passes the
    reference's orthonormality check (drift <= 1e-8, manifold.py:66-70; fp32
    drift alone is ~1e-7), and the oracle continued from the blob tracks the
    GPU tracker that wrote it (SURVEY.md §8(b) export rule)."""
    from oracle import prost_oracle as orc
    from paper_1302_2073_b200.synth import SceneSpec, SceneStream

    W, H = 64, 48
    cfg = pkg.RunConfig(subspace_dim=8, p=0.5, mu=1e-4, cg_max_iters=2, target_width=W,
                        target_height=H, grayscale=True, i_init=50, seed=3)
    frames = SceneStream(SceneSpec(width=W, height=H, rank=4, seed=7)).next_frames(226)
    tr = pkg.StreamTracker(cfg, precision="fp32")
    for v in frames[:220]:
        tr.push(pkg.FrameBuffer(W, H, 1, v))
    raw_drift = np.linalg.norm(tr.state.basis.data.T @ tr.state.basis.data - np.eye(8))
    blob = tr.snapshot_bytes()
    params = cfg.params(50)
    U, y, w, fi, pre = unpack_snapshot(blob, params)
    drift = np.linalg.norm(U.T @ U - np.eye(8))
    print(f"fp32 drift {raw_drift:.2e} -> exported {drift:.2e}")
    assert drift <= 1e-8
    SubspaceBasis(U)  # the reference's check (raises DimensionError above 1e-8)
    assert fi == 220 and pre is not None and pre.frozen
    # the reconstruction is unchanged by the re-wrap
    bg_gpu = tr.background_frame().data
    o = orc.PipelineOracle(W, H, 1, orc.OracleParams(
        k=8, p=0.5, mu=1e-4, delta=params.delta, omega=params.omega, t_init=params.t_init,
        t_min=params.t_min, tau=params.tau, max_iters=2), i_init=50, seed=3)
    o.norm = orc.Normalizer(pre.mean.copy(), pre.frames_seen, pre.frozen, pre.std, pre.value_sum,
                            pre.value_sumsq, pre.value_count)
    o.state = orc.CoreState(U, y, w, fi, 0)
    assert np.linalg.norm(o.background() - bg_gpu) <= 1e-6 * np.linalg.norm(bg_gpu)
    for v in frames[220:]:
        a = tr.push(pkg.FrameBuffer(W, H, 1, v))
        b = o.push(v)
        assert np.mean(a.mask.labels != b.mask) <= 1e-3
    bg = tr.background_frame().data
    assert np.linalg.norm(bg - o.background()) <= 1e-4 * np.linalg.norm(o.background())
    assert orc.subspace_sine(tr.state.basis.data, o.state.U) <= 1e-3
