"""GPU parity: the CUDA path (through the C-ABI) against the reference's golden
vectors and the CPU oracle.

Two instantiations are checked:
  * fp64 (parity instantiation): one-step agreement with the reference to
    1e-10 and identical decisions (CG iterations / Armijo evaluations / labels);
  * fp32 (the product path): north_star tolerances — principal-angle sine of U
    <= 1e-3, background relative L2 <= 1e-4, mask disagreement <= 0.1% — plus a
    teacher-forced one-step bound of 1e-5 on the angle.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import prost_oracle as orc

pytestmark = pytest.mark.gpu

pkg = pytest.importorskip("paper_1302_2073_b200")


def load(name):
    return np.load(GOLDEN / f"{name}.npz")


def traj_params(z):
    k, p, mu, delta, omega, t_init, t_min, tau, iters, seed = z["prm"]
    params = pkg.ProstParams(k=int(k), cfg=pkg.LpConfig(p=p, mu=mu), delta=delta, omega=omega,
                             t_init=t_init, t_min=t_min, tau=tau,
                             cg=pkg.CgOptions(max_iters=int(iters)))
    return params, int(seed)


def sine(A, B):
    return orc.subspace_sine(A, B)


# ---------------------------------------------------------------------------
# process_frame (tracker.py:121-156), teacher forced along the reference
# trajectory: every frame starts from the reference's own state.


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_process_frame_teacher_forced(precision):
    z = load("step_trajectory")
    params, seed = traj_params(z)
    frames = z["frames"]
    U_prev = z["U0"]
    y_prev = np.zeros(params.k)
    w_prev = np.ones(frames.shape[1])
    same_counts = 0
    for i, x in enumerate(frames):
        st = pkg.TrackerState(pkg.SubspaceBasis(U_prev), y_prev, w_prev, frame_index=i)
        new, r, fit = pkg.process_frame(st, x, params, precision=precision)
        assert new.frame_index == i + 1
        oprm = orc.OracleParams(k=params.k, p=params.cfg.p, mu=params.cfg.mu, delta=params.delta,
                                omega=params.omega, t_init=params.t_init, t_min=params.t_min,
                                tau=params.tau, max_iters=params.cg.max_iters)
        ofit = orc.fit(U_prev, x, None if i == 0 else y_prev, oprm, w_prev)
        np.testing.assert_allclose(fit.residual, ofit.residual, rtol=0,
                                   atol=1e-9 if precision == "fp64" else 1e-4)
        same = [fit.iterations, fit.cost_evals, fit.grad_evals] == list(z["counts"][i])
        same_counts += same
        if precision == "fp64":
            assert same, (i, fit, z["counts"][i])
            np.testing.assert_allclose(new.basis.data, z["U"][i], rtol=0, atol=1e-10)
            np.testing.assert_allclose(new.y, z["y"][i], rtol=1e-10, atol=1e-10)
            np.testing.assert_allclose(r, z["residual"][i], rtol=0, atol=1e-9)
            np.testing.assert_array_equal(new.weights, z["w"][i])
            assert fit.cost == pytest.approx(z["cost"][i], rel=1e-12)
        else:
            assert sine(new.basis.data, z["U"][i]) <= 1e-5
            np.testing.assert_allclose(r, z["residual"][i], rtol=0, atol=1e-4)
            assert np.mean(new.weights != z["w"][i]) <= 0.01
            assert fit.cost == pytest.approx(z["cost"][i], rel=1e-5)
        U_prev, y_prev, w_prev = z["U"][i], z["y"][i], z["w"][i]
    assert same_counts >= 0.95 * len(frames)


def test_process_frame_free_running_fp64():
    z = load("step_trajectory")
    params, seed = traj_params(z)
    st = pkg.bootstrap(z["frames"].shape[1], params, seed)
    np.testing.assert_array_equal(st.basis.data, z["U0"])
    for i, x in enumerate(z["frames"]):
        st, r, fit = pkg.process_frame(st, x, params, precision="fp64")
        assert sine(st.basis.data, z["U"][i]) <= 1e-9
        np.testing.assert_array_equal(st.weights, z["w"][i])
        assert fit.cost == pytest.approx(z["cost"][i], rel=1e-9)


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_fit_cases(precision):
    """fit_coordinates golden cases (p = 0.5, 0.25, 2, 1; cold and warm starts),
    observed through process_frame's fitted coordinates and counters."""
    z = load("fit_vectors")
    for case in range(4):
        key = f"c{case}_"
        p, mu, iters = z[key + "prm"]
        U = z[key + "U"]
        m, k = U.shape
        params = pkg.ProstParams(k=k, cfg=pkg.LpConfig(p=p, mu=mu), delta=0.35, omega=5e-5,
                                 cg=pkg.CgOptions(max_iters=int(iters)))
        y0 = z[key + "y0"]
        cold = bool(np.isnan(y0).all())
        st = pkg.TrackerState(pkg.SubspaceBasis(U), np.zeros(k) if cold else y0, z[key + "w"],
                              frame_index=0 if cold else 1)
        _, _, fit = pkg.process_frame(st, z[key + "x"], params, precision=precision)
        tol = 1e-10 if precision == "fp64" else 2e-4
        np.testing.assert_allclose(fit.y, z[key + "y"], rtol=tol, atol=tol)
        # FitResult.residual: x - U y at the fitted coordinates (fit.py:50-63)
        np.testing.assert_allclose(fit.residual, z[key + "residual"], rtol=0,
                                   atol=1e-9 if precision == "fp64" else 2e-4)
        assert fit.cost == pytest.approx(float(z[key + "cost"]), rel=tol)
        if precision == "fp64":
            assert [fit.iterations, fit.cost_evals, fit.grad_evals] == list(z[key + "counts"])


@pytest.mark.parametrize("precision", ["fp64", "fp32", "fp32-resident", "fp32-streamed"])
def test_periodic_reorthonormalization(precision, monkeypatch):
    """The unconditional QR at the 1000th geodesic step (manifold.py:192-196),
    replayed from the reference's state at step 997 (fp32: default TMEM kernel,
    register-resident kernel, streamed kernels)."""
    if precision.startswith("fp32-"):
        monkeypatch.setenv("PROST_KERNEL", precision.split("-")[1])
        precision = "fp32"
    z = load("qr_chain")
    params = pkg.ProstParams(k=3, cfg=pkg.LpConfig(p=0.5, mu=0.06125), delta=0.35, omega=5e-5,
                             t_init=1e-2, t_min=1e-3, tau=1e-3, cg=pkg.CgOptions(max_iters=2))
    # rebuild the reference state at frame 997 with the oracle (pinned bit-exact)
    oprm = orc.OracleParams(k=3, p=0.5, mu=0.06125, delta=0.35, omega=5e-5, t_init=1e-2,
                            t_min=1e-3, tau=1e-3, max_iters=2)
    ost = orc.core_init(48, oprm, 3)
    for x in z["frames"][:998]:
        ost, _, _ = orc.core_step(ost, x, oprm)
    np.testing.assert_array_equal(ost.U, z["U997"])
    st = pkg.TrackerState(pkg.SubspaceBasis(ost.U, steps_since_qr=ost.since_qr), ost.y, ost.w,
                          frame_index=ost.frame_index)
    for i in range(998, 1003):
        st, _, _ = pkg.process_frame(st, z["frames"][i], params, precision=precision)
        np.testing.assert_allclose(st.basis.data, z[f"U{i}"], rtol=0,
                                   atol=1e-10 if precision == "fp64" else 2e-5)
        assert st.basis.steps_since_qr == int(z[f"since{i}"])
    U = st.basis.data
    assert np.linalg.norm(U.T @ U - np.eye(3)) < (1e-12 if precision == "fp64" else 1e-5)


def test_rejects_non_finite_frame_without_mutation():
    z = load("step_trajectory")
    params, seed = traj_params(z)
    st = pkg.bootstrap(z["frames"].shape[1], params, seed)
    st, _, _ = pkg.process_frame(st, z["frames"][0], params)
    bad = z["frames"][1].copy()
    bad[7] = np.nan
    with pytest.raises(pkg.NonFiniteError):
        pkg.process_frame(st, bad, params)
    with pytest.raises(pkg.DimensionError):
        pkg.process_frame(st, bad[:-1], params)
    # the functional seam never mutates its input; the next good frame proceeds
    st2, _, _ = pkg.process_frame(st, z["frames"][1], params, precision="fp64")
    assert st2.frame_index == 2


# ---------------------------------------------------------------------------
# StreamTracker.push (jobs.py:186-239) against the reference's own run


@pytest.mark.parametrize("name", ["push_gray", "push_rgb"])
@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_stream_tracker_golden(name, precision):
    z = load(name)
    k, p, mu, iters, i_init, seed, channels = z["cfg"]
    cfg = pkg.RunConfig(subspace_dim=int(k), p=p, mu=mu, cg_max_iters=int(iters), target_width=32,
                        target_height=24, grayscale=False, i_init=int(i_init), seed=int(seed))
    tr = pkg.StreamTracker(cfg, precision=precision)
    for i, v in enumerate(z["frames"]):
        rec = tr.push(pkg.FrameBuffer(32, 24, int(channels), v))
        assert rec.frame_index == i + 1
        assert rec.step == z["step"][i]
        bg = tr.background_frame().data
        if precision == "fp64":
            np.testing.assert_array_equal(rec.raw_mask.labels, z["raw_mask"][i])
            np.testing.assert_array_equal(rec.mask.labels, z["mask"][i])
            np.testing.assert_allclose(rec.residual, z["residual"][i], rtol=0, atol=1e-9)
            assert rec.fit_cost == pytest.approx(z["fit_cost"][i], rel=1e-10)
            np.testing.assert_allclose(bg, z["background"][i], rtol=0, atol=1e-10)
        else:
            assert np.mean(rec.raw_mask.labels != z["raw_mask"][i]) <= 0.001
            assert np.mean(rec.mask.labels != z["mask"][i]) <= 0.001
            ref_bg = z["background"][i]
            assert np.linalg.norm(bg - ref_bg) <= 1e-4 * np.linalg.norm(ref_bg)
            assert rec.fit_cost == pytest.approx(z["fit_cost"][i], rel=1e-4)
    st = tr.state
    tol = 1e-9 if precision == "fp64" else 1e-3
    assert sine(st.basis.data, z["U"]) <= tol
    np.testing.assert_allclose(tr.stats.mean, z["mean"], rtol=0, atol=1e-12 if precision == "fp64" else 1e-6)
    assert tr.stats.std == pytest.approx(float(z["std"]), rel=1e-12 if precision == "fp64" else 1e-6)


def test_stream_tracker_rejects_bad_input():
    cfg = pkg.RunConfig(subspace_dim=4, target_width=16, target_height=8, grayscale=False, i_init=3)
    tr = pkg.StreamTracker(cfg)
    rng = np.random.default_rng(0)
    tr.push(pkg.FrameBuffer(16, 8, 1, rng.random(128)))
    with pytest.raises(pkg.SequenceError):  # jobs.py:195-198
        tr.push(pkg.FrameBuffer(16, 8, 3, rng.random(384)))
    # an off-resolution frame is resampled to the model resolution (jobs.py:181-184)
    rec = tr.push(pkg.FrameBuffer(8, 8, 1, rng.random(64)))
    assert rec.frame_index == 2 and rec.mask.width == 16 and rec.mask.height == 8
    bad = rng.random(128)
    bad[3] = np.inf
    with pytest.raises(pkg.NonFiniteError):
        tr.push(pkg.FrameBuffer(16, 8, 1, bad))
    assert tr.frame_index == 2
    rec = tr.push(pkg.FrameBuffer(16, 8, 1, rng.random(128)))
    assert rec.frame_index == 3


# ---------------------------------------------------------------------------
# larger configurations: oracle comparison at the C0 shape and batched streams


def c0_stream(n_frames, width=160, height=120, seed=0):
    from paper_1302_2073_b200.synth import SceneSpec, SceneStream

    spec = SceneSpec(width=width, height=height, channels=1, rank=5, noise=0.02, seed=seed)
    return SceneStream(spec).next_frames(n_frames)


def oracle_for(cfg, i_init, width, height, channels=1):
    prm = cfg.params(i_init)
    return orc.PipelineOracle(width, height, channels, orc.OracleParams(
        k=prm.k, p=prm.cfg.p, mu=prm.cfg.mu, delta=prm.delta, omega=prm.omega,
        t_init=prm.t_init, t_min=prm.t_min, tau=prm.tau, max_iters=prm.cg.max_iters),
        i_init=i_init, seed=cfg.seed)


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_c0_shape_against_oracle(precision):
    """C0 shape (160x120, k=15, p=0.5, mu=1e-4, 2 CG iterations), 60 frames
    through the init window: masks, background and basis against the oracle."""
    n_frames, i_init = 60, 20
    frames = c0_stream(n_frames)
    cfg = pkg.RunConfig(subspace_dim=15, p=0.5, mu=1e-4, cg_max_iters=2, target_width=160,
                        target_height=120, grayscale=True, i_init=i_init, seed=0)
    tr = pkg.StreamTracker(cfg, precision=precision)
    ref = oracle_for(cfg, i_init, 160, 120)
    worst = 0.0
    for v in frames:
        a = tr.push(pkg.FrameBuffer(160, 120, 1, v))
        b = ref.push(v)
        worst = max(worst, float(np.mean(a.mask.labels != b.mask)))
        if precision == "fp64":
            np.testing.assert_array_equal(a.raw_mask.labels, b.raw_mask)
            assert a.fit_cost == pytest.approx(b.fit_cost, rel=1e-10)
    bg = tr.background_frame().data
    rbg = ref.background()
    rel = np.linalg.norm(bg - rbg) / np.linalg.norm(rbg)
    ang = sine(tr.state.basis.data, ref.state.U)
    if precision == "fp64":
        assert rel <= 1e-10 and ang <= 1e-9
    else:
        assert worst <= 0.001 and rel <= 1e-4 and ang <= 1e-3


def test_batched_streams_bitwise_match_single_streams():
    """Streams batched into one launch give bit-identical results to the same
    streams run alone (deterministic fixed-order reductions)."""
    import torch

    W, H, S, F = 64, 48, 3, 8
    cfg = pkg.RunConfig(subspace_dim=15, p=0.5, mu=1e-4, cg_max_iters=2, target_width=W,
                        target_height=H, grayscale=True, i_init=4, seed=0)
    streams = [c0_stream(F, W, H, seed=s) for s in range(S)]
    bt = pkg.BatchTracker(cfg, S, seeds=[0, 1, 2])
    masks = torch.empty((S, W * H), dtype=torch.uint8, device="cuda")
    out_b = []
    for f in range(F):
        frames = torch.from_numpy(np.stack([s[f] for s in streams]).astype(np.float32)).cuda()
        bt.push(frames, mask=masks)
        out_b.append(masks.cpu().numpy().copy())
    bt.synchronize()
    for s in range(S):
        single = pkg.BatchTracker(cfg, 1, seeds=[s])
        m1 = torch.empty((1, W * H), dtype=torch.uint8, device="cuda")
        for f in range(F):
            single.push(torch.from_numpy(streams[s][f][None].astype(np.float32)).cuda(), mask=m1)
            np.testing.assert_array_equal(m1.cpu().numpy()[0], out_b[f][s])
        Ub = bt.native.get_core_state(s)[0]
        U1 = single.native.get_core_state(0)[0]
        np.testing.assert_array_equal(Ub, U1)


def test_cluster_team_sums_match_global_slots(monkeypatch):
    """Teams run as thread-block clusters (team sums over DSMEM with the
    hardware cluster barrier) give the same bits as the global-slot team sums
    (C0 shape, one-stream latency layout: G = 10 fits one cluster)."""
    import torch
    from paper_1302_2073_b200 import _native as nat

    W, H, F = 160, 120, 12
    frames = c0_stream(F)
    cfg = pkg.RunConfig(subspace_dim=15, p=0.5, mu=1e-4, cg_max_iters=2, target_width=W,
                        target_height=H, grayscale=True, i_init=4, seed=0)

    def run():
        bt = pkg.BatchTracker(cfg, 1, seeds=[0], latency=True)
        mask = torch.empty((1, W * H), dtype=torch.uint8, device="cuda")
        bg = torch.empty((1, W * H), dtype=torch.float32, device="cuda")
        out = []
        for f in range(F):
            info = bt.push(torch.from_numpy(frames[f][None].astype(np.float32)).cuda(), background=bg,
                           mask=mask, fit=True)
            out.append((mask.cpu().numpy().copy(), bg.cpu().numpy().copy(), info[0].fit_cost))
        return out, bt.native.get_core_state(0)[0], bt.native.query(nat.Q_CLUSTER)

    a, Ua, cla = run()
    monkeypatch.setenv("PROST_CLUSTER", "0")
    b, Ub, clb = run()
    assert (cla, clb) == (1, 0)
    for (ma, ba, ca), (mb, bb, cb) in zip(a, b):
        np.testing.assert_array_equal(ma, mb)
        np.testing.assert_array_equal(ba, bb)
        assert ca == cb
    np.testing.assert_array_equal(Ua, Ub)


def test_slice_prefetch_does_not_change_results(monkeypatch):
    """The L2 bulk prefetch of each slice's later slots (default on) only moves
    data earlier: C3 shape, 12 streams (one round of 11 teams and a second),
    bit-identical to PROST_PREFETCH=0."""
    import torch

    S, F = 12, 6
    W, H = 320, 240
    cfg = pkg.RunConfig(subspace_dim=15, p=0.5, mu=1e-4, cg_max_iters=2, target_width=W,
                        target_height=H, grayscale=True, i_init=3, seed=0)
    from paper_1302_2073_b200.synth import SceneStream, config_spec

    frames = np.stack([SceneStream(config_spec("C3", s)).next_frames(F) for s in range(S)], 1)

    def run():
        bt = pkg.BatchTracker(cfg, S, seeds=list(range(S)))
        mask = torch.empty((S, W * H), dtype=torch.uint8, device="cuda")
        bg = torch.empty((S, W * H), dtype=torch.float32, device="cuda")
        out = []
        for f in range(F):
            bt.push(torch.from_numpy(frames[f].astype(np.float32)).cuda(), background=bg, mask=mask)
            out.append((mask.cpu().numpy().copy(), bg.cpu().numpy().copy()))
        return out, bt.native.get_core_state(S - 1)[0]

    monkeypatch.setenv("PROST_PREFETCH", "1")
    a, Ua = run()
    monkeypatch.setenv("PROST_PREFETCH", "0")
    b, Ub = run()
    for (ma, ba), (mb, bb) in zip(a, b):
        np.testing.assert_array_equal(ma, mb)
        np.testing.assert_array_equal(ba, bb)
    np.testing.assert_array_equal(Ua, Ub)


def test_profiled_instance_matches(monkeypatch):
    """The k_tmem instance with the timing counters (profile(True), the
    bench's counters pass) computes the same bits as the counter-free one the
    frames normally run on: C3 shape, 12 streams, frames alternating between
    the two instances."""
    import torch
    from paper_1302_2073_b200.synth import SceneStream, config_spec

    S, F = 12, 6
    W, H = 320, 240
    cfg = pkg.RunConfig(subspace_dim=15, p=0.5, mu=1e-4, cg_max_iters=2, target_width=W,
                        target_height=H, grayscale=True, i_init=3, seed=0)
    frames = np.stack([SceneStream(config_spec("C3", s)).next_frames(F) for s in range(S)], 1)

    def run(alternate):
        bt = pkg.BatchTracker(cfg, S, seeds=list(range(S)))
        mask = torch.empty((S, W * H), dtype=torch.uint8, device="cuda")
        bg = torch.empty((S, W * H), dtype=torch.float32, device="cuda")
        out = []
        for f in range(F):
            bt.native.profile(alternate and f % 2 == 1)
            bt.push(torch.from_numpy(frames[f].astype(np.float32)).cuda(), background=bg, mask=mask)
            out.append((mask.cpu().numpy().copy(), bg.cpu().numpy().copy()))
        if alternate:  # the last profiled launch wrote its per-CTA counters
            assert bt.native.resident_counters()["rounds"] > 0
        bt.native.profile(False)
        return out, bt.native.get_core_state(S - 1)[0]

    a, Ua = run(False)
    b, Ub = run(True)
    for (ma, ba), (mb, bb) in zip(a, b):
        np.testing.assert_array_equal(ma, mb)
        np.testing.assert_array_equal(ba, bb)
    np.testing.assert_array_equal(Ua, Ub)


def test_large_batch_properties():
    """C3 shape (320x240, k=15) with 8 streams for 6 frames: size-independent
    properties — orthonormality, raw mask == threshold of the residual, mask ==
    3x3 majority of the raw mask, background inside [0, 1]."""
    import torch

    W, H, S, F = 320, 240, 8, 6
    cfg = pkg.RunConfig(subspace_dim=15, p=0.5, mu=1e-4, cg_max_iters=2, target_width=W,
                        target_height=H, grayscale=True, i_init=3, seed=0)
    bt = pkg.BatchTracker(cfg, S, seeds=list(range(S)))
    data = [c0_stream(F, W, H, seed=s) for s in range(S)]
    n = W * H
    mask = torch.empty((S, n), dtype=torch.uint8, device="cuda")
    raw = torch.empty((S, n), dtype=torch.uint8, device="cuda")
    res = torch.empty((S, n), dtype=torch.float32, device="cuda")
    bg = torch.empty((S, n), dtype=torch.float32, device="cuda")
    for f in range(F):
        fr = torch.from_numpy(np.stack([d[f] for d in data]).astype(np.float32)).cuda()
        info = bt.push(fr, background=bg, residual=res, mask=mask, raw_mask=raw, fit=True)
        assert all(info[s].frame_index == f + 1 for s in range(S))
        r = res.cpu().numpy()
        rm = raw.cpu().numpy()
        mk = mask.cpu().numpy()
        np.testing.assert_array_equal(rm, (np.abs(r) >= 0.35).astype(np.uint8))
        for s in range(S):
            np.testing.assert_array_equal(mk[s], orc.majority3x3(rm[s], W, H))
        b = bg.cpu().numpy()
        assert b.min() >= 0.0 and b.max() <= 1.0
    for s in range(S):
        U = bt.native.get_core_state(s)[0]
        assert np.linalg.norm(U.T @ U - np.eye(15)) < 1e-4


@pytest.mark.gpu
def test_tmem_k20_matches_streamed(monkeypatch):
    """k = 20 (BASELINE C2) runs on the TMEM kernel with 32-column rows and
    agrees with the streamed kernels."""
    import torch
    from paper_1302_2073_b200 import _native as nat

    W, H, S, F = 320, 240, 2, 8
    cfg = pkg.RunConfig(subspace_dim=20, p=0.5, mu=1e-4, cg_max_iters=2, target_width=W,
                        target_height=H, grayscale=True, i_init=4, seed=0)
    data = [c0_stream(F, W, H, seed=s) for s in range(S)]
    out = {}
    for path, code in (("tmem", 2), ("streamed", 0)):
        monkeypatch.setenv("PROST_KERNEL", path)
        bt = pkg.BatchTracker(cfg, S, seeds=list(range(S)))
        assert bt.native.query(nat.Q_RESIDENT) == code
        mask = torch.empty((S, W * H), dtype=torch.uint8, device="cuda")
        bg = torch.empty((S, W * H), dtype=torch.float32, device="cuda")
        for f in range(F):
            fr = torch.from_numpy(np.stack([d[f] for d in data]).astype(np.float32)).cuda()
            bt.push(fr, background=bg, mask=mask)
        out[path] = (mask.cpu().numpy(), bg.cpu().numpy())
    (m1, b1), (m2, b2) = out["tmem"], out["streamed"]
    assert np.mean(m1 != m2) <= 0.001
    assert np.linalg.norm(b1 - b2) <= 1e-5 * np.linalg.norm(b2)


def test_tmem_rgb_matches_streamed(monkeypatch):
    """Three channel planes (BASELINE C1) on the TMEM kernel: slices span the
    stacked planes, per-channel threshold flags are combined into the per-pixel
    label (pipeline.py:210-211) and the 3-channel weight expansion
    (jobs.py:218-221); agrees with the streamed kernels."""
    import torch
    from paper_1302_2073_b200 import _native as nat
    from paper_1302_2073_b200.synth import SceneSpec, SceneStream

    W, H, S, F = 96, 64, 2, 9
    cfg = pkg.RunConfig(subspace_dim=15, p=0.5, mu=1e-4, cg_max_iters=2, target_width=W,
                        target_height=H, grayscale=False, i_init=4, seed=0)
    data = [SceneStream(SceneSpec(width=W, height=H, channels=3, rank=6, n_objects=(2, 3),
                                  shape="ellipse", seed=s)).next_frames(F) for s in range(S)]
    out = {}
    for path, code in (("tmem", 2), ("streamed", 0)):
        monkeypatch.setenv("PROST_KERNEL", path)
        bt = pkg.BatchTracker(cfg, S, seeds=list(range(S)))
        assert bt.native.query(nat.Q_RESIDENT) == code
        mask = torch.empty((S, W * H), dtype=torch.uint8, device="cuda")
        raw = torch.empty((S, W * H), dtype=torch.uint8, device="cuda")
        bg = torch.empty((S, 3 * W * H), dtype=torch.float32, device="cuda")
        for f in range(F):
            fr = torch.from_numpy(np.stack([d[f] for d in data]).astype(np.float32)).cuda()
            bt.push(fr, background=bg, mask=mask, raw_mask=raw)
        out[path] = (mask.cpu().numpy(), raw.cpu().numpy(), bg.cpu().numpy())
    (m1, r1, b1), (m2, r2, b2) = out["tmem"], out["streamed"]
    assert np.mean(r1 != r2) <= 0.001 and np.mean(m1 != m2) <= 0.001
    assert np.linalg.norm(b1 - b2) <= 1e-5 * np.linalg.norm(b2)


@pytest.mark.parametrize("mode", ["tmem", "resident"])
def test_resident_kernels_match_streamed(mode, monkeypatch):
    """The TMEM-resident (default for fp32 single-channel streams) and the
    register-resident frame kernels agree with the multi-kernel streamed path
    on a C3-shaped batch."""
    import torch
    from paper_1302_2073_b200 import _native as nat

    W, H, S, F = 320, 240, 6, 8
    cfg = pkg.RunConfig(subspace_dim=15, p=0.5, mu=1e-4, cg_max_iters=2, target_width=W,
                        target_height=H, grayscale=True, i_init=4, seed=0)
    data = [c0_stream(F, W, H, seed=s) for s in range(S)]
    out = {}
    for path, code in ((mode, {"tmem": 2, "resident": 1}[mode]), ("streamed", 0)):
        monkeypatch.setenv("PROST_KERNEL", path)
        bt = pkg.BatchTracker(cfg, S, seeds=list(range(S)))
        assert bt.native.query(nat.Q_RESIDENT) == code
        mask = torch.empty((S, W * H), dtype=torch.uint8, device="cuda")
        bg = torch.empty((S, W * H), dtype=torch.float32, device="cuda")
        for f in range(F):
            fr = torch.from_numpy(np.stack([d[f] for d in data]).astype(np.float32)).cuda()
            info = bt.push(fr, background=bg, mask=mask, fit=True)
        out[path] = (mask.cpu().numpy(), bg.cpu().numpy(),
                     [bt.native.get_core_state(s)[0] for s in range(S)],
                     [info[s].fit_cost for s in range(S)])
    (m1, b1, U1, c1), (m2, b2, U2, c2) = out[mode], out["streamed"]
    assert np.mean(m1 != m2) <= 0.001
    assert np.linalg.norm(b1 - b2) <= 1e-5 * np.linalg.norm(b2)
    for s in range(S):
        assert sine(U1[s], U2[s]) <= 1e-4
        assert c1[s] == pytest.approx(c2[s], rel=1e-5)


@pytest.mark.gpu
def test_pipelined_host_io_matches_device_io():
    """Host frames in / host outputs out run pipelined on the handle's own
    streams (copies of one frame overlap the kernels of the next); the results
    equal the device-buffer path's, frame after frame and back to back."""
    import torch

    W, H, S, F = 64, 48, 4, 9
    cfg = pkg.RunConfig(subspace_dim=8, p=0.5, mu=1e-4, cg_max_iters=2, target_width=W,
                        target_height=H, grayscale=True, i_init=4, seed=0)
    data = np.stack([c0_stream(F, W, H, seed=s) for s in range(S)], 1).astype(np.float32)
    dev_bt = pkg.BatchTracker(cfg, S, seeds=list(range(S)))
    host_bt = pkg.BatchTracker(cfg, S, seeds=list(range(S)))
    mask_d = torch.empty((S, W * H), dtype=torch.uint8, device="cuda")
    bg_d = torch.empty((S, W * H), dtype=torch.float32, device="cuda")
    frames_h = [torch.from_numpy(data[f]).pin_memory() for f in range(F)]
    mask_h = [torch.empty((S, W * H), dtype=torch.uint8).pin_memory() for _ in range(F)]
    bg_h = [torch.empty((S, W * H), dtype=torch.float32).pin_memory() for _ in range(F)]
    ref_masks, ref_bgs = [], []
    for f in range(F):
        dev_bt.push(torch.from_numpy(data[f]).cuda(), background=bg_d, mask=mask_d)
        ref_masks.append(mask_d.cpu().numpy())
        ref_bgs.append(bg_d.cpu().numpy())
    for f in range(F):  # back to back, every frame its own output buffers
        host_bt.push(frames_h[f], background=bg_h[f], mask=mask_h[f])
    host_bt.join()
    torch.cuda.synchronize()
    for f in range(F):
        np.testing.assert_array_equal(mask_h[f].numpy(), ref_masks[f])
        np.testing.assert_array_equal(bg_h[f].numpy(), ref_bgs[f])
    U_d = dev_bt.native.get_core_state(0)[0]
    U_h = host_bt.native.get_core_state(0)[0]
    np.testing.assert_array_equal(U_h, U_d)


@pytest.mark.gpu
@pytest.mark.parametrize("k", [8, 30])
def test_u8_frame_ingest(k):
    """8-bit frames are divided by 255 on load (frameio.py:136, SURVEY §8(f)
    row 1): the same result as pushing the scaled float32 frames — the TMEM
    kernel (k = 8) and the TMA-fed streamed kernels (k = 30: statistics,
    pass 0, geodesic sweep read the bytes themselves)."""
    import torch
    from paper_1302_2073_b200 import _native as nat

    W, H, S, F = (64, 48, 3, 6) if k == 8 else (128, 64, 2, 8)
    cfg = pkg.RunConfig(subspace_dim=k, p=0.5, mu=1e-4, cg_max_iters=2, target_width=W,
                        target_height=H, grayscale=True, i_init=3, seed=0)
    data = np.stack([c0_stream(F, W, H, seed=s) for s in range(S)], 1)
    q = np.clip(np.rint(data * 255.0), 0, 255).astype(np.uint8)
    q[0, 0, :256] = np.arange(256)  # every 8-bit value through the device conversion
    scaled = (q.astype(np.float64) * (1.0 / 255.0)).astype(np.float32)
    outs = []
    for frames in (q, scaled):
        bt = pkg.BatchTracker(cfg, S, seeds=list(range(S)))
        assert (bt.native.query(nat.Q_TMA) > 0) == (k == 30)
        mask = torch.empty((S, W * H), dtype=torch.uint8, device="cuda")
        bg = torch.empty((S, W * H), dtype=torch.float32, device="cuda")
        for f in range(F):
            bt.push(torch.from_numpy(frames[f]).cuda(), background=bg, mask=mask)
        outs.append((mask.cpu().numpy(), bg.cpu().numpy()))
    np.testing.assert_array_equal(outs[0][0], outs[1][0])
    np.testing.assert_array_equal(outs[0][1], outs[1][1])


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
@pytest.mark.parametrize("shape", [(30, 17), (41, 9)])
def test_ragged_shapes_against_oracle(precision, shape):
    """Widths that are not a multiple of 4 (byte-wise median path) and pixel
    counts that need padding (P % 4 != 0: padded rows carry weight 0), through
    the statistics window, against the oracle (fp32 runs the TMEM kernel)."""
    W, H = shape
    n_frames, i_init = 14, 5
    frames = c0_stream(n_frames, W, H, seed=5)
    cfg = pkg.RunConfig(subspace_dim=4, p=0.5, mu=1e-4, cg_max_iters=2, target_width=W,
                        target_height=H, grayscale=True, i_init=i_init, seed=2)
    tr = pkg.StreamTracker(cfg, precision=precision)
    ref = oracle_for(cfg, i_init, W, H)
    worst = 0.0
    for v in frames:
        a = tr.push(pkg.FrameBuffer(W, H, 1, v))
        b = ref.push(v)
        worst = max(worst, float(np.mean(a.mask.labels != b.mask)))
        if precision == "fp64":
            np.testing.assert_array_equal(a.raw_mask.labels, b.raw_mask)
            np.testing.assert_array_equal(a.mask.labels, b.mask)
    rel = np.linalg.norm(tr.background_frame().data - ref.background()) / np.linalg.norm(ref.background())
    ang = sine(tr.state.basis.data, ref.state.U)
    if precision == "fp64":
        assert rel <= 1e-10 and ang <= 1e-9
    else:
        assert worst <= 0.01 and rel <= 1e-4 and ang <= 1e-3


@pytest.mark.gpu
def test_pipelined_u8_frames_f64_outputs_async_fit():
    """Pinned 8-bit host frames in, float64 host backgrounds (converted through
    the download staging buffer), masks, raw masks and an asynchronously
    delivered FitInfo out, back to back on the pipelined path: identical to
    the synchronous device-buffer path (upload and download staging are
    separate buffers; raw labels and FitInfo have per-slot buffers)."""
    import torch

    W, H, S, F = 64, 48, 4, 9
    cfg = pkg.RunConfig(subspace_dim=8, p=0.5, mu=1e-4, cg_max_iters=2, target_width=W,
                        target_height=H, grayscale=True, i_init=4, seed=0)
    data = np.stack([c0_stream(F, W, H, seed=s) for s in range(S)], 1)
    q = np.clip(np.rint(data * 255.0), 0, 255).astype(np.uint8)
    dev_bt = pkg.BatchTracker(cfg, S, seeds=list(range(S)))
    host_bt = pkg.BatchTracker(cfg, S, seeds=list(range(S)))
    mask_d = torch.empty((S, W * H), dtype=torch.uint8, device="cuda")
    raw_d = torch.empty((S, W * H), dtype=torch.uint8, device="cuda")
    bg_d = torch.empty((S, W * H), dtype=torch.float64, device="cuda")
    ref = []
    for f in range(F):
        info = dev_bt.push(torch.from_numpy(q[f]).cuda(), background=bg_d, mask=mask_d,
                           raw_mask=raw_d, fit=True)
        ref.append((mask_d.cpu().numpy(), raw_d.cpu().numpy(), bg_d.cpu().numpy(),
                    [info[s].fit_cost for s in range(S)], [info[s].frame_index for s in range(S)]))
    frames_h = [torch.from_numpy(q[f]).pin_memory() for f in range(F)]
    outs = [(torch.empty((S, W * H), dtype=torch.uint8).pin_memory(),
             torch.empty((S, W * H), dtype=torch.uint8).pin_memory(),
             torch.empty((S, W * H), dtype=torch.float64).pin_memory(),
             pkg.FitInfoBuffer(S)) for _ in range(F)]
    for f in range(F):
        m, r, b, fi = outs[f]
        host_bt.push(frames_h[f], background=b, mask=m, raw_mask=r, fit_out=fi)
    host_bt.join()
    torch.cuda.synchronize()
    for f in range(F):
        m, r, b, fi = outs[f]
        np.testing.assert_array_equal(m.numpy(), ref[f][0])
        np.testing.assert_array_equal(r.numpy(), ref[f][1])
        np.testing.assert_array_equal(b.numpy(), ref[f][2])
        np.testing.assert_array_equal(fi.fit_costs(), np.array(ref[f][3]))
        assert [rec.frame_index for rec in fi.records()] == ref[f][4]


@pytest.mark.gpu
def test_off_resolution_frames_stay_on_device():
    """Off-resolution frames are resampled on the device and pushed from there
    (jobs.py:181-184): the same records as pushing the host-resampled frames
    (pipeline.py:164-193, bit-identical fp64 resampling)."""
    from paper_1302_2073_b200.resample import resample

    rng = np.random.default_rng(4)
    cfg = pkg.RunConfig(subspace_dim=4, p=0.5, mu=1e-4, cg_max_iters=2, target_width=24,
                        target_height=16, grayscale=True, i_init=3, seed=1)
    a, b = pkg.StreamTracker(cfg), pkg.StreamTracker(cfg)
    for _ in range(6):
        fb = pkg.FrameBuffer(37, 21, 1, rng.random(37 * 21))
        ra = a.push(fb)
        rb = b.push(resample(fb, 24, 16))
        np.testing.assert_array_equal(ra.mask.labels, rb.mask.labels)
        np.testing.assert_array_equal(ra.residual, rb.residual)
        assert ra.fit_cost == rb.fit_cost


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["f32", "u8"])
@pytest.mark.parametrize("path", ["tmem", "tma"])
def test_frame_blocking_matches_single_frame_pushes(dtype, path):
    """push_many (F frames per stream; the next frame's pass 0 run inside the
    geodesic sweep) gives bit-identical masks, raw masks, backgrounds,
    residuals, FitInfo and bases to pushing the same frames one at a time —
    across the statistics window (separate pass 0 there) and past it (fused).
    path "tmem": the slice kept on chip across the frames (k = 15); "tma": the
    TMA-fed streamed kernels (k = 30), k_geo_tma<K, true>."""
    import torch
    from paper_1302_2073_b200 import _native as nat

    if path == "tmem":
        W, H, S, F, B, K = 64, 48, 6, 12, 4, 15
    else:
        W, H, S, F, B, K = 128, 64, 2, 12, 4, 30
    cfg = pkg.RunConfig(subspace_dim=K, p=0.5, mu=1e-4, cg_max_iters=2, target_width=W,
                        target_height=H, grayscale=True, i_init=5, seed=0)
    data = np.stack([c0_stream(F, W, H, seed=s) for s in range(S)], 1)  # [F, S, n]
    if dtype == "u8":
        data = np.clip(np.rint(data * 255.0), 0, 255).astype(np.uint8)
    else:
        data = data.astype(np.float32)
    one = pkg.BatchTracker(cfg, S, seeds=list(range(S)))
    blk = pkg.BatchTracker(cfg, S, seeds=list(range(S)))
    if path == "tma":
        assert blk.native.query(nat.Q_TMA) > 0
    n = W * H
    ref = {k: [] for k in ("mask", "raw", "bg", "res", "cost", "fi")}
    m1 = torch.empty((S, n), dtype=torch.uint8, device="cuda")
    r1 = torch.empty((S, n), dtype=torch.uint8, device="cuda")
    b1 = torch.empty((S, n), dtype=torch.float32, device="cuda")
    e1 = torch.empty((S, n), dtype=torch.float32, device="cuda")
    for f in range(F):
        info = one.push(torch.from_numpy(data[f]).cuda(), background=b1, residual=e1, mask=m1,
                        raw_mask=r1, fit=True)
        ref["mask"].append(m1.cpu().numpy())
        ref["raw"].append(r1.cpu().numpy())
        ref["bg"].append(b1.cpu().numpy())
        ref["res"].append(e1.cpu().numpy())
        ref["cost"].append([info[s].fit_cost for s in range(S)])
        ref["fi"].append([info[s].frame_index for s in range(S)])
    mb = torch.empty((B, S, n), dtype=torch.uint8, device="cuda")
    rb = torch.empty((B, S, n), dtype=torch.uint8, device="cuda")
    bb = torch.empty((B, S, n), dtype=torch.float32, device="cuda")
    eb = torch.empty((B, S, n), dtype=torch.float32, device="cuda")
    for f0 in range(0, F, B):
        info = blk.push_many(torch.from_numpy(data[f0:f0 + B]).cuda(), background=bb, residual=eb,
                             mask=mb, raw_mask=rb, fit=True)
        for i in range(B):
            f = f0 + i
            np.testing.assert_array_equal(mb[i].cpu().numpy(), ref["mask"][f])
            np.testing.assert_array_equal(rb[i].cpu().numpy(), ref["raw"][f])
            np.testing.assert_array_equal(bb[i].cpu().numpy(), ref["bg"][f])
            np.testing.assert_array_equal(eb[i].cpu().numpy(), ref["res"][f])
            assert [info[i * S + s].fit_cost for s in range(S)] == ref["cost"][f]
            assert [info[i * S + s].frame_index for s in range(S)] == ref["fi"][f]
    for s in range(S):
        np.testing.assert_array_equal(blk.native.get_core_state(s)[0], one.native.get_core_state(s)[0])
    if path == "tma":  # host frames and host outputs through the same blocked path
        hst = pkg.BatchTracker(cfg, S, seeds=list(range(S)))
        mh = np.empty((B, S, n), dtype=np.uint8)
        bh = np.empty((B, S, n), dtype=np.float32)
        for f0 in range(0, F, B):
            hst.push_many(np.ascontiguousarray(data[f0:f0 + B]), background=bh, mask=mh)
            for i in range(B):
                np.testing.assert_array_equal(mh[i], ref["mask"][f0 + i])
                np.testing.assert_array_equal(bh[i], ref["bg"][f0 + i])
