"""Generate golden vectors by running the REFERENCE package itself.

Run in the build container (the only place /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src:/root/repo python tests/golden/make_golden.py

Writes small compressed fixtures next to this script.  They pin the CPU oracle
(`oracle/prost_oracle.py`, checked in `tests/test_oracle_golden.py`) and are
also used directly by the GPU parity tests.  Nothing at test or bench time
reads /root/reference.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(HERE.parents[1]))

import prost  # noqa: E402  (the reference)
from prost.cost import LpConfig, cost_and_gradient  # noqa: E402
from prost.fit import CgOptions, fit_coordinates  # noqa: E402
from prost.jobs import RunConfig, StreamTracker  # noqa: E402
from prost.manifold import SubspaceBasis, random_orthonormal  # noqa: E402
from prost.pipeline import FrameBuffer  # noqa: E402
from prost.tracker import ProstParams, bootstrap, process_frame  # noqa: E402

from paper_1302_2073_b200.synth import SceneSpec, SceneStream  # noqa: E402


def save(name, **arrays):
    path = HERE / f"{name}.npz"
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


def cost_vectors():
    rng = np.random.default_rng(11)
    out = {}
    for p in (0.25, 0.5, 0.7, 1.0, 2.0):
        r = rng.standard_normal(257) * 0.5
        w = np.where(rng.random(257) < 0.2, 5e-5, 1.0)
        c, g = cost_and_gradient(r, LpConfig(p=p, mu=1e-4), w)
        key = f"p{p}"
        out[key + "_r"], out[key + "_w"] = r, w
        out[key + "_cost"], out[key + "_grad"] = np.array(c), g
    save("cost_vectors", **out)


def fit_vectors():
    rng = np.random.default_rng(12)
    out = {}
    for case, (m, k, p, mu, iters) in enumerate(
        [(200, 4, 0.5, 1e-4, 2), (150, 6, 0.25, 0.02, 5), (90, 3, 2.0, 0.01, 5), (120, 5, 1.0, 1e-3, 3)]
    ):
        basis = random_orthonormal(m, k, seed=100 + case)
        x = basis.data @ rng.standard_normal(k)
        spikes = rng.choice(m, size=m // 8, replace=False)
        x[spikes] += rng.choice((-1.0, 1.0), size=spikes.size)
        y0 = None if case % 2 == 0 else rng.standard_normal(k)
        w = np.where(rng.random(m) < 0.1, 5e-5, 1.0)
        res = fit_coordinates(basis, x, y0, LpConfig(p=p, mu=mu), w, CgOptions(max_iters=iters))
        key = f"c{case}_"
        out[key + "U"], out[key + "x"], out[key + "w"] = basis.data, x, w
        out[key + "y0"] = np.full(k, np.nan) if y0 is None else y0
        out[key + "prm"] = np.array([p, mu, iters], dtype=float)
        out[key + "y"], out[key + "residual"] = res.y, res.residual
        out[key + "cost"] = np.array(res.cost)
        out[key + "counts"] = np.array([res.iterations, res.cost_evals, res.grad_evals])
    save("fit_vectors", **out)


def step_trajectory():
    """process_frame chain on a small normalized scene: every frame's state."""
    spec = SceneSpec(width=24, height=16, channels=1, rank=3, seed=5)
    frames = SceneStream(spec).next_frames(40)
    frames = (frames - frames[:10].mean(axis=0)) / frames[:10].std()
    params = ProstParams(k=4, cfg=LpConfig(p=0.5, mu=1e-4), delta=0.35, omega=5e-5,
                         t_init=5e-3, t_min=1e-4, tau=np.log(50) / 20,
                         cg=CgOptions(max_iters=2))
    state = bootstrap(spec.n, params, seed=7)
    U0 = state.basis.data.copy()
    Us, ys, ws, rs, costs, counts = [], [], [], [], [], []
    for x in frames:
        state, r, fit = process_frame(state, x, params)
        Us.append(state.basis.data)
        ys.append(state.y)
        ws.append(state.weights)
        rs.append(r)
        costs.append(fit.cost)
        counts.append([fit.iterations, fit.cost_evals, fit.grad_evals])
    save("step_trajectory", frames=frames, U0=U0, U=np.array(Us), y=np.array(ys),
         w=np.array(ws), residual=np.array(rs), cost=np.array(costs), counts=np.array(counts),
         prm=np.array([4, 0.5, 1e-4, 0.35, 5e-5, 5e-3, 1e-4, np.log(50) / 20, 2, 7]))


def qr_chain():
    """1003 tiny steps: the unconditional re-orthonormalization at step 1000."""
    rng = np.random.default_rng(13)
    params = ProstParams(k=3, cfg=LpConfig(p=0.5, mu=0.06125), delta=0.35, omega=5e-5,
                         t_init=1e-2, t_min=1e-3, tau=1e-3, cg=CgOptions(max_iters=2))
    state = bootstrap(48, params, seed=3)
    frames = rng.standard_normal((1003, 48))
    keep = {}
    for i, x in enumerate(frames):
        state, r, fit = process_frame(state, x, params)
        if i in (997, 998, 999, 1000, 1001, 1002):
            keep[f"U{i}"] = state.basis.data
            keep[f"y{i}"] = state.y
            keep[f"since{i}"] = np.array(state.basis.steps_since_qr)
    save("qr_chain", frames=frames, **keep)


def push_run(name, channels, n_frames=14, i_init=5):
    spec = SceneSpec(width=32, height=24, channels=channels, rank=3, n_objects=(2, 2),
                     seed=21 + channels, fg_from=3)
    raw = SceneStream(spec).next_frames(n_frames)
    cfg = RunConfig(subspace_dim=4, p=0.5, mu=1e-4, cg_max_iters=2, target_width=32,
                    target_height=24, grayscale=False, i_init=i_init, seed=9)
    tr = StreamTracker(cfg)
    masks, raws, res, costs, steps, bgs = [], [], [], [], [], []
    for v in raw:
        rec = tr.push(FrameBuffer(32, 24, channels, v))
        masks.append(rec.mask.labels)
        raws.append(rec.raw_mask.labels)
        res.append(rec.residual)
        costs.append(rec.fit_cost)
        steps.append(rec.step)
        bgs.append(tr.background_frame().data)
    st = tr.state
    save(name, frames=raw, mask=np.array(masks), raw_mask=np.array(raws),
         residual=np.array(res), fit_cost=np.array(costs), step=np.array(steps),
         background=np.array(bgs), U=st.basis.data, y=st.y, w=st.weights,
         mean=tr.stats.mean, std=np.array(tr.stats.std),
         cfg=np.array([4, 0.5, 1e-4, 2, i_init, 9, channels]))


def snapshot_run(n_before=8, n_after=6, i_init=5):
    """PROSTSNAP1 bytes of a gray StreamTracker after n_before frames, and the
    reference's continuation after restore_bytes (jobs.py:241-277)."""
    spec = SceneSpec(width=32, height=24, channels=1, rank=3, n_objects=(2, 2), seed=31, fg_from=2)
    raw = SceneStream(spec).next_frames(n_before + n_after)
    cfg = RunConfig(subspace_dim=4, p=0.5, mu=1e-4, cg_max_iters=2, target_width=32,
                    target_height=24, grayscale=True, i_init=i_init, seed=4)
    tr = StreamTracker(cfg)
    for v in raw[:n_before]:
        tr.push(FrameBuffer(32, 24, 1, v))
    blob = tr.snapshot_bytes()
    tr2 = StreamTracker.restore_bytes(blob, cfg)
    masks, bgs, costs = [], [], []
    for v in raw[n_before:]:
        rec = tr2.push(FrameBuffer(32, 24, 1, v))
        masks.append(rec.mask.labels)
        costs.append(rec.fit_cost)
        bgs.append(tr2.background_frame().data)
    save("snapshot_gray", frames=raw, blob=np.frombuffer(blob, dtype=np.uint8),
         mask=np.array(masks), background=np.array(bgs), fit_cost=np.array(costs),
         cfg=np.array([4, 0.5, 1e-4, 2, i_init, 4, n_before]))


def resample_vectors():
    """pipeline.py:164-193 and 245-258 of the reference on seeded inputs."""
    from prost.pipeline import SegmentationMask, resample, upsample_mask

    rng = np.random.default_rng(17)
    keep = {}
    cases = [(1, 37, 23, 16, 12), (3, 20, 15, 33, 27), (1, 40, 30, 80, 60), (3, 64, 48, 32, 24)]
    for i, (c, w, h, ow, oh) in enumerate(cases):
        data = rng.random(c * w * h)
        out = resample(FrameBuffer(w, h, c, data), ow, oh)
        keep[f"in{i}"] = data
        keep[f"out{i}"] = out.data
        keep[f"dims{i}"] = np.array([c, w, h, ow, oh])
        lab = (rng.random(w * h) < 0.3).astype(np.uint8)
        up = upsample_mask(SegmentationMask(w, h, lab), ow, oh)
        keep[f"lab{i}"] = lab
        keep[f"up{i}"] = up.labels
    save("resample_vectors", **keep)


def confusion_vectors():
    """evaluate.py:87-106 of the reference on seeded masks and ground truth."""
    from prost.evaluate import ConfusionCounts, accumulate
    from prost.frameio import GroundTruthFrame
    from prost.pipeline import SegmentationMask

    rng = np.random.default_rng(23)
    keep = {}
    levels = np.array([0, 50, 85, 170, 255], dtype=np.uint8)
    for i, (w, h) in enumerate([(32, 24), (160, 120), (7, 5)]):
        lab = (rng.random(w * h) < 0.3).astype(np.uint8)
        gt = levels[rng.integers(0, 5, size=w * h)]
        c = accumulate(ConfusionCounts(), SegmentationMask(w, h, lab), GroundTruthFrame(w, h, gt))
        keep[f"mask{i}"] = lab
        keep[f"gt{i}"] = gt
        keep[f"dims{i}"] = np.array([w, h])
        keep[f"counts{i}"] = np.array([c.tp, c.fp, c.tn, c.fn])
    save("confusion_vectors", **keep)


def pnm_vectors():
    """frameio.decode_pnm of the reference on P5 / P6 bytes with varied headers."""
    from prost.frameio import decode_pnm

    rng = np.random.default_rng(29)
    keep = {}
    specs = [(b"P5", 7, 5, b"P5\n7 5\n255\n"), (b"P6", 6, 4, b"P6 6\t4 255\n"),
             (b"P6", 33, 17, b"P6\n  33   17\n255 ")]
    for i, (magic, w, h, header) in enumerate(specs):
        c = 1 if magic == b"P5" else 3
        blob = header + rng.integers(0, 256, size=w * h * c, dtype=np.uint8).tobytes() + b"tail"
        fb = decode_pnm(blob)
        keep[f"blob{i}"] = np.frombuffer(blob, dtype=np.uint8)
        keep[f"data{i}"] = fb.data
        keep[f"dims{i}"] = np.array([fb.width, fb.height, fb.channels])
    save("pnm_vectors", **keep)


if __name__ == "__main__":
    print("reference prost", prost.__version__, "numpy", np.__version__)
    cost_vectors()
    fit_vectors()
    step_trajectory()
    qr_chain()
    push_run("push_gray", 1)
    push_run("push_rgb", 3)
    snapshot_run()
    resample_vectors()
    confusion_vectors()
    pnm_vectors()
