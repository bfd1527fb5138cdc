"""Parity drivers shared by the GPU tests: the CUDA path (through the C-ABI,
`BatchTracker` / `NativeTracker`) against the CPU oracle (`oracle/`, pinned
bit-exactly to the reference by tests/test_oracle_golden.py) on the same
seeded BASELINE-config streams.

Two protocols (SURVEY.md §8(c) tiers 1-2):

* teacher forced (`teacher_forced`): before every frame the checked streams of
  the batch are loaded with the oracle's exact state (basis, coordinates,
  weights, frame index, running statistics) through `prost_set_core_state` /
  `prost_set_preproc`; one GPU frame then runs for the whole batch and is
  compared with the oracle's next state.  This isolates the kernel's own error
  from the reference's chaotic amplification (a perturbation at fp32 rounding
  level grows ~25% per frame at mu = 1e-4; tools/horizon.py).
* free running (`free_running`): both run on their own up to a frame budget
  (the measured self-divergence horizon), compared every frame.

Frames are the fp32 frames the GPU receives, widened to float64 for the
oracle, so the inputs are identical.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from oracle import prost_oracle as orc

import paper_1302_2073_b200 as pkg
from paper_1302_2073_b200.synth import CONFIGS, SceneStream, config_spec
from paper_1302_2073_b200.tracker import PreprocSnapshot


def oracle_for(cfg, i_init, width, height, channels, seed):
    prm = cfg.params(i_init)
    return orc.PipelineOracle(width, height, channels, orc.OracleParams(
        k=prm.k, p=prm.cfg.p, mu=prm.cfg.mu, delta=prm.delta, omega=prm.omega,
        t_init=prm.t_init, t_min=prm.t_min, tau=prm.tau, max_iters=prm.cg.max_iters),
        i_init=i_init, seed=seed)


def config_frames(name, stream, count, **over):
    """`count` consecutive fp32 frames of BASELINE config `name`, stream `stream`."""
    return SceneStream(config_spec(name, stream, **over), dtype=np.float64).next_frames(
        count).astype(np.float32)


def force(native, s, o):
    """Load stream s of a native handle with the oracle's state."""
    st, nz = o.state, o.norm
    native.set_core_state(s, st.U, st.y, st.w, st.frame_index, st.since_qr)
    native.set_preproc(s, PreprocSnapshot(mean=nz.mean, frames_seen=nz.seen, frozen=nz.frozen,
                                          std=nz.std, value_sum=nz.s1, value_sumsq=nz.s2,
                                          value_count=nz.count))


@dataclass
class Worst:
    """Worst per-frame disagreement over the stream-frames whose CG decisions
    (iterations, Armijo cost evaluations) match the oracle's, and a separate
    record of the frames where they differ.

    A decision can only differ where the reference itself sits on a near-tie:
    its Armijo test `cost(trial) <= f + c*alpha*slope` holds or fails by a
    relative margin below the fp32 path's cost error (the oracle reports the
    margin, `Fit.armijo_margin`).  Such ties occur every ~10-20 frames per
    C3 stream at mu = 1e-4 (margins down to 1e-12 measured), and taking the
    other branch changes that frame's step legitimately (one-step sine up to
    ~4e-4), so those frames are held to the north_star tolerances instead and
    each must be a reference near-tie."""

    sine: float = 0.0
    bg_rel: float = 0.0
    raw: float = 0.0
    mask: float = 0.0
    cost_rel: float = 0.0
    frames: int = 0
    same_decisions: int = 0
    flips: list = field(default_factory=list)  # (t, s, sine, bg_rel, mask, oracle margin)
    log: list = field(default_factory=list)

    def add(self, t, s, sine, bg_rel, raw, mask, cost_rel, same, margin=float("nan")):
        self.frames += 1
        self.log.append((t, s, sine, bg_rel, raw, mask, cost_rel, bool(same), margin))
        self.raw = max(self.raw, raw)
        self.mask = max(self.mask, mask)
        if not same:
            self.flips.append((t, s, sine, bg_rel, mask, margin))
            return
        self.same_decisions += 1
        self.sine = max(self.sine, sine)
        self.bg_rel = max(self.bg_rel, bg_rel)
        self.cost_rel = max(self.cost_rel, cost_rel)

    @property
    def decision_rate(self) -> float:
        return self.same_decisions / max(1, self.frames)

    @property
    def first_flip(self):
        return min((f[0] for f in self.flips), default=None)

    def __str__(self):
        fl = ", ".join(f"t={t} s={s} sine={a:.1e} margin={m:.1e}" for t, s, a, _, _, m in self.flips)
        return (f"{self.frames} stream-frames: sine {self.sine:.2e}, bg relL2 {self.bg_rel:.2e}, "
                f"raw mask {self.raw:.5f}, mask {self.mask:.5f}, cost rel {self.cost_rel:.2e}, "
                f"identical decisions {self.decision_rate:.4f} (differing: {fl or 'none'})")


class BatchRun:
    """A BatchTracker of `n_streams` streams of BASELINE config `name`
    (stream s seeded with s for both its frames and its basis) plus oracles
    for the `check` streams."""

    def __init__(self, name, n_streams, check, n_frames, i_init=100, latency=False,
                 precision="fp32", truth=False, **scene_over):
        import torch

        self.torch = torch
        c = CONFIGS[name]
        tracker = dict(c["tracker"])
        if "height" in scene_over:
            tracker["target_height"] = scene_over["height"]
        self.cfg = pkg.RunConfig(i_init=i_init, **tracker)
        self.W, self.H = self.cfg.target_width, self.cfg.target_height
        self.C = 1 if self.cfg.grayscale else 3
        self.P = self.W * self.H
        self.n = self.P * self.C
        self.S = n_streams
        self.check = list(check)
        self.bt = pkg.BatchTracker(self.cfg, n_streams, seeds=list(range(n_streams)),
                                   precision=precision, latency=latency)
        # checked streams get their own scene; the others replay stream 0's
        # frames (their content does not matter, only that the batch is full)
        self.truth = None
        if truth:
            self.frames, self.truth = {}, {}
            for s in self.check:
                f, fg, bgt = SceneStream(config_spec(name, s, **scene_over),
                                         dtype=np.float64).next_frames(n_frames, truth=True)
                self.frames[s] = f.astype(np.float32)
                self.truth[s] = (fg, bgt)
            self.quality = {"gpu": {s: [] for s in self.check},
                            "oracle": {s: [] for s in self.check}}
        else:
            self.frames = {s: config_frames(name, s, n_frames, **scene_over) for s in self.check}
        filler = self.frames[self.check[0]]
        self.batch = np.empty((n_frames, n_streams, self.n), dtype=np.float32)
        for s in range(n_streams):
            self.batch[:, s] = self.frames.get(s, filler)
        self.oracles = {s: oracle_for(self.cfg, i_init, self.W, self.H, self.C, s)
                        for s in self.check}
        dev = "cuda"
        dt = torch.float32 if precision == "fp32" else torch.float64
        self.mask = torch.empty((n_streams, self.P), dtype=torch.uint8, device=dev)
        self.raw = torch.empty((n_streams, self.P), dtype=torch.uint8, device=dev)
        self.bg = torch.empty((n_streams, self.n), dtype=dt, device=dev)
        self.t = 0

    def step(self, forced: bool, compare: bool, worst: Worst):
        """Frame t for the whole batch (+ the oracles); compare the checked streams."""
        torch = self.torch
        t = self.t
        if forced and t > 0:
            for s in self.check:
                force(self.bt.native, s, self.oracles[s])
        x = torch.from_numpy(self.batch[t]).cuda()
        info = self.bt.push(x, background=self.bg, mask=self.mask, raw_mask=self.raw, fit=True)
        recs = {s: self.oracles[s].push(self.frames[s][t].astype(np.float64)) for s in self.check}
        if compare:
            bg = self.bg.cpu().numpy().astype(np.float64)
            mask = self.mask.cpu().numpy()
            raw = self.raw.cpu().numpy()
            for s in self.check:
                o, r = self.oracles[s], recs[s]
                assert info[s].frame_index == r.frame_index == t + 1
                U = self.bt.native.get_core_state(s)[0]
                rb = o.background()
                worst.add(
                    t, s,
                    orc.subspace_sine(U, o.state.U),
                    float(np.linalg.norm(bg[s] - rb) / np.linalg.norm(rb)),
                    float(np.mean(raw[s] != r.raw_mask)),
                    float(np.mean(mask[s] != r.mask)),
                    abs(info[s].fit_cost - r.fit_cost) / abs(r.fit_cost),
                    (info[s].iterations, info[s].cost_evals) == (r.fit.iterations,
                                                                 r.fit.cost_evals),
                    r.fit.armijo_margin)
        if self.truth is not None:
            bg = self.bg.cpu().numpy().astype(np.float64) if not compare else bg
            mask = self.mask.cpu().numpy() if not compare else mask
            for s in self.check:
                fg_true, bg_true = self.truth[s][0][t], self.truth[s][1][t]
                self.quality["gpu"][s].append((f_measure(mask[s], fg_true),
                                               rel_l2(bg[s], bg_true)))
                self.quality["oracle"][s].append((f_measure(recs[s].mask, fg_true),
                                                  rel_l2(self.oracles[s].background(), bg_true)))
        self.t += 1


def f_measure(mask, truth) -> float:
    """F1 of a foreground mask against the planted objects (evaluate.py's
    F-measure: 2PR / (P + R))."""
    tp = float(np.sum((mask != 0) & (truth != 0)))
    fp = float(np.sum((mask != 0) & (truth == 0)))
    fn = float(np.sum((mask == 0) & (truth != 0)))
    return 2 * tp / max(2 * tp + fp + fn, 1.0)


def rel_l2(a, b) -> float:
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def teacher_forced(run: BatchRun, frames, compare=lambda t: True) -> Worst:
    w = Worst()
    for _ in range(frames):
        run.step(forced=True, compare=compare(run.t), worst=w)
    return w


def free_running(run: BatchRun, frames) -> Worst:
    w = Worst()
    for _ in range(frames):
        run.step(forced=False, compare=True, worst=w)
    return w
