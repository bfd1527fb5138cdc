"""Seeded synthetic video streams for the BASELINE configurations.

The reference ships no generator for these streams; the
paper's changedetection.net data is not available here either, so these
seeded streams stand in for it with the shapes, ranks and value ranges that
`BASELINE.json` states.  Builder-fixed choices (marked † in SURVEY.md) are
fixed here once and echoed by `SceneSpec.describe()`.

Model per frame t (all intensities on the [0, 1] scale the reference uses,
`pipeline.py:1-11`):

    bg_t  = clip(mu0 + A * B c_t, 0, 1),  B ~ N(0,1)^{n x rank},
            c_0 ~ N(0, I),  c_{t+1} = c_t + walk * N(0, I)
    frame = clip(paint(bg_t, objects_t) + N(0, noise^2), 0, 1)

Objects are axis-aligned rectangles or filled ellipses with a uniform
intensity (one value per channel), moving with an integer velocity and
bouncing off the frame edges.  With `jitter > 0` the background is drawn on
a larger canvas and cropped at a seeded integer offset each frame (bilinear
resampling at integer shifts is an exact crop).
"""

from __future__ import annotations

from dataclasses import dataclass, asdict

import numpy as np

__all__ = ["SceneSpec", "SceneStream", "CONFIGS", "config_spec"]


@dataclass(frozen=True)
class SceneSpec:
    width: int
    height: int
    channels: int = 1
    rank: int = 5
    amplitude: float = 0.05
    walk: float = 0.01
    mean_lo: float = 0.3
    mean_hi: float = 0.7
    n_objects: tuple = (1, 3)
    area: tuple = (0.10, 0.20)      # total object area as a fraction of the frame
    shape: str = "rect"             # "rect" or "ellipse"
    max_speed: int = 3
    noise: float = 0.02
    jitter: int = 0
    fg_from: int = 0                # first frame with foreground
    seed: int = 0

    @property
    def pixels(self) -> int:
        return self.width * self.height

    @property
    def n(self) -> int:
        return self.pixels * self.channels

    def describe(self) -> dict:
        d = asdict(self)
        d["n_objects"] = list(self.n_objects)
        d["area"] = list(self.area)
        return d


class SceneStream:
    """Deterministic frame source: `next_frames(count)` continues the stream."""

    def __init__(self, spec: SceneSpec, dtype=np.float64):
        self.spec = spec
        self.dtype = dtype
        rng = np.random.default_rng(spec.seed)
        self._rng = rng
        cw = spec.width + 2 * spec.jitter
        ch = spec.height + 2 * spec.jitter
        self._canvas = (spec.channels, ch, cw)
        cn = spec.channels * ch * cw
        self._mu0 = rng.uniform(spec.mean_lo, spec.mean_hi, size=cn)
        self._basis = rng.standard_normal((cn, spec.rank))
        self._coef = rng.standard_normal(spec.rank)
        n_obj = int(rng.integers(spec.n_objects[0], spec.n_objects[1] + 1))
        total = rng.uniform(spec.area[0], spec.area[1]) * spec.pixels
        share = rng.dirichlet(np.ones(n_obj)) * total
        self._objects = []
        for a in share:
            aspect = rng.uniform(0.6, 1.6)
            if spec.shape == "ellipse":
                a = a * 4.0 / np.pi  # bounding box of an ellipse with area a
            h = int(np.clip(round(np.sqrt(a / aspect)), 2, spec.height - 1))
            w = int(np.clip(round(a / max(h, 1)), 2, spec.width - 1))
            y0 = int(rng.integers(0, spec.height - h + 1))
            x0 = int(rng.integers(0, spec.width - w + 1))
            vy, vx = (int(v) for v in rng.integers(-spec.max_speed, spec.max_speed + 1, size=2))
            color = rng.uniform(0.0, 1.0, size=spec.channels)
            self._objects.append([y0, x0, h, w, vy, vx, color])
        self._t = 0
        yy, xx = np.mgrid[0:spec.height, 0:spec.width]
        self._grid = (yy, xx)

    def _background(self) -> np.ndarray:
        s = self.spec
        bg = self._mu0 + s.amplitude * (self._basis @ self._coef)
        bg = bg.reshape(self._canvas)
        if s.jitter:
            dy, dx = (int(v) for v in self._rng.integers(-s.jitter, s.jitter + 1, size=2))
            y0 = s.jitter + dy
            x0 = s.jitter + dx
            bg = bg[:, y0:y0 + s.height, x0:x0 + s.width]
        return np.clip(bg, 0.0, 1.0)

    def _paint(self, img: np.ndarray, fg=None) -> None:
        s = self.spec
        yy, xx = self._grid
        for ob in self._objects:
            y0, x0, h, w, vy, vx, color = ob
            if s.shape == "ellipse":
                cy, cx = y0 + (h - 1) / 2.0, x0 + (w - 1) / 2.0
                sel = ((yy - cy) / (h / 2.0)) ** 2 + ((xx - cx) / (w / 2.0)) ** 2 <= 1.0
                for c in range(s.channels):
                    img[c][sel] = color[c]
                if fg is not None:
                    fg[sel] = 1
            else:
                for c in range(s.channels):
                    img[c, y0:y0 + h, x0:x0 + w] = color[c]
                if fg is not None:
                    fg[y0:y0 + h, x0:x0 + w] = 1
            # advance with bouncing
            ny, nx = y0 + vy, x0 + vx
            if ny < 0 or ny + h > s.height:
                vy = -vy
                ny = min(max(y0 + vy, 0), s.height - h)
            if nx < 0 or nx + w > s.width:
                vx = -vx
                nx = min(max(x0 + vx, 0), s.width - w)
            ob[0], ob[1], ob[4], ob[5] = ny, nx, vy, vx

    def next_frames(self, count: int, truth: bool = False):
        """Return the next `count` frames as a (count, n) array (channel-planar).

        With `truth=True` also the ground truth the frames were drawn from
        (same random stream): (frames, foreground masks u8 (count, pixels),
        clean backgrounds (count, n))."""
        s = self.spec
        out = np.empty((count, s.n), dtype=self.dtype)
        if truth:
            fgs = np.zeros((count, s.pixels), dtype=np.uint8)
            bgs = np.empty((count, s.n))
        for i in range(count):
            img = self._background()
            if truth:
                bgs[i] = img.reshape(-1)
            if self._t >= s.fg_from:
                self._paint(img, fgs[i].reshape(s.height, s.width) if truth else None)
            if s.noise > 0.0:
                img = img + self._rng.normal(0.0, s.noise, size=img.shape)
            out[i] = np.clip(img, 0.0, 1.0).reshape(-1)
            self._coef = self._coef + s.walk * self._rng.standard_normal(s.rank)
            self._t += 1
        return (out, fgs, bgs) if truth else out


# Tracker settings per BASELINE config; the generator specs
# are builder-fixed stand-ins for the reference's absent dataset.
CONFIGS = {
    "C0": dict(tracker=dict(subspace_dim=15, p=0.5, mu=1e-4, cg_max_iters=2,
                            target_width=160, target_height=120, grayscale=True),
               scene=dict(width=160, height=120, channels=1, rank=5, noise=0.02),
               frames=300, streams=1),
    "C1": dict(tracker=dict(subspace_dim=15, p=0.5, mu=1e-4, cg_max_iters=2,
                            target_width=320, target_height=240, grayscale=False),
               scene=dict(width=320, height=240, channels=3, rank=8, n_objects=(4, 6),
                          shape="ellipse", noise=0.02, fg_from=0),
               frames=1000, streams=1),
    "C2": dict(tracker=dict(subspace_dim=20, p=0.5, mu=1e-4, cg_max_iters=2,
                            target_width=640, target_height=480, grayscale=True),
               scene=dict(width=640, height=480, channels=1, rank=6, noise=0.03,
                          jitter=3, area=(0.03, 0.08)),
               frames=2000, streams=1),
    "C3": dict(tracker=dict(subspace_dim=15, p=0.5, mu=1e-4, cg_max_iters=2,
                            target_width=320, target_height=240, grayscale=True),
               scene=dict(width=320, height=240, channels=1, rank=5, noise=0.02),
               frames=1000, streams=256),
    "C4": dict(tracker=dict(subspace_dim=30, p=0.5, mu=1e-4, cg_max_iters=2,
                            target_width=3840, target_height=2160, grayscale=True),
               scene=dict(width=3840, height=2160, channels=1, rank=10, noise=0.02,
                          area=(0.03, 0.08), max_speed=8),
               frames=500, streams=1, shard="pixel"),
}


def config_spec(name: str, stream: int = 0, **overrides) -> SceneSpec:
    """SceneSpec of BASELINE config `name` for stream index `stream` (seed = stream)."""
    kw = dict(CONFIGS[name]["scene"])
    kw.update(overrides)
    kw.setdefault("seed", stream)
    return SceneSpec(**kw)


class DeviceScenes:
    """The same scene model for many streams at once, advanced on a CUDA device
    (torch) so that benchmarks can stage long runs of consecutive frames in
    HBM.  Stream s starts from exactly the state `SceneStream(specs[s])` draws
    (background mean, basis, coefficients, objects); the per-frame random walk
    and pixel noise then come from a seeded torch generator, so the frames
    follow the model but are not bit-identical to `SceneStream`'s.  Background
    jitter (C2) is not supported here.
    """

    def __init__(self, specs, device, seed: int = 0):
        import torch

        if any(s.jitter for s in specs):
            raise ValueError("DeviceScenes does not model background jitter")
        s0 = specs[0]
        if any((s.width, s.height, s.channels, s.rank) != (s0.width, s0.height, s0.channels, s0.rank)
               for s in specs):
            raise ValueError("all streams must share shape and rank")
        self.torch = torch
        self.specs = list(specs)
        self.dev = torch.device(device)
        self.gen = torch.Generator(device=self.dev)
        self.gen.manual_seed(seed)
        S, C, H, W = len(specs), s0.channels, s0.height, s0.width
        self.shape = (S, C, H, W)
        host = [SceneStream(s, dtype=np.float32) for s in specs]
        f32 = dict(dtype=torch.float32, device=self.dev)
        self.mu0 = torch.tensor(np.stack([h._mu0 for h in host]), **f32)            # [S, n]
        self.basis = torch.tensor(np.stack([h._basis for h in host]), **f32)        # [S, n, r]
        self.coef = torch.tensor(np.stack([h._coef for h in host]), **f32)          # [S, r]
        self.amp = torch.tensor([s.amplitude for s in specs], **f32)[:, None]
        self.walk = torch.tensor([s.walk for s in specs], **f32)[:, None]
        self.noise = torch.tensor([s.noise for s in specs], **f32)[:, None]
        self.fg_from = torch.tensor([s.fg_from for s in specs], device=self.dev)
        nob = max(len(h._objects) for h in host)
        i32 = dict(dtype=torch.int64, device=self.dev)
        ob = np.zeros((S, nob, 6), dtype=np.int64)
        col = np.zeros((S, nob, C), dtype=np.float32)
        act = np.zeros((S, nob), dtype=bool)
        for i, h in enumerate(host):
            for j, o in enumerate(h._objects):
                ob[i, j] = o[:6]
                col[i, j] = o[6]
                act[i, j] = True
        self.ob = torch.tensor(ob, **i32)      # y0, x0, h, w, vy, vx
        self.col = torch.tensor(col, **f32)    # [S, nob, C]
        self.act = torch.tensor(act, device=self.dev)
        self.ellipse = torch.tensor([s.shape == "ellipse" for s in specs], device=self.dev)
        self.yy = torch.arange(H, device=self.dev)[None, :, None]
        self.xx = torch.arange(W, device=self.dev)[None, None, :]
        self.t = 0

    def _frame(self):
        torch = self.torch
        S, C, H, W = self.shape
        bg = self.mu0 + self.amp * torch.bmm(self.basis, self.coef[:, :, None])[:, :, 0]
        img = bg.clamp(0.0, 1.0).view(S, C, H, W)
        paint = self.t >= self.fg_from  # [S]
        for j in range(self.ob.shape[1]):
            y0, x0, h, w, vy, vx = (self.ob[:, j, c] for c in range(6))
            rect = ((self.yy >= y0[:, None, None]) & (self.yy < (y0 + h)[:, None, None]) &
                    (self.xx >= x0[:, None, None]) & (self.xx < (x0 + w)[:, None, None]))
            cy = (y0 + (h - 1) / 2.0)[:, None, None]
            cx = (x0 + (w - 1) / 2.0)[:, None, None]
            ell = (((self.yy - cy) / (h / 2.0)[:, None, None]) ** 2 +
                   ((self.xx - cx) / (w / 2.0)[:, None, None]) ** 2) <= 1.0
            sel = torch.where(self.ellipse[:, None, None], ell, rect)
            sel = sel & (self.act[:, j] & paint)[:, None, None]
            img = torch.where(sel[:, None], self.col[:, j, :, None, None], img)
            # advance with bouncing (SceneStream._paint)
            ny, nx = y0 + vy, x0 + vx
            by = (ny < 0) | (ny + h > H)
            bx = (nx < 0) | (nx + w > W)
            vy = torch.where(by, -vy, vy)
            vx = torch.where(bx, -vx, vx)
            ny = torch.where(by, torch.minimum(torch.clamp(y0 + vy, min=0), H - h), ny)
            nx = torch.where(bx, torch.minimum(torch.clamp(x0 + vx, min=0), W - w), nx)
            adv = paint & self.act[:, j]
            self.ob[:, j, 0] = torch.where(adv, ny, y0)
            self.ob[:, j, 1] = torch.where(adv, nx, x0)
            self.ob[:, j, 4] = torch.where(adv, vy, self.ob[:, j, 4])
            self.ob[:, j, 5] = torch.where(adv, vx, self.ob[:, j, 5])
        img = img.reshape(S, -1)
        img = img + self.noise * torch.randn(img.shape, generator=self.gen, device=self.dev)
        self.coef = self.coef + self.walk * torch.randn(self.coef.shape, generator=self.gen,
                                                        device=self.dev)
        self.t += 1
        return img.clamp_(0.0, 1.0)

    def next_frames(self, count: int):
        """The next `count` frames of every stream: a float32 [count, S, n] tensor."""
        S, C, H, W = self.shape
        out = self.torch.empty((count, S, C * H * W), dtype=self.torch.float32, device=self.dev)
        for i in range(count):
            out[i] = self._frame()
        return out
