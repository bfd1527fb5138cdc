"""CPU oracle for the pROST per-frame hot path — TEST INFRASTRUCTURE ONLY.

This module is a plain-numpy (float64) restatement of the reference
algorithm for the path `BASELINE.json` names: the per-frame step
`process_frame` (reference `pkg/src/prost/tracker.py:121-156`) and the
`StreamTracker.push` pipeline around it (`pkg/src/prost/jobs.py:186-239`).

Rules:
  * Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline`
    / `--impl reference` leg may import it.  The product package
    `paper_1302_2073_b200` never does; it fails loudly when its CUDA library
    is missing.
  * It is pinned against golden vectors produced by running the reference
    package itself (`tests/golden/make_golden.py` → `tests/golden/*.npz`,
    checked by `tests/test_oracle_golden.py`).  The comparisons there are
    bit-exact where the arithmetic is the same sequence of numpy operations.

Every function cites the reference file:line it restates.  Paths are
relative to `/root/reference/pkg/src/prost/`.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

# manifold.py:35-40
DRIFT_TOL = 1e-8
NORM_FLOOR = 1e-14
QR_EVERY = 1000
# pipeline.py:19
STD_FLOOR = 1e-6


class OracleError(ValueError):
    """Raised where the reference raises one of its ProstError subclasses."""

    def __init__(self, kind: str, msg: str):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind


# --------------------------------------------------------------------------
# parameters


@dataclass(frozen=True)
class OracleParams:
    """Flattened ProstParams + LpConfig + CgOptions (tracker.py:45-76,
    cost.py:29-45, fit.py:24-47)."""

    k: int
    p: float
    mu: float
    delta: float
    omega: float = 1.0
    t_init: float = 5e-3
    t_min: float = 1e-4
    tau: float = 0.0
    max_iters: int = 5
    grad_tol: float = 1e-8
    initial_step: float = 1.0
    shrink: float = 0.5
    sufficient_decrease: float = 1e-4
    max_backtracks: int = 20


def decay_rate(t_init: float, t_min: float, i_init: int) -> float:
    """tracker.py:90-96."""
    return -float(np.log(t_min / t_init)) / i_init


def step_at(i: int, prm: OracleParams) -> float:
    """tracker.py:99-103."""
    return max(float(np.exp(-prm.tau * i)) * prm.t_init, prm.t_min)


def mu_from_delta(delta: float, p: float) -> float:
    """cost.py:115-127."""
    return delta * delta * (1.0 - p)


# --------------------------------------------------------------------------
# cost (cost.py:57-112)


def penalty(r: np.ndarray, p: float, mu: float):
    """Return (terms, base) with base = r^2 + mu (cost.py:57-66)."""
    base = r * r + mu
    if p == 2.0:
        return base, base
    if p == 1.0:
        return np.sqrt(base), base
    return np.exp((0.5 * p) * np.log(base)), base


def lp_cost(r: np.ndarray, p: float, mu: float, w=None) -> float:
    """cost.py:69-77."""
    terms, _ = penalty(r, p, mu)
    if w is not None:
        terms = terms * w
    return float(np.sum(terms))


def lp_cost_grad(r: np.ndarray, p: float, mu: float, w=None):
    """cost.py:80-93: (sum of weighted terms, p*r*terms/base)."""
    terms, base = penalty(r, p, mu)
    if w is not None:
        terms = terms * w
    return float(np.sum(terms)), (p * r) * (terms / base)


# --------------------------------------------------------------------------
# coordinate fit (fit.py:66-153)


@dataclass
class Fit:
    y: np.ndarray
    residual: np.ndarray
    cost: float
    iterations: int
    cost_evals: int
    grad_evals: int
    # parity-protocol instrumentation (not part of the reference's FitResult):
    # the smallest relative distance |cost - rhs| / |f| of any Armijo test of
    # this fit.  A second implementation whose cost differs from the
    # reference's by more than this may legitimately take the other branch.
    armijo_margin: float = float("inf")


def fit(U: np.ndarray, x: np.ndarray, y0, prm: OracleParams, w=None) -> Fit:
    """Polak–Ribière+ CG with Armijo backtracking, restated from fit.py:66-153."""
    if not np.all(np.isfinite(x)):
        raise OracleError("NonFiniteError", "frame contains non-finite values")
    k = U.shape[1]
    y = (U.T @ x) if y0 is None else y0.astype(float, copy=True)
    n_cost = 0
    n_grad = 0

    def value_and_coord_grad(res):
        nonlocal n_cost, n_grad
        n_cost += 1
        n_grad += 1
        c, g = lp_cost_grad(res, prm.p, prm.mu, w)
        return c, -(U.T @ g)

    res = x - U @ y
    f, gr = value_and_coord_grad(res)
    d = -gr
    done_iters = 0
    margin = float("inf")
    for it in range(prm.max_iters):
        gnorm = float(np.linalg.norm(gr))
        if gnorm <= prm.grad_tol:
            break
        if it > 0 and it % k == 0:
            d = -gr
        slope = float(d @ gr)
        if slope >= 0.0:
            d = -gr
            slope = -gnorm * gnorm
        ud = U @ d
        alpha = prm.initial_step
        ok = False
        for _ in range(prm.max_backtracks):
            trial = res - alpha * ud
            n_cost += 1
            tc = lp_cost(trial, prm.p, prm.mu, w)
            rhs = f + prm.sufficient_decrease * alpha * slope
            margin = min(margin, abs(tc - rhs) / max(abs(f), 1e-300))
            if tc <= rhs:
                ok = True
                break
            alpha *= prm.shrink
        if not ok:
            break
        done_iters = it + 1
        y = y + alpha * d
        res = trial
        f_new, gr_new = value_and_coord_grad(res)
        f = f_new
        beta = max(0.0, float(gr_new @ (gr_new - gr)) / (gnorm * gnorm))
        d = -gr_new + beta * d
        gr = gr_new
    return Fit(y, res, f, done_iters, n_cost, n_grad, margin)


# --------------------------------------------------------------------------
# Grassmann geometry (manifold.py:43-197)


def drift(U: np.ndarray) -> float:
    """manifold.py:43-46."""
    return float(np.linalg.norm(U.T @ U - np.eye(U.shape[1])))


def orthonormal_init(m: int, k: int, seed: int) -> np.ndarray:
    """manifold.py:100-113: Gaussian draw, thin QR, sign fix diag(R) > 0."""
    g = np.random.default_rng(seed).standard_normal((m, k))
    q, r = np.linalg.qr(g)
    return q * np.where(np.diag(r) < 0.0, -1.0, 1.0)


def rank_one_direction(U: np.ndarray, eta: np.ndarray, y: np.ndarray):
    """manifold.py:116-156 → (s, v, sigma); sigma == 0 flags a zero direction."""
    proj = eta - U @ (U.T @ eta)
    ln = float(np.linalg.norm(proj))
    rn = float(np.linalg.norm(y))
    if ln < NORM_FLOOR or rn < NORM_FLOOR:
        return np.zeros(U.shape[0]), np.zeros(U.shape[1]), 0.0
    return proj / ln, y / rn, ln * rn


def geodesic(U: np.ndarray, s, v, sigma: float, t: float, since_qr: int):
    """manifold.py:159-197 (descending). Returns (U', steps_since_qr')."""
    if t < 0.0:
        raise OracleError("ConfigError", "negative step")
    if sigma == 0.0 or t == 0.0:
        return U, since_qr
    phi = sigma * t
    in_span = U @ v
    Un = U + np.outer((np.cos(phi) - 1.0) * in_span + (-1.0 * np.sin(phi)) * s, v)
    since = since_qr + 1
    if since >= QR_EVERY or drift(Un) > DRIFT_TOL:
        q, r = np.linalg.qr(Un)
        Un = q * np.where(np.diag(r) < 0.0, -1.0, 1.0)
        since = 0
    return Un, since


# --------------------------------------------------------------------------
# one tracker step (tracker.py:121-156)


@dataclass
class CoreState:
    U: np.ndarray
    y: np.ndarray
    w: np.ndarray
    frame_index: int = 0
    since_qr: int = 0


def core_init(m: int, prm: OracleParams, seed: int) -> CoreState:
    """tracker.py:106-118."""
    return CoreState(orthonormal_init(m, prm.k, seed), np.zeros(prm.k), np.ones(m), 0, 0)


def core_step(st: CoreState, x: np.ndarray, prm: OracleParams):
    """tracker.py:121-156 → (new state, residual against U', Fit)."""
    if x.shape != (st.U.shape[0],):
        raise OracleError("DimensionError", "frame length")
    warm = None if st.frame_index == 0 else st.y
    ft = fit(st.U, x, warm, prm, st.w)
    # cost.py:103-112: eta = -(gradient wrt residual)
    eta = -lp_cost_grad(ft.residual, prm.p, prm.mu, st.w)[1]
    s, v, sigma = rank_one_direction(st.U, eta, ft.y)
    t = step_at(st.frame_index, prm)
    Un, since = geodesic(st.U, s, v, sigma, t, st.since_qr)
    res = x - Un @ ft.y
    w = np.where(np.abs(res) < prm.delta, 1.0, prm.omega)
    return CoreState(Un, ft.y, w, st.frame_index + 1, since), res, ft


# --------------------------------------------------------------------------
# image-side pipeline (pipeline.py:99-242, jobs.py:186-239)


@dataclass
class Normalizer:
    """Running mean + pooled std (pipeline.py:99-161)."""

    mean: np.ndarray
    seen: int = 0
    frozen: bool = False
    std: float = 0.0
    s1: float = 0.0
    s2: float = 0.0
    count: int = 0

    def fold(self, v: np.ndarray) -> None:  # pipeline.py:120-132
        self.seen += 1
        self.mean += (v - self.mean) / self.seen
        self.s1 += float(np.sum(v))
        self.s2 += float(np.sum(v * v))
        self.count += v.size

    def running_std(self) -> float:  # pipeline.py:134-140
        if self.count < 2:
            return STD_FLOOR
        var = (self.s2 - self.s1 ** 2 / self.count) / (self.count - 1)
        return max(float(np.sqrt(max(var, 0.0))), STD_FLOOR)

    def scale(self) -> float:  # pipeline.py:158-161
        return self.std if self.frozen else self.running_std()


def threshold(res: np.ndarray, pixels: int, channels: int, delta: float) -> np.ndarray:
    """pipeline.py:196-212: max over channel planes of |r| >= delta."""
    return (np.abs(res.reshape(channels, pixels)).max(axis=0) >= delta).astype(np.uint8)


def majority3x3(labels: np.ndarray, width: int, height: int) -> np.ndarray:
    """pipeline.py:215-228: sum of the edge-replicated 3x3 window >= 5."""
    g = np.pad(labels.reshape(height, width).astype(np.int32), 1, mode="edge")
    votes = sum(g[dy:dy + height, dx:dx + width] for dy in range(3) for dx in range(3))
    return (votes >= 5).astype(np.uint8).reshape(-1)


@dataclass
class PushRecord:
    frame_index: int
    mask: np.ndarray
    raw_mask: np.ndarray
    residual: np.ndarray
    fit_cost: float
    step: float
    fit: Fit = field(repr=False, default=None)


class PipelineOracle:
    """StreamTracker.push / background_frame restated (jobs.py:154-239) for
    frames already at model resolution (resample is the identity there,
    pipeline.py:172-173)."""

    def __init__(self, width: int, height: int, channels: int, prm: OracleParams,
                 i_init: int = 100, seed: int = 0):
        self.width, self.height, self.channels = width, height, channels
        self.prm, self.i_init, self.seed = prm, i_init, seed
        self.norm: Normalizer | None = None
        self.state: CoreState | None = None

    @property
    def pixels(self) -> int:
        return self.width * self.height

    def push(self, vec: np.ndarray) -> PushRecord:
        if self.state is None:  # jobs.py:189-194
            m = vec.size
            self.norm = Normalizer(np.zeros(m))
            self.state = core_init(m, self.prm, self.seed)
        nz = self.norm
        if not nz.frozen:  # jobs.py:201-209
            if self.state.frame_index < self.i_init:
                nz.fold(vec)
                x = (vec - nz.mean) / nz.running_std()
            else:
                nz.std = nz.running_std()
                nz.frozen = True
                x = (vec - nz.mean) / nz.std
        else:
            x = (vec - nz.mean) / nz.std
        t = step_at(self.state.frame_index, self.prm)
        self.state, res, ft = core_step(self.state, x, self.prm)
        raw = threshold(res, self.pixels, self.channels, self.prm.delta)
        if self.channels == 3:  # jobs.py:218-221, pipeline.py:231-242
            self.state.w = np.tile(np.where(raw != 0, self.prm.omega, 1.0), 3)
        return PushRecord(self.state.frame_index, majority3x3(raw, self.width, self.height),
                          raw, res, ft.cost, t, ft)

    def background(self) -> np.ndarray:
        """jobs.py:231-239."""
        bgn = self.state.U @ self.state.y
        return np.clip(bgn * self.norm.scale() + self.norm.mean, 0.0, 1.0)


def subspace_sine(A: np.ndarray, B: np.ndarray) -> float:
    """Sine of the largest principal angle (evaluate.py:207-218)."""
    off = B - A @ (A.T @ B)
    return float(np.linalg.svd(off, compute_uv=False)[0])


# --------------------------------------------------------------------------
# Resampling shell (pipeline.py:164-193, 245-258)


def resample_planes(data: np.ndarray, channels: int, width: int, height: int, out_w: int,
                    out_h: int) -> np.ndarray:
    """pipeline.py:164-193: bilinear per plane, half-pixel centres, clipped
    source coordinates; identity sizes return the data unchanged."""
    if (out_w, out_h) == (width, height):
        return data

    def axis(n_out, n_in):
        src = (np.arange(n_out) + 0.5) * (n_in / n_out) - 0.5
        src = np.clip(src, 0.0, n_in - 1.0)
        lo = np.floor(src).astype(int)
        return lo, np.minimum(lo + 1, n_in - 1), src - lo

    x0, x1, wx = axis(out_w, width)
    y0, y1, wy = axis(out_h, height)
    wx = wx[None, :]
    wy = wy[:, None]
    out = []
    for plane in data.reshape(channels, height, width):
        top = (1.0 - wx) * plane[np.ix_(y0, x0)] + wx * plane[np.ix_(y0, x1)]
        bottom = (1.0 - wx) * plane[np.ix_(y1, x0)] + wx * plane[np.ix_(y1, x1)]
        out.append(((1.0 - wy) * top + wy * bottom).reshape(-1))
    return np.concatenate(out)


def upsample_labels(labels: np.ndarray, width: int, height: int, out_w: int, out_h: int) -> np.ndarray:
    """pipeline.py:245-258: nearest neighbour on categorical labels."""
    if (out_w, out_h) == (width, height):
        return labels
    xs = np.minimum(((np.arange(out_w) + 0.5) * (width / out_w)).astype(int), width - 1)
    ys = np.minimum(((np.arange(out_h) + 0.5) * (height / out_h)).astype(int), height - 1)
    return labels.reshape(height, width)[np.ix_(ys, xs)].reshape(-1)
