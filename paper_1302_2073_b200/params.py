"""Tracker parameters, mirroring the reference's configuration types.

`LpConfig` (cost.py:29-45), `CgOptions` (fit.py:24-47), `ProstParams`
(tracker.py:45-76), `RunConfig` (jobs.py:74-139) and the schedule helpers
`tau_from_init` / `step_size` (tracker.py:90-103) and
`smoothing_from_threshold` (cost.py:115-127): same names, defaults, argument
meaning and validation errors.  These are host-side scalars; they are packed
into the C-ABI's `prost_params` by `to_native`.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional

from .errors import ConfigError

__all__ = [
    "LpConfig",
    "CgOptions",
    "ProstParams",
    "RunConfig",
    "DEFAULT_I_INIT",
    "tau_from_init",
    "step_size",
    "smoothing_from_threshold",
]

DEFAULT_I_INIT = 100  # jobs.py:71


@dataclass(frozen=True)
class LpConfig:
    """Exponent p in (0, 2] and smoothing offset mu > 0 (cost.py:29-45)."""

    p: float
    mu: float

    def __post_init__(self):
        if not (0.0 < self.p <= 2.0):
            raise ConfigError(f"p must be in (0, 2], got {self.p}")
        if not self.mu > 0.0:
            raise ConfigError(f"mu must be > 0, got {self.mu}")


@dataclass(frozen=True)
class CgOptions:
    """Budget and line-search knobs of the coordinate solver (fit.py:24-47)."""

    max_iters: int = 5
    grad_tol: float = 1e-8
    initial_step: float = 1.0
    shrink: float = 0.5
    sufficient_decrease: float = 1e-4
    max_backtracks: int = 20

    def __post_init__(self):
        if self.max_iters < 1:
            raise ConfigError(f"max_iters must be >= 1, got {self.max_iters}")
        if self.grad_tol < 0.0:
            raise ConfigError(f"grad_tol must be >= 0, got {self.grad_tol}")
        if not (0.0 < self.shrink < 1.0):
            raise ConfigError(f"shrink must be in (0, 1), got {self.shrink}")
        if not (0.0 < self.sufficient_decrease <= 0.5):
            raise ConfigError(
                f"sufficient_decrease must be in (0, 0.5], got {self.sufficient_decrease}"
            )
        if self.max_backtracks < 1:
            raise ConfigError(f"max_backtracks must be >= 1, got {self.max_backtracks}")


@dataclass(frozen=True)
class ProstParams:
    """All tracker tunables (tracker.py:45-76)."""

    k: int
    cfg: LpConfig
    delta: float
    omega: float = 1.0
    t_init: float = 5e-3
    t_min: float = 1e-4
    tau: float = 0.0
    cg: CgOptions = field(default_factory=CgOptions)

    def __post_init__(self):
        if self.k < 1:
            raise ConfigError(f"subspace dimension must be >= 1, got {self.k}")
        if not self.delta > 0.0:
            raise ConfigError(f"delta must be > 0, got {self.delta}")
        if not (0.0 < self.omega <= 1.0):
            raise ConfigError(f"omega must be in (0, 1], got {self.omega}")
        if not (0.0 < self.t_min <= self.t_init):
            raise ConfigError(
                f"need 0 < t_min <= t_init, got t_min={self.t_min}, t_init={self.t_init}"
            )
        if self.tau < 0.0:
            raise ConfigError(f"tau must be >= 0, got {self.tau}")


def tau_from_init(t_init: float, t_min: float, i_init: int) -> float:
    """Decay rate bringing the step from t_init to t_min in i_init frames (tracker.py:90-96)."""
    if not (0.0 < t_min <= t_init):
        raise ConfigError(f"need 0 < t_min <= t_init, got t_min={t_min}, t_init={t_init}")
    if i_init < 1:
        raise ConfigError(f"i_init must be >= 1, got {i_init}")
    return -float(math.log(t_min / t_init)) / i_init


def step_size(i: int, params: ProstParams) -> float:
    """max(e^(-tau i) t_init, t_min) (tracker.py:99-103)."""
    if i < 0:
        raise ConfigError(f"frame index must be >= 0, got {i}")
    return max(float(math.exp(-params.tau * i)) * params.t_init, params.t_min)


def smoothing_from_threshold(delta: float, p: float) -> float:
    """mu = delta^2 (1 - p) (cost.py:115-127)."""
    if not (0.0 < p < 1.0):
        raise ConfigError(f"threshold coupling requires 0 < p < 1, got p={p}")
    if not delta > 0.0:
        raise ConfigError(f"delta must be > 0, got {delta}")
    return delta * delta * (1.0 - p)


@dataclass(frozen=True)
class RunConfig:
    """Fully-resolved pipeline configuration (jobs.py:74-139); same defaults."""

    subspace_dim: int = 15
    p: float = 0.25
    mu: Optional[float] = None
    delta: float = 0.35
    omega: float = 5e-5
    t_init: float = 5e-3
    t_min: float = 1e-4
    i_init: Optional[int] = None
    tau: Optional[float] = None
    cg_max_iters: int = 5
    target_width: int = 160
    target_height: int = 120
    grayscale: bool = False
    seed: int = 0

    def resolved_mu(self) -> float:
        if self.mu is not None:
            return self.mu
        if self.p < 1.0:
            return smoothing_from_threshold(self.delta, self.p)
        return 1e-3

    def params(self, i_init: int) -> ProstParams:
        tau = self.tau if self.tau is not None else tau_from_init(self.t_init, self.t_min, i_init)
        return ProstParams(
            k=self.subspace_dim,
            cfg=LpConfig(p=self.p, mu=self.resolved_mu()),
            delta=self.delta,
            omega=self.omega,
            t_init=self.t_init,
            t_min=self.t_min,
            tau=tau,
            cg=CgOptions(max_iters=self.cg_max_iters),
        )

    def echo(self, i_init: int) -> dict:
        return {
            "subspace_dim": self.subspace_dim,
            "p": self.p,
            "mu": self.resolved_mu(),
            "delta": self.delta,
            "omega": self.omega,
            "t_init": self.t_init,
            "t_min": self.t_min,
            "i_init": i_init,
            "tau": self.params(i_init).tau,
            "cg_max_iters": self.cg_max_iters,
            "target_width": self.target_width,
            "target_height": self.target_height,
            "grayscale": self.grayscale,
            "seed": self.seed,
        }


def to_native(params: ProstParams, width: int, height: int, channels: int, i_init: int):
    """Pack into the C-ABI `prost_params` struct."""
    from ._native import Params

    return Params(
        k=params.k, width=width, height=height, channels=channels,
        cg_max_iters=params.cg.max_iters, max_backtracks=params.cg.max_backtracks,
        i_init=i_init, reserved=0, p=params.cfg.p, mu=params.cfg.mu, delta=params.delta,
        omega=params.omega, t_init=params.t_init, t_min=params.t_min, tau=params.tau,
        grad_tol=params.cg.grad_tol, initial_step=params.cg.initial_step,
        shrink=params.cg.shrink, sufficient_decrease=params.cg.sufficient_decrease,
    )
