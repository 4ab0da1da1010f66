"""Controllers, counters, solver configuration and the error classes of the
reference API (integrators.py:20-50, :157-193; linalg.py:14-34;
adjoint.py:33-34; checkpointing.py:173-198), re-exported unchanged in
meaning so reference callers keep their ``except`` clauses.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib


class IntegrationError(RuntimeError):
    pass


class StiffnessError(IntegrationError):
    """Adaptive step size underflow (adaptive stepping is not built: SURVEY 8f)."""


class ConvergenceError(RuntimeError):
    def __init__(self, message, residual=None):
        super().__init__(message)
        self.residual = residual


class GradientExplosionError(RuntimeError):
    """Adjoint state became non-finite during the reverse sweep."""


class DeviceError(RuntimeError):
    """CUDA failure inside the native library."""


def raise_status(code: int, msg: str):
    if code == _lib.OB_OK:
        return
    if code == _lib.OB_ERR_VALUE:
        raise ValueError(msg)
    if code == _lib.OB_ERR_INTEGRATION:
        raise IntegrationError(msg)
    if code == _lib.OB_ERR_STIFFNESS:
        raise StiffnessError(msg)
    if code == _lib.OB_ERR_CONVERGENCE:
        # theta_step wraps solver failures (integrators.py:239-242)
        raise IntegrationError(f"implicit step failed: {msg}") from ConvergenceError(msg)
    if code == _lib.OB_ERR_GRADIENT_EXPLOSION:
        raise GradientExplosionError(msg)
    if code == _lib.OB_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise DeviceError(msg)


@dataclass
class NfeCounters:
    nfe_forward: int = 0
    nfe_backward: int = 0
    steps_accepted: int = 0
    steps_rejected: int = 0
    steps_recomputed: int = 0

    def as_dict(self):
        return {k: getattr(self, k) for k in ("nfe_forward", "nfe_backward", "steps_accepted",
                                              "steps_rejected", "steps_recomputed")}

    def add(self, other: "NfeCounters"):
        for k in self.as_dict():
            setattr(self, k, getattr(self, k) + getattr(other, k))


@dataclass
class StoreCounters:
    stored_states: int = 0
    stored_stage_vectors: int = 0
    max_live_slots: int = 0
    recomputed_steps: int = 0


@dataclass(frozen=True)
class FixedController:
    n_steps: int

    def __post_init__(self):
        if self.n_steps < 1:
            raise ValueError("fixed mode requires at least one step")


@dataclass(frozen=True)
class FixedGridController:
    """Fixed stepping through an explicit ascending array of times."""

    times: tuple

    def __post_init__(self):
        ts = tuple(float(t) for t in self.times)
        object.__setattr__(self, "times", ts)
        if len(ts) < 2 or any(b <= a for a, b in zip(ts, ts[1:])):
            raise ValueError("times must be strictly increasing, length >= 2")


@dataclass(frozen=True)
class AdaptiveController:
    """Error-controlled stepping with an embedded pair (integrators.py:178-193):
    WRMS norm, PI controller, per-sample step sizes.  ``max_accepted`` is this
    build's per-sample capacity of accepted steps (device record storage);
    exceeding it raises NotImplementedError naming the sample."""

    abstol: float = 1e-6
    reltol: float = 1e-6
    h_init: float = 1e-3
    h_min: float = 1e-14
    h_max: float = np.inf
    safety: float = 0.9
    max_steps: int = 1_000_000
    max_accepted: int = 1000

    def __post_init__(self):
        if self.abstol <= 0 or self.reltol <= 0:
            raise ValueError("tolerances must be positive")
        if not (self.h_min <= self.h_init <= self.h_max):
            raise ValueError("need h_min <= h_init <= h_max")
        if self.max_accepted < 1:
            raise ValueError("max_accepted must be >= 1")


def boundary_times(ctrl, t0, tF) -> np.ndarray:
    """The fp64 step grid (integrators.py:274-280): np.linspace for a fixed
    step count, the explicit grid (checked to span [t0, tF]) otherwise."""
    if tF <= t0:
        raise ValueError("tF must exceed t0")
    if isinstance(ctrl, FixedController):
        return np.linspace(t0, tF, ctrl.n_steps + 1)
    if isinstance(ctrl, FixedGridController):
        ts = np.asarray(ctrl.times, dtype=np.float64)
        if abs(ts[0] - t0) > 1e-12 * max(1.0, abs(t0)) or abs(ts[-1] - tF) > 1e-12 * max(1.0, abs(tF)):
            raise ValueError("time grid must span [t0, tF]")
        return ts
    raise TypeError(f"unknown controller {ctrl!r}")


@dataclass(frozen=True)
class SolverConfig:
    newton_tol: float = 1e-10
    newton_maxit: int = 50
    gmres_tol: float = 1e-12
    gmres_maxit: int = 200
    gmres_restart: int = 30

    def __post_init__(self):
        if not (0.0 < self.newton_tol < 1.0 and 0.0 < self.gmres_tol < 1.0):
            raise ValueError("tolerances must lie in (0, 1)")
        if min(self.newton_maxit, self.gmres_maxit, self.gmres_restart) < 1:
            raise ValueError("iteration caps must be >= 1")

    def to_desc(self) -> _lib.SolverDesc:
        d = _lib.SolverDesc()
        d.newton_tol = self.newton_tol
        d.gmres_tol = self.gmres_tol
        d.newton_maxit = self.newton_maxit
        d.gmres_maxit = self.gmres_maxit
        d.gmres_restart = self.gmres_restart
        return d
