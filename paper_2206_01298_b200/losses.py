"""Losses (reference LossSpec / MinMaxScaling / terminal_loss, losses.py:10-107).

Batched semantics: the loss is the mean over samples of the reference's
per-sample loss, so every seed carries an extra 1/B.
  * ``mse`` / ``mae``: the reference's observation losses -- the mean over K
    observation times and N components of r^2 / |r|, r = scale(u(t_k)) - y_k,
    with optional min-max scaling (losses.py:40-107).  ``values`` holds one
    observation per time, each [B, N] (or [N], shared by every sample); a single
    array with one time is accepted as the K=1 terminal case.  Observation
    times must land on step boundaries (adjoint.py:213-221); seeds are injected
    into the adjoint at those boundaries (adjoint.py:235-253).
  * ``half_sqnorm``: ell(u) = 0.5 ||u(tF)||^2 (the BASELINE configs' loss).
  * ``ce_head``: for ConvField states: global-average-pool + linear 64 -> 10
    + softmax cross-entropy; values = (head params [10*64 + 10], labels [B]);
    the head gradient comes back as GradResult.dtheta_head.
  * ``cnf_nll``: for CnfField states [z, Delta]: -log p(x) = 0.5||z||^2 +
    D/2 log(2 pi) + Delta (standard-normal base, log p(x) = log N(z(1)) - Delta(1)).
The last three are terminal (one time, tF).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

KINDS = ("half_sqnorm", "mse", "mae", "cnf_nll", "ce_head")
OBSERVATION_KINDS = ("mse", "mae")


@dataclass(frozen=True)
class MinMaxScaling:
    """Per-component affine map u' = (u - lo) / (hi - lo); components with
    hi <= lo pass through unchanged (losses.py:10-37)."""

    lo: np.ndarray
    hi: np.ndarray

    def __post_init__(self):
        lo = np.asarray(self.lo, dtype=np.float64)
        hi = np.asarray(self.hi, dtype=np.float64)
        if lo.shape != hi.shape or lo.ndim != 1:
            raise ValueError("lo and hi must be vectors of one length")
        object.__setattr__(self, "lo", lo)
        object.__setattr__(self, "hi", hi)

    @property
    def degenerate(self) -> np.ndarray:
        return self.hi <= self.lo

    @property
    def span(self) -> np.ndarray:
        return np.where(self.degenerate, 1.0, self.hi - self.lo)

    def apply(self, u):
        return np.where(self.degenerate, u, (u - self.lo) / self.span)

    def invert(self, v):
        return np.where(self.degenerate, v, v * self.span + self.lo)

    def chain(self, seed_scaled):
        return np.where(self.degenerate, seed_scaled, seed_scaled / self.span)


@dataclass(frozen=True)
class LossSpec:
    kind: str
    times: tuple
    values: object = None
    scaling: MinMaxScaling = None

    def __post_init__(self):
        if self.kind not in KINDS:
            raise ValueError(f"unknown loss kind {self.kind!r}")
        ts = tuple(float(t) for t in self.times)
        if not ts:
            raise ValueError("need one observation vector per time")
        if any(b <= a for a, b in zip(ts, ts[1:])):
            raise ValueError("observation times must be strictly increasing")
        object.__setattr__(self, "times", ts)
        if self.kind in OBSERVATION_KINDS:
            vals = self.values
            if vals is None:
                raise ValueError(f"{self.kind} needs observed values")
            if not isinstance(vals, (tuple, list)):
                vals = (vals,)
            if len(vals) != len(ts):
                raise ValueError("need one observation vector per time")
            shapes = {tuple(v.shape) for v in vals}
            if len(shapes) != 1:
                raise ValueError("all observations must share the state dimension")
            object.__setattr__(self, "values", tuple(vals))
        else:
            if len(ts) != 1:
                raise ValueError(f"{self.kind} is a terminal loss (one time)")
            if self.scaling is not None:
                raise ValueError(f"{self.kind} takes no scaling")
            if self.kind == "ce_head" and (self.values is None or len(self.values) != 2):
                raise ValueError("ce_head needs (head parameters, labels)")

    @property
    def n_obs(self) -> int:
        return len(self.times)


def terminal_loss(kind, t_final, observed=None, scaling=None) -> LossSpec:
    return LossSpec(kind, (t_final,), observed, scaling)


def match_boundaries(times, boundary_times):
    """Boundary index of each observation time (adjoint.py:213-221)."""
    bt = np.asarray(boundary_times, dtype=np.float64)
    idx = []
    for tk in times:
        j = int(np.argmin(np.abs(bt - tk)))
        if abs(bt[j] - tk) > 1e-9 * max(1.0, abs(tk)):
            raise ValueError(f"time {tk} does not align with a step boundary")
        idx.append(j)
    return idx
