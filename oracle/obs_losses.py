"""Observation losses for the oracle (TEST INFRASTRUCTURE ONLY -- imported by
tests/, __graft_entry__.smoke() and bench.py's CPU legs, never by the product).

Batched restatement of the reference's LossSpec / MinMaxScaling /
loss_and_grad_seed (odegrad/losses.py:10-107) and _match_boundaries
(adjoint.py:213-221).  Per sample the loss is the mean over the K observations
and N components of |r| (mae) or r^2 (mse), r = scale(pred) - obs; the batch
loss is the mean over samples, so every seed carries an extra 1/B.
"""

from __future__ import annotations

import numpy as np


class MinMax:
    """u' = (u - lo) / (hi - lo); components with hi <= lo pass through (losses.py:10-37)."""

    def __init__(self, lo, hi):
        self.lo = np.asarray(lo, dtype=np.float64)
        self.hi = np.asarray(hi, dtype=np.float64)
        self.degenerate = self.hi <= self.lo
        self.span = np.where(self.degenerate, 1.0, self.hi - self.lo)

    def apply(self, u):
        return np.where(self.degenerate, u, (u - self.lo) / self.span)

    def chain(self, s):
        return np.where(self.degenerate, s, s / self.span)


def match_boundaries(times, boundary_times):
    """Boundary index of each observation time, 1e-9 relative tolerance (adjoint.py:213-221)."""
    bt = np.asarray(boundary_times, dtype=np.float64)
    out = []
    for tk in times:
        j = int(np.argmin(np.abs(bt - tk)))
        if abs(bt[j] - tk) > 1e-9 * max(1.0, abs(tk)):
            raise ValueError(f"time {tk} does not align with a step boundary")
        out.append(j)
    return out


class ObsLoss:
    """kind in {mae, mse}; steps: boundary indices (strictly increasing);
    values: [K, B, N] observations; scaling: MinMax or None."""

    def __init__(self, kind, steps, values, scaling=None):
        if kind not in ("mae", "mse"):
            raise ValueError(kind)
        self.kind = kind
        self.steps = list(steps)
        self.values = np.asarray(values, dtype=np.float64)
        self.scaling = scaling

    def loss_and_seeds(self, preds, batch_global=None):
        """preds: [K, B, N] -> (batch-mean loss, seeds [K, B, N])  (losses.py:78-107)."""
        preds = np.asarray(preds, dtype=np.float64)
        K, B, N = preds.shape
        Bg = batch_global or B
        denom = float(K * N)
        total = 0.0
        seeds = np.empty_like(preds)
        for k in range(K):
            pc = self.scaling.apply(preds[k]) if self.scaling is not None else preds[k]
            r = pc - self.values[k]
            if self.kind == "mae":
                total += float(np.sum(np.abs(r)))
                s = np.sign(r) / denom
            else:
                total += float(np.sum(r * r))
                s = 2.0 * r / denom
            if self.scaling is not None:
                s = self.scaling.chain(s)
            seeds[k] = s / Bg
        return total / denom / Bg, seeds
