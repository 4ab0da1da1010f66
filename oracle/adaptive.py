"""Adaptive explicit stepping for the oracle (TEST INFRASTRUCTURE ONLY --
imported by tests/, __graft_entry__.smoke() and bench.py's CPU legs, never by
the product).

Restates, per sample:
  * AdaptiveController (integrators.py:178-193),
  * the adaptive branch of integrate (integrators.py:294-349): WRMS error norm
    (:247-249), PI controller with exponents (0.7/p, -0.4/p), safety factor,
    clamp [0.2, 5], overflow -> rejection with h*0.2, FSAL carry of k_last on
    accept and of ks[0] on reject, StiffnessError on h underflow / max_steps,
  * the adaptive forward_pass (adjoint.py:162-186): one integrate per
    observation interval, boundary times = accepted t + h, observation states,
  * and the reverse sweep over the frozen per-sample grid (store_all /
    store_solutions; revolve is rejected as in checkpointing.py:218-220).
The batch result follows the batched conventions of core.grad_terminal:
loss and dtheta are sample means (seeds carry 1/B), du0 is per sample.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import core as oc
from .obs_losses import match_boundaries

EMBEDDED = {   # (b_emb, order) of the embedded tableaux (tableaux.py:84-118)
    "bosh3": ([7 / 24, 1 / 4, 1 / 3, 1 / 8], 3),
    "dopri5": ([5179 / 57600, 0, 7571 / 16695, 393 / 640, -92097 / 339200, 187 / 2100, 1 / 40], 5),
}


class StiffnessError(oc.IntegrationError):
    pass


@dataclass(frozen=True)
class AdaptiveCtrl:
    abstol: float = 1e-6
    reltol: float = 1e-6
    h_init: float = 1e-3
    h_min: float = 1e-14
    h_max: float = np.inf
    safety: float = 0.9
    max_steps: int = 1_000_000


def wrms(err, u_old, u_new, ctrl):
    """integrators.py:247-249."""
    scale = ctrl.abstol + ctrl.reltol * np.maximum(np.abs(u_old), np.abs(u_new))
    return float(np.sqrt(np.mean((err / scale) ** 2)))


class _Row:
    """One sample of a batched oracle field."""

    def __init__(self, fld, b):
        self.fld, self.b = fld, b

    def eval(self, u, t, c):
        return self.fld.eval(u[None, :], t, c)[0]


def _step(tab, sf, u, t, h, c, k_first):
    """explicit_rk_step returning the stage derivatives too."""
    s = tab.stages
    stages, ks = [], []
    for i in range(s):
        ui = u.copy()
        for j in range(i):
            if tab.a[i, j] != 0.0:
                ui = ui + (h * tab.a[i, j]) * ks[j]
        stages.append(ui)
        if i == 0 and k_first is not None:
            ks.append(k_first)
        else:
            ks.append(sf.eval(ui, t + tab.c[i] * h, c))
    un = u.copy()
    for i in range(s):
        if tab.b[i] != 0.0:
            un = un + (h * tab.b[i]) * ks[i]
    if not np.all(np.isfinite(un)):
        raise oc.IntegrationError(f"state overflowed at t={t} (h={h})")
    return oc.Record(-1, t, h, u, stages, un), (ks[-1] if tab.fsal else None), ks


def integrate_adaptive(tab, name, sf, u, t0, tF, ctrl, c, emit, stats):
    """integrators.py:294-349 for one sample; emit(rec) per accepted step."""
    b_emb, p = EMBEDDED[name]
    alpha, beta = 0.7 / p, 0.4 / p
    h = min(ctrl.h_init, tF - t0)
    t = t0
    err_prev = 1.0
    k_carry = None
    taken = 0
    while t < tF - 1e-14 * max(1.0, abs(tF)):
        if taken >= ctrl.max_steps:
            raise StiffnessError(f"adaptive integration exceeded {ctrl.max_steps} steps at t={t}")
        h = min(h, tF - t)
        try:
            rec, k_last, ks = _step(tab, sf, u, t, h, c, k_carry)
        except oc.IntegrationError:
            stats["rejected"] += 1
            k_carry = None
            if h <= ctrl.h_min * (1 + 1e-12):
                raise StiffnessError(f"step size underflow at t={t}: stiffness suspected")
            h = max(h * 0.2, ctrl.h_min)
            taken += 1
            continue
        err = np.zeros_like(u)
        for i in range(tab.stages):
            d = tab.b[i] - b_emb[i]
            if d != 0.0:
                err = err + (h * d) * ks[i]
        enorm = max(wrms(err, u, rec.u_next, ctrl), 1e-10)
        taken += 1
        if enorm <= 1.0:
            u = rec.u_next
            t = t + h
            emit(rec)
            k_carry = k_last
            factor = ctrl.safety * enorm ** (-alpha) * err_prev ** beta
            err_prev = enorm
        else:
            stats["rejected"] += 1
            k_carry = ks[0]
            if h <= ctrl.h_min * (1 + 1e-12):
                raise StiffnessError(f"step size underflow at t={t}: stiffness suspected")
            factor = min(ctrl.safety * enorm ** (-alpha), 1.0)
        factor = min(5.0, max(0.2, factor))
        h = min(max(h * factor, ctrl.h_min), ctrl.h_max)
    return u


def forward_adaptive(tab, name, sf, u0, t0, tF, ctrl, obs_times, c, stats):
    """adjoint.py:162-186: per observation interval; returns (records, boundary
    times, observation states, u_final)."""
    recs = []
    bt = [t0]

    def emit(rec):
        rec.n = len(recs)
        recs.append(rec)
        bt.append(rec.t + rec.h)

    pts = [t0] + [tk for tk in obs_times if tk > t0]
    if abs(pts[-1] - tF) > 1e-12 * max(1.0, abs(tF)):
        pts.append(tF)
    u = u0
    obs_states = [u0.copy()] if obs_times and obs_times[0] == t0 else []
    for a, b in zip(pts, pts[1:]):
        u = integrate_adaptive(tab, name, sf, u, a, b, ctrl, c, emit, stats)
        if any(abs(b - tk) <= 1e-9 * max(1.0, abs(tk)) for tk in obs_times):
            obs_states.append(u.copy())
    return recs, bt, obs_states, u


def grad_adaptive(fld, scheme_name, U0, t0, tF, ctrl: AdaptiveCtrl, policy="store_all",
                  obs=None, obs_times=None):
    """Batched adaptive grad.  obs: an obs_losses.ObsLoss whose ``steps`` are
    ignored (observation times come from ``obs_times``); without obs the loss
    is the BASELINE 0.5 mean ||u(tF)||^2."""
    if policy.startswith("revolve"):
        raise ValueError("revolve checkpointing needs fixed stepping")
    if scheme_name not in EMBEDDED:
        raise oc.IntegrationError("adaptive mode needs an embedded explicit scheme")
    tab = oc.explicit_tableau(scheme_name)
    U0 = np.asarray(U0, dtype=np.float64)
    B = U0.shape[0]
    times = tuple(obs_times) if obs is not None else (tF,)
    out = {"u_final": np.empty_like(U0), "du0": np.empty_like(U0), "dtheta": np.zeros(fld.n_params),
           "loss": 0.0, "grids": [], "accepted": [], "rejected": [], "nfe_forward": [],
           "nfe_backward": [], "steps_recomputed": [], "predictions": None}
    preds_all = []
    for b in range(B):
        c = oc.Counters()
        stats = {"rejected": 0}
        sf = oc.SampleField(fld)
        recs, bt, obs_states, uf = forward_adaptive(tab, scheme_name, sf, U0[b], t0, tF, ctrl,
                                                    times, c, stats)
        out["u_final"][b] = uf
        inj = {}
        if obs is not None:
            preds = np.stack(obs_states)[:, None, :]
            vals = obs.values[:, b:b + 1, :]
            o1 = type(obs)(obs.kind, range(len(times)), vals, obs.scaling)
            loss_b, seeds = o1.loss_and_seeds(preds, batch_global=B)
            preds_all.append(preds[:, 0])
            for j, sd in zip(match_boundaries(times, bt), seeds):
                inj[j] = inj.get(j, 0.0) + sd[0]
            lam = np.zeros_like(uf)
        else:
            loss_b = 0.5 * float(uf @ uf) / B
            lam = uf / B
        out["loss"] += loss_b
        mu = np.zeros(fld.n_params)
        n = len(recs)
        recomputed = 0
        for m in range(n - 1, -1, -1):
            rec = recs[m]
            if policy == "store_solutions" and m < n - 1:     # replay from u_m (integrators.py:352-368)
                rec, _, _ = _step(tab, sf, rec.u, rec.t, rec.h, c, None)
                rec.n = m
                recomputed += 1
            if m + 1 in inj:
                lam = lam + inj[m + 1]
            l2, mu = oc.rk_adjoint_step(tab, fld, oc.Record(m, rec.t, rec.h, rec.u[None],
                                                           [s_[None] for s_ in rec.stages],
                                                           rec.u_next[None]), lam[None], mu, c)
            lam = l2[0]
        if 0 in inj:
            lam = lam + inj[0]
        out["du0"][b] = lam
        out["dtheta"] += mu
        out["grids"].append(np.array(bt))
        out["accepted"].append(n)
        out["rejected"].append(stats["rejected"])
        out["nfe_forward"].append(c.nfe_forward)
        out["nfe_backward"].append(c.nfe_backward)
        out["steps_recomputed"].append(recomputed)
    if obs is not None:
        out["predictions"] = np.stack(preds_all, axis=1)     # [K, B, N]
    return out
