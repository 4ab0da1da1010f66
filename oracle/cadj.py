"""Continuous-adjoint baseline for the oracle (TEST INFRASTRUCTURE ONLY --
imported by tests/, never by the product): restates _AugmentedReverseField and
continuous_adjoint_solve (adjoint.py:294-331) per sample with the oracle's
explicit step (FSAL carry included, integrators.py:274-292)."""

import numpy as np

from . import core as oc


class _Aug:
    """y = (u, lam, mu); d/dtau = (-f, J^T lam, P^T lam) at t = tF - tau."""

    def __init__(self, fld, n, t_f):
        self.fld, self.n, self.t_f = fld, n, t_f

    def eval(self, y, tau, c):
        t = self.t_f - tau
        u, lam = y[: self.n], y[self.n: 2 * self.n]
        jtv, ptv = self.fld.vjp(u[None], t, lam[None], c)
        f = self.fld.eval(u[None], t, c)[0]
        return np.concatenate([-f, jtv[0], ptv])


def continuous_adjoint_solve(fld, scheme_name, dphi_du, u_final, t0, tF, n_steps):
    """Batched: per-sample lam0 [B, N], mu0 summed over samples."""
    tab = oc.explicit_tableau(scheme_name)
    U = np.asarray(u_final, dtype=np.float64)
    D = np.asarray(dphi_du, dtype=np.float64)
    B, n = U.shape
    lam0 = np.empty_like(U)
    mu0 = np.zeros(fld.n_params)
    ts = np.linspace(0.0, tF - t0, n_steps + 1)
    for b in range(B):
        aug = _Aug(fld, n, tF)
        y = np.concatenate([U[b], D[b], np.zeros(fld.n_params)])
        c = oc.Counters()
        k = None
        for i in range(n_steps):
            rec, k = oc.rk_step(tab, aug, y, ts[i], ts[i + 1] - ts[i], c, k_first=k)
            y = rec.u_next
        lam0[b] = y[n: 2 * n]
        mu0 += y[2 * n:]
    return lam0, mu0
