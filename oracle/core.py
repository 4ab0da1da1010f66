"""TEST INFRASTRUCTURE ONLY -- float64 CPU restatement of the reference
discrete-adjoint gradient path, batched over independent samples (rows).

Every function cites the reference file:line it restates (paths relative to
``/root/reference/pkg/src/odegrad``).  Batching changes no per-sample
arithmetic except BLAS blocking inside the affine layers (GEMM over rows vs the
reference's per-sample GEMV) and the order of the batch sum of the parameter
cotangent; both are rounding-level (<= 1e-14 relative, pinned by
``tests/test_oracle_golden.py`` against reference-generated fixtures).

Implicit (theta) steps run Newton + GMRES *per sample*, exactly like the
reference, because their iteration counts are data dependent.
"""

from __future__ import annotations

from dataclasses import dataclass, field as dc_field

import numpy as np

try:
    from scipy.special import erf as _erf
except ImportError:  # pragma: no cover
    import math
    _erf = np.vectorize(math.erf)

from .revolve import revolve_schedule

# ---------------------------------------------------------------------------
# errors (integrators.py:20-25, linalg.py:14-19, adjoint.py:33-34)


class IntegrationError(RuntimeError):
    pass


class ConvergenceError(RuntimeError):
    def __init__(self, message, residual=None):
        super().__init__(message)
        self.residual = residual


class GradientExplosionError(RuntimeError):
    pass


# ---------------------------------------------------------------------------
# tableaux (tableaux.py:95-140) -- literature-standard coefficients


@dataclass(frozen=True)
class Tableau:
    name: str
    a: np.ndarray
    b: np.ndarray
    c: np.ndarray
    fsal: bool

    @property
    def stages(self):
        return len(self.b)


def _t(name, a, b, c, fsal=False):
    return Tableau(name, np.asarray(a, float), np.asarray(b, float), np.asarray(c, float), fsal)


def explicit_tableau(name):
    if name == "euler":
        return _t(name, [[0.0]], [1.0], [0.0])
    if name == "midpoint":
        return _t(name, [[0, 0], [0.5, 0]], [0.0, 1.0], [0.0, 0.5])
    if name == "bosh3":
        return _t(name, [[0, 0, 0, 0], [1 / 2, 0, 0, 0], [0, 3 / 4, 0, 0], [2 / 9, 1 / 3, 4 / 9, 0]],
                  [2 / 9, 1 / 3, 4 / 9, 0.0], [0, 1 / 2, 3 / 4, 1.0], fsal=True)
    if name == "rk4":
        return _t(name, [[0, 0, 0, 0], [0.5, 0, 0, 0], [0, 0.5, 0, 0], [0, 0, 1.0, 0]],
                  [1 / 6, 1 / 3, 1 / 3, 1 / 6], [0.0, 0.5, 0.5, 1.0])
    if name == "dopri5":
        row7 = [35 / 384, 0, 500 / 1113, 125 / 192, -2187 / 6784, 11 / 84, 0]
        a = [[0] * 7,
             [1 / 5, 0, 0, 0, 0, 0, 0],
             [3 / 40, 9 / 40, 0, 0, 0, 0, 0],
             [44 / 45, -56 / 15, 32 / 9, 0, 0, 0, 0],
             [19372 / 6561, -25360 / 2187, 64448 / 6561, -212 / 729, 0, 0, 0],
             [9017 / 3168, -355 / 33, 46732 / 5247, 49 / 176, -5103 / 18656, 0, 0],
             row7]
        return _t(name, a, row7, [0, 1 / 5, 3 / 10, 4 / 5, 8 / 9, 1, 1], fsal=True)
    raise ValueError(name)


THETA_SCHEMES = {"beuler": 1.0, "cn": 0.5}


# ---------------------------------------------------------------------------
# counters (integrators.py:28-50)


@dataclass
class Counters:
    nfe_forward: int = 0
    nfe_backward: int = 0
    steps_accepted: int = 0
    steps_recomputed: int = 0


@dataclass
class StoreCounters:
    stored_states: int = 0
    stored_stage_vectors: int = 0
    max_live_slots: int = 0
    recomputed_steps: int = 0


# ---------------------------------------------------------------------------
# activations (kernels.py:45-77 / numpy path :97-115); softplus is new (C4)

_S12 = 1.0 / np.sqrt(2.0)
_ISQ2PI = 1.0 / np.sqrt(2.0 * np.pi)


def act(z, name):
    if name == "identity":
        return z.copy()
    if name == "relu":
        return np.maximum(z, 0.0)
    if name == "tanh":
        return np.tanh(z)
    if name == "gelu":
        return 0.5 * z * (1.0 + _erf(z * _S12))
    if name == "softplus":
        return np.maximum(z, 0.0) + np.log1p(np.exp(-np.abs(z)))
    raise ValueError(name)


def act_prime(z, name):
    if name == "identity":
        return np.ones_like(z)
    if name == "relu":
        return (z > 0.0).astype(np.float64)          # ReLU'(0) = 0 (kernels.py:68-70)
    if name == "tanh":
        t = np.tanh(z)
        return 1.0 - t * t
    if name == "gelu":
        return 0.5 * (1.0 + _erf(z * _S12)) + z * _ISQ2PI * np.exp(-0.5 * z * z)
    if name == "softplus":
        return 1.0 / (1.0 + np.exp(-z))
    raise ValueError(name)


def act_second(z, name):
    """Second derivative (needed by the CNF Hutchinson VJP only)."""
    if name == "softplus":
        s = 1.0 / (1.0 + np.exp(-z))
        return s * (1.0 - s)
    if name == "tanh":
        t = np.tanh(z)
        return -2.0 * t * (1.0 - t * t)
    if name in ("identity", "relu"):
        return np.zeros_like(z)
    raise ValueError(name)


# ---------------------------------------------------------------------------
# MLP kernels, batched over rows (kernels.py:122-225; nn.py:126-183)


class Mlp:
    """Flat-theta MLP: per layer W row-major [out, in] then b (kernels.py:9-16)."""

    def __init__(self, widths, activation, theta, time_input=False):
        self.widths = tuple(int(w) for w in widths)
        self.activation = activation
        self.time_input = bool(time_input)
        self.theta = np.asarray(theta, dtype=np.float64)
        self.layers = []
        off = 0
        for l in range(len(self.widths) - 1):
            nin, nout = self.widths[l], self.widths[l + 1]
            self.layers.append((off, off + nout * nin, nin, nout))
            off += nout * nin + nout
        self.n_params = off
        assert self.theta.shape == (off,), (self.theta.shape, off)

    def W(self, l):
        o, ob, nin, nout = self.layers[l]
        return self.theta[o:ob].reshape(nout, nin)

    def b(self, l):
        o, ob, nin, nout = self.layers[l]
        return self.theta[ob:ob + nout]

    def input(self, U, t):
        # time appended last (nn.py:126-129)
        if self.time_input:
            return np.concatenate([U, np.full((U.shape[0], 1), float(t))], axis=1)
        return U

    def forward(self, X):
        """(out, acts, pre) like mlp_forward_kernel (kernels.py:122-152)."""
        acts, pre = [], []
        a = X
        L = len(self.layers)
        for l in range(L):
            acts.append(a)
            if a.shape[0] == 1:     # per-sample call: the reference's GEMV (kernels.py:143)
                z = (np.dot(self.W(l), a[0]) + self.b(l))[None, :]
            else:
                z = a @ self.W(l).T + self.b(l)
            pre.append(z)
            a = act(z, self.activation) if l < L - 1 else z
        return a, acts, pre

    def vjp(self, acts, pre, V, want_theta=True):
        """(d_input, dtheta summed over rows) like mlp_vjp_kernel (kernels.py:155-183)."""
        L = len(self.layers)
        dth = np.zeros(self.n_params) if want_theta else None
        d = V
        for l in range(L - 1, -1, -1):
            o, ob, nin, nout = self.layers[l]
            if l < L - 1:
                d = d * act_prime(pre[l], self.activation)
            if want_theta:
                if d.shape[0] == 1:
                    dth[o:ob] = np.outer(d[0], acts[l][0]).ravel()
                else:
                    dth[o:ob] = (d.T @ acts[l]).ravel()
                dth[ob:ob + nout] = d.sum(axis=0)
            d = np.dot(d[0], self.W(l))[None, :] if d.shape[0] == 1 else d @ self.W(l)
        return d, dth

    def jvp(self, pre, S0):
        """(df/dx) s through the cached linearization (kernels.py:209-225)."""
        s = S0
        L = len(self.layers)
        for l in range(L):
            s = np.dot(self.W(l), s[0])[None, :] if s.shape[0] == 1 else s @ self.W(l).T
            if l < L - 1:
                s = s * act_prime(pre[l], self.activation)
        return s


class MlpField:
    """Batched ``MlpField`` (integrators.py:76-102): recomputes the forward on
    every jvp / vjp / vjp_u call like the reference."""

    def __init__(self, mlp: Mlp):
        self.mlp = mlp
        self.n_params = mlp.n_params
        self.n = mlp.widths[-1]

    def _check(self, U):
        if not np.all(np.isfinite(U)):      # as_state (nn.py:26-35)
            raise ValueError("vector contains non-finite entries")

    def eval(self, U, t, c: Counters):
        self._check(U)
        c.nfe_forward += 1
        out, _, _ = self.mlp.forward(self.mlp.input(U, t))
        return out

    def jvp(self, U, t, Wt, c: Counters):
        self._check(U)
        c.nfe_forward += 1
        _, _, pre = self.mlp.forward(self.mlp.input(U, t))
        S0 = np.concatenate([Wt, np.zeros((Wt.shape[0], 1))], axis=1) if self.mlp.time_input else Wt
        return self.mlp.jvp(pre, S0)

    def vjp(self, U, t, V, c: Counters):
        self._check(U)
        c.nfe_backward += 1
        _, acts, pre = self.mlp.forward(self.mlp.input(U, t))
        d, dth = self.mlp.vjp(acts, pre, V)
        return d[:, :self.n], dth

    def vjp_u(self, U, t, V, c: Counters):
        self._check(U)
        c.nfe_backward += 1
        _, acts, pre = self.mlp.forward(self.mlp.input(U, t))
        d, _ = self.mlp.vjp(acts, pre, V, want_theta=False)
        return d[:, :self.n]


class StiffField:
    """C5 RHS f(u) = a*u + s*MLP(u) assembled like a reference ``CallableField``
    (integrators.py:105-141) from the nn.py products."""

    def __init__(self, mlp: Mlp, diag, scale):
        self.mlp = mlp
        self.a = np.asarray(diag, dtype=np.float64)
        self.s = float(scale)
        self.n_params = mlp.n_params
        self.n = mlp.widths[-1]

    def eval(self, U, t, c):
        c.nfe_forward += 1
        out, _, _ = self.mlp.forward(U)
        return self.a * U + self.s * out

    def jvp(self, U, t, Wt, c):
        c.nfe_forward += 1
        _, _, pre = self.mlp.forward(U)
        return self.a * Wt + self.s * self.mlp.jvp(pre, Wt)

    def vjp(self, U, t, V, c):
        c.nfe_backward += 1
        _, acts, pre = self.mlp.forward(U)
        d, dth = self.mlp.vjp(acts, pre, V)
        return self.a * V + self.s * d, self.s * dth

    def vjp_u(self, U, t, V, c):
        c.nfe_backward += 1
        _, acts, pre = self.mlp.forward(U)
        d, _ = self.mlp.vjp(acts, pre, V, want_theta=False)
        return self.a * V + self.s * d


# ---------------------------------------------------------------------------
# solvers (linalg.py:22-142)


@dataclass(frozen=True)
class SolverCfg:
    newton_tol: float = 1e-10
    newton_maxit: int = 50
    gmres_tol: float = 1e-12
    gmres_maxit: int = 200
    gmres_restart: int = 30


def gmres(apply_a, rhs, cfg: SolverCfg):
    """Restarted GMRES(m), MGS Arnoldi, Givens on the fly, x0 = 0
    (linalg.py:37-114).  Returns (x, total Arnoldi steps)."""
    n = rhs.shape[0]
    x = np.zeros(n)
    bnorm = np.linalg.norm(rhs)
    if bnorm == 0.0:
        return np.zeros(n), 0
    tol = cfg.gmres_tol * bnorm
    m = min(cfg.gmres_restart, n)
    total = 0
    while True:
        r = rhs - apply_a(x)
        beta = np.linalg.norm(r)
        if beta <= tol:
            return x, total
        if total >= cfg.gmres_maxit:
            break
        Q = np.zeros((m + 1, n))
        H = np.zeros((m + 1, m))
        cs, sn, g = np.zeros(m), np.zeros(m), np.zeros(m + 1)
        Q[0] = r / beta
        g[0] = beta
        used = 0
        broke = False
        for k in range(m):
            if total >= cfg.gmres_maxit:
                break
            w = apply_a(Q[k])
            total += 1
            for i in range(k + 1):
                H[i, k] = w @ Q[i]
                w = w - H[i, k] * Q[i]
            H[k + 1, k] = np.linalg.norm(w)
            if H[k + 1, k] > 1e-300:
                Q[k + 1] = w / H[k + 1, k]
            else:
                broke = True
            for i in range(k):
                top = cs[i] * H[i, k] + sn[i] * H[i + 1, k]
                H[i + 1, k] = -sn[i] * H[i, k] + cs[i] * H[i + 1, k]
                H[i, k] = top
            den = np.hypot(H[k, k], H[k + 1, k])
            if den == 0.0:
                cs[k], sn[k] = 1.0, 0.0
            else:
                cs[k], sn[k] = H[k, k] / den, H[k + 1, k] / den
            H[k, k] = cs[k] * H[k, k] + sn[k] * H[k + 1, k]
            H[k + 1, k] = 0.0
            g[k + 1] = -sn[k] * g[k]
            g[k] = cs[k] * g[k]
            used = k + 1
            if abs(g[used]) <= tol or broke:
                break
        if used == 0:
            break
        y = np.linalg.solve(H[:used, :used], g[:used])
        x = x + Q[:used].T @ y
    r = rhs - apply_a(x)
    res = np.linalg.norm(r)
    if res <= tol:
        return x, total
    raise ConvergenceError(f"GMRES did not converge in {total} iterations (residual {res:.3e})",
                           residual=res)


def newton(residual, apply_jac, u0, cfg: SolverCfg):
    """Newton with GMRES inner solves, absolute ||F||_2 tolerance
    (linalg.py:117-142).  Returns (u, iterations, gmres_iters list)."""
    u = u0.copy()
    r = residual(u)
    rn = np.linalg.norm(r)
    its = []
    for it in range(cfg.newton_maxit):
        if rn <= cfg.newton_tol:
            return u, it, its
        if not np.all(np.isfinite(r)):
            raise ConvergenceError("Newton residual is non-finite", residual=rn)
        delta, k = gmres(lambda w: apply_jac(u, w), -r, cfg)
        its.append(k)
        u = u + delta
        r = residual(u)
        rn = np.linalg.norm(r)
    if rn <= cfg.newton_tol:
        return u, cfg.newton_maxit, its
    raise ConvergenceError(f"Newton did not converge in {cfg.newton_maxit} iterations",
                           residual=rn)


# ---------------------------------------------------------------------------
# steps (integrators.py:196-244)


@dataclass
class Record:
    n: int
    t: float
    h: float
    u: np.ndarray
    stages: list
    u_next: np.ndarray


def rk_step(tab: Tableau, fld, u, t, h, c: Counters, k_first=None):
    """explicit_rk_step (integrators.py:196-222): ascending-j stage sums with
    (h*a_ij) formed first, exact zeros skipped; FSAL reuse of k_first."""
    s = tab.stages
    stages, ks = [], []
    for i in range(s):
        ui = u.copy()
        for j in range(i):
            aij = tab.a[i, j]
            if aij != 0.0:
                ui = ui + (h * aij) * ks[j]
        stages.append(ui)
        if i == 0 and k_first is not None:
            ks.append(k_first)
        else:
            ks.append(fld.eval(ui, t + tab.c[i] * h, c))
    un = u.copy()
    for i in range(s):
        if tab.b[i] != 0.0:
            un = un + (h * tab.b[i]) * ks[i]
    if not np.all(np.isfinite(un)):
        raise IntegrationError(f"state overflowed at t={t} (h={h})")
    return Record(-1, t, h, u, stages, un), (ks[-1] if tab.fsal else None)


class SampleField:
    """Row view of a batched field: lets per-sample solvers drive it."""

    def __init__(self, fld, row_extra=None):
        self.fld = fld

    def eval(self, u, t, c):
        return self.fld.eval(u[None, :], t, c)[0]

    def jvp(self, u, t, w, c):
        return self.fld.jvp(u[None, :], t, w[None, :], c)[0]

    def vjp(self, u, t, v, c):
        d, p = self.fld.vjp(u[None, :], t, v[None, :], c)
        return d[0], p

    def vjp_u(self, u, t, v, c):
        return self.fld.vjp_u(u[None, :], t, v[None, :], c)[0]


def theta_step_sample(theta, sf: SampleField, u, t, h, cfg, c, stats=None):
    """theta_step for one sample (integrators.py:225-244)."""
    f0 = sf.eval(u, t, c)
    base = u + h * (1.0 - theta) * f0
    t1 = t + h

    def residual(x):
        return x - base - (h * theta) * sf.eval(x, t1, c)

    def apply_jac(x, w):
        return w - (h * theta) * sf.jvp(x, t1, w, c)

    try:
        un, its, gits = newton(residual, apply_jac, u, cfg)
    except ConvergenceError as err:
        raise IntegrationError(f"implicit step at t={t} failed: {err}") from err
    if stats is not None:
        stats["newton"].append(its)
        stats["gmres"].extend(gits)
    return un


def theta_step(theta, fld, U, t, h, cfg, c, sample_counters=None, stats=None):
    """Batched theta step: an independent Newton-GMRES solve per sample."""
    sf = SampleField(fld)
    out = np.empty_like(U)
    for bi in range(U.shape[0]):
        cb = Counters()
        st = stats[bi] if stats is not None else None
        out[bi] = theta_step_sample(theta, sf, U[bi], t, h, cfg, cb, st)
        c.nfe_forward += cb.nfe_forward
        if sample_counters is not None:
            sample_counters[bi].nfe_forward += cb.nfe_forward
    return Record(-1, t, h, U, [U.copy(), out.copy()], out)


# ---------------------------------------------------------------------------
# adjoint steps (adjoint.py:67-126)


def rk_adjoint_step(tab, fld, rec: Record, lam, mu, c: Counters):
    """Reverse stage order: w_i = b_i lam + sum_{j>i, a_ji != 0} a_ji Lam_j;
    Lam_i = h J(U_i)^T w_i; lam += Lam_i; mu += h P(U_i)^T w_i (adjoint.py:67-94)."""
    s = tab.stages
    if len(rec.stages) != s:
        raise ValueError("stages mismatch")
    Lam = [None] * s
    lam_new = lam.copy()
    mu = mu.copy()
    for i in reversed(range(s)):
        w = tab.b[i] * lam
        for j in range(i + 1, s):
            if tab.a[j, i] != 0.0:
                w = w + tab.a[j, i] * Lam[j]
        jtv, ptv = fld.vjp(rec.stages[i], rec.t + tab.c[i] * rec.h, w, c)
        Lam[i] = rec.h * jtv
        lam_new += Lam[i]
        mu += rec.h * ptv
    if not (np.all(np.isfinite(lam_new)) and np.all(np.isfinite(mu))):
        raise GradientExplosionError("non-finite adjoint state in reverse sweep")
    return lam_new, mu


def theta_adjoint_step(theta, fld, rec: Record, lam, mu, cfg, c: Counters,
                       sample_counters=None, stats=None):
    """Transposed GMRES solve then the two VJP pairs (adjoint.py:97-126),
    per sample."""
    sf = SampleField(fld)
    U0, U1 = rec.stages
    t1 = rec.t + rec.h
    h = rec.h
    lam_out = np.empty_like(lam)
    mu = mu.copy()
    for bi in range(lam.shape[0]):
        cb = Counters()

        def apply_at(v):
            return v - (h * theta) * sf.vjp_u(U1[bi], t1, v, cb)

        lam_s, k = gmres(apply_at, lam[bi], cfg)
        if stats is not None:
            stats[bi]["gmres_adj"].append(k)
        _, p1 = sf.vjp(U1[bi], t1, lam_s, cb)
        mu = mu + (h * theta) * p1
        if theta < 1.0:
            j0, p0 = sf.vjp(U0[bi], rec.t, lam_s, cb)
            lam_out[bi] = lam_s + h * (1.0 - theta) * j0
            mu = mu + h * (1.0 - theta) * p0
        else:
            lam_out[bi] = lam_s
        c.nfe_backward += cb.nfe_backward
        if sample_counters is not None:
            sample_counters[bi].nfe_backward += cb.nfe_backward
    if not (np.all(np.isfinite(lam_out)) and np.all(np.isfinite(mu))):
        raise GradientExplosionError("non-finite adjoint state in reverse sweep")
    return lam_out, mu


# ---------------------------------------------------------------------------
# checkpoint store + forward/backward (checkpointing.py:201-340,
# adjoint.py:151-279, integrators.py:252-292, :352-368)


@dataclass
class Scheme:
    name: str
    kind: str
    tab: Tableau = None
    theta: float = 0.0


def scheme(name):
    if name in THETA_SCHEMES:
        return Scheme(name, "theta", None, THETA_SCHEMES[name])
    return Scheme(name, "rk", explicit_tableau(name))


def parse_policy(text):
    text = text.strip()
    if text.startswith("revolve"):
        return "revolve", int(text.split(":", 1)[1]) if ":" in text else 1
    if text not in ("store_all", "store_solutions"):
        raise ValueError(text)
    return text, 0


@dataclass
class Run:
    """Per-call state of the gradient (counters, store, per-sample stats)."""
    sch: Scheme
    fld: object
    cfg: SolverCfg
    B: int
    c: Counters = dc_field(default_factory=Counters)
    sc: StoreCounters = dc_field(default_factory=StoreCounters)
    sample: list = None
    stats: list = None

    def __post_init__(self):
        self.sample = [Counters() for _ in range(self.B)]
        self.stats = [{"newton": [], "gmres": [], "gmres_adj": []} for _ in range(self.B)]

    def step(self, U, t, h, k_carry):
        if self.sch.kind == "rk":
            before = self.c.nfe_forward
            rec, k = rk_step(self.sch.tab, self.fld, U, t, h, self.c, k_first=k_carry)
            for s in self.sample:
                s.nfe_forward += self.c.nfe_forward - before
            return rec, k
        rec = theta_step(self.sch.theta, self.fld, U, t, h, self.cfg, self.c,
                         self.sample, self.stats)
        return rec, None

    def replay(self, U, t, h):
        self.c.steps_recomputed += 1
        self.sc.recomputed_steps += 1
        rec, _ = self.step(U, t, h, None)     # replay never reuses FSAL (integrators.py:363)
        return rec

    def adjoint(self, rec, lam, mu):
        if self.sch.kind == "rk":
            before = self.c.nfe_backward
            out = rk_adjoint_step(self.sch.tab, self.fld, rec, lam, mu, self.c)
            for s in self.sample:
                s.nfe_backward += self.c.nfe_backward - before
            return out
        return theta_adjoint_step(self.sch.theta, self.fld, rec, lam, mu, self.cfg, self.c,
                                  self.sample, self.stats)


def grad_terminal(fld, scheme_name, U0, t0, tF, n_steps, policy="store_all", seed_fn=None,
                  cfg: SolverCfg = None, times=None, obs=None, mu0=None, injections=None):
    """forward_pass + terminal seed + backward_sweep for a batch of samples.

    ``seed_fn(u_final) -> (loss, lam_N)``; default is the BASELINE loss
    L = 0.5 * mean_b ||u_b(T)||^2 with seed lam_N = u_b(T) / B.
    ``obs`` (an obs_losses.ObsLoss) replaces the terminal loss by observations
    at step boundaries: states captured in the forward (adjoint.py:196-210),
    seeds injected into lambda before reversing the step that ends at each
    observed boundary and at boundary 0 last (adjoint.py:235-253).
    ``mu0`` (terminal mu, adjoint_terminal adjoint.py:47-52) and ``injections``
    ({boundary index: [B, N] seed}, inject_observation :135-140) drive the sweep of
    backward_sweep (:235-253) with caller-formed seeds.
    Returns a dict with u_final, du0, dtheta (batch sum of per-sample mu),
    loss, counters, store counters, per-sample counters, solver stats and the
    state at every boundary (``states``).
    """
    sch = scheme(scheme_name)
    cfg = cfg or SolverCfg()
    U0 = np.asarray(U0, dtype=np.float64)
    B = U0.shape[0]
    run = Run(sch, fld, cfg, B)
    kind, nc = parse_policy(policy)
    ts = np.linspace(t0, tF, n_steps + 1) if times is None else np.asarray(times, float)
    n_steps = len(ts) - 1

    # forward (integrate fixed branch, integrators.py:274-292) + store.on_step
    sched = phase2 = None
    fwd_store = set()
    if kind == "revolve":
        sched = revolve_schedule(n_steps, nc)
        first = next(i for i, a in enumerate(sched) if a[0] == "reverse")
        fwd_store = {a[1] for a in sched[:first] if a[0] == "store"}
        phase2 = sched[first:]
    slots, sols, meta = {}, {}, []
    final = None
    U = U0.copy()
    k_carry = None
    capture = {}
    want = set(obs.steps) if obs is not None else set()
    if 0 in want:
        capture[0] = U0.copy()
    states = [U0.copy()]
    for n in range(n_steps):
        t, h = ts[n], ts[n + 1] - ts[n]
        rec, k_carry = run.step(U, t, h, k_carry)
        if n + 1 in want:
            capture[n + 1] = rec.u_next.copy()
        rec.n = n
        run.c.steps_accepted += 1
        last = n == n_steps - 1
        if kind == "store_all":
            if last:
                final = rec
            else:
                slots[n] = rec
                run.sc.stored_states += 1
                run.sc.stored_stage_vectors += len(rec.stages)
        elif kind == "store_solutions":
            if last:
                final = rec
            else:
                sols[n] = rec.u.copy()
                run.sc.stored_states += 1
        else:
            if n in fwd_store:
                slots[n] = rec
                run.sc.stored_states += 1
                run.sc.stored_stage_vectors += len(rec.stages)
                run.sc.max_live_slots = max(run.sc.max_live_slots, len(slots))
            if last:
                final = rec
        meta.append((t, h))
        U = rec.u_next
        states.append(U.copy())
    if kind != "revolve":
        run.sc.max_live_slots = max(len(slots), len(sols))
    u_final = U

    inj = {}
    preds = None
    if obs is not None:
        preds = np.stack([capture[j] for j in obs.steps])
        loss, seeds = obs.loss_and_seeds(preds)
        for j, sd in zip(obs.steps, seeds):
            inj[j] = inj.get(j, 0.0) + sd
        lam = np.zeros_like(U0)
    elif seed_fn is None:
        loss = float(np.mean(0.5 * np.sum(u_final * u_final, axis=1)))
        lam = u_final / B
    else:
        loss, lam = seed_fn(u_final)
    mu = np.zeros(fld.n_params) if mu0 is None else np.asarray(mu0, dtype=np.float64).copy()
    for j, sd in (injections or {}).items():
        inj[j] = inj.get(j, 0.0) + np.asarray(sd, dtype=np.float64)

    def records():
        if kind == "store_all":
            yield final
            for n in range(n_steps - 2, -1, -1):
                yield slots[n]
        elif kind == "store_solutions":
            yield final
            for n in range(n_steps - 2, -1, -1):
                t, h = meta[n]
                rec = run.replay(sols[n], t, h)
                rec.n = n
                yield rec
        else:
            hand = final
            state = final.u_next
            for kd, step, a, b in phase2:
                if kd == "restore":
                    state = U0.copy() if step == -1 else slots[step].u_next.copy()
                    hand = None
                elif kd == "advance":
                    for n in range(a, b):
                        t, h = meta[n]
                        rec = run.replay(state, t, h)
                        rec.n = n
                        state = rec.u_next
                        hand = rec
                elif kd == "store":
                    assert hand is not None and hand.n == step and len(slots) < nc
                    slots[step] = hand
                    run.sc.max_live_slots = max(run.sc.max_live_slots, len(slots))
                else:
                    if hand is not None and hand.n == step:
                        rec = hand
                    else:
                        rec = slots.pop(step)
                    yield rec

    for rec in records():
        if rec.n + 1 in inj:
            lam = lam + inj[rec.n + 1]
        lam, mu = run.adjoint(rec, lam, mu)
    if 0 in inj:
        lam = lam + inj[0]
    return {
        "u_final": u_final, "du0": lam, "dtheta": mu, "loss": loss, "predictions": preds,
        "counters": run.c, "store": run.sc, "sample_counters": run.sample,
        "stats": run.stats, "states": states,
    }


def sweep_with_seeds(fld, scheme_name, U0, t0, tF, n_steps, lamN, muN=None, injections=None,
                     policy="store_all", cfg: SolverCfg = None):
    """backward_sweep from a caller-formed terminal AdjointState (adjoint.py:47-52,
    :235-253): lambda_N = lamN [B, N], mu_N = muN, plus boundary injections."""
    r = grad_terminal(fld, scheme_name, U0, t0, tF, n_steps, policy,
                      seed_fn=lambda uf: (0.0, np.asarray(lamN, dtype=np.float64).copy()),
                      cfg=cfg, mu0=muN, injections=injections)
    return {"lam": r["du0"], "mu": r["dtheta"], "states": r["states"], "u_final": r["u_final"]}


def rel_error(approx, ref):
    """Inf-norm error relative to max|ref| (adjoint.py:368-373)."""
    a = np.asarray(approx, dtype=np.float64)
    r = np.asarray(ref, dtype=np.float64)
    return float(np.max(np.abs(a - r)) / max(float(np.max(np.abs(r))), 1e-300))
