"""Seeded synthetic inputs for the five BASELINE configurations (C1..C5).

Everything is generated on the host in float64 with ``numpy.random.default_rng``
(PCG64), in a fixed documented draw order, so the GPU path, the CPU oracle and
the golden fixtures all consume identical bytes.  fp32 configs round the fp64
draws to fp32 once; the oracle is fed the *rounded* values (as fp64) so input
rounding is never counted as error.

Draw order per config (all from one generator seeded with ``seed``):
  1. parameters, layer by layer: weight (row-major [out, in]) then bias;
  2. config-specific extras (C5 diagonal, C4 Rademacher probes, C3 head + labels);
  3. the initial state ``u0`` (standard normal, [B, N]).

Parameter layout follows the reference flat-theta convention
(``pkg/src/odegrad/kernels.py:9-16``): per layer W row-major [out x in], then b.
The conv config (C3, no reference RHS) uses per conv layer W as
[Cout][kh][kw][Cin] followed by b[Cout]; its head is kept in a separate vector.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

ACT_IDS = {"identity": 0, "relu": 1, "tanh": 2, "gelu": 3, "softplus": 4}


def xavier_uniform_mlp(rng, widths):
    """Xavier/Glorot-uniform weights (bound sqrt(6/(fan_in+fan_out))), zero biases."""
    parts = []
    for l in range(len(widths) - 1):
        nin, nout = widths[l], widths[l + 1]
        bound = np.sqrt(6.0 / (nin + nout))
        parts.append(rng.uniform(-bound, bound, size=nout * nin))
        parts.append(np.zeros(nout))
    return np.concatenate(parts)


def n_params_mlp(widths):
    return sum(widths[l + 1] * widths[l] + widths[l + 1] for l in range(len(widths) - 1))


@dataclass
class ConfigInputs:
    name: str
    dtype: str                   # "f64" | "f32"
    kind: str                    # "mlp" | "stiff" | "cnf" | "conv"
    widths: tuple
    activation: str
    time_input: bool
    scheme: str
    n_steps: int
    t0: float
    tF: float
    policy: str
    theta: np.ndarray            # float64 (already rounded for fp32 configs)
    u0: np.ndarray               # float64 [B, ...]
    extras: dict = field(default_factory=dict)

    @property
    def batch(self) -> int:
        return int(self.u0.shape[0])

    @property
    def np_dtype(self):
        return np.float32 if self.dtype == "f32" else np.float64

    def subset(self, n: int) -> "ConfigInputs":
        """First ``n`` samples (all per-sample extras sliced alike)."""
        ex = {}
        for k, v in self.extras.items():
            if isinstance(v, np.ndarray) and v.ndim >= 1 and v.shape[0] == self.batch \
                    and k in _PER_SAMPLE_EXTRAS:
                ex[k] = v[:n].copy()
            else:
                ex[k] = v
        return ConfigInputs(self.name, self.dtype, self.kind, self.widths, self.activation,
                            self.time_input, self.scheme, self.n_steps, self.t0, self.tF,
                            self.policy, self.theta, self.u0[:n].copy(), ex)


_PER_SAMPLE_EXTRAS = {"eps", "labels"}


def _round(x, dtype):
    if dtype == "f32":
        return x.astype(np.float32).astype(np.float64)
    return x


def make_c1(batch=512, seed=1) -> ConfigInputs:
    """C1: MLP 64-256-64 tanh fp64, RK4 x10 on [0,1], store_all, B=512."""
    rng = np.random.default_rng(seed)
    widths = (64, 256, 64)
    theta = xavier_uniform_mlp(rng, widths)
    u0 = rng.standard_normal((batch, 64))
    return ConfigInputs("C1", "f64", "mlp", widths, "tanh", False, "rk4", 10, 0.0, 1.0,
                        "store_all", theta, u0)


def make_c2(batch=4096, seed=2, policy="revolve:8") -> ConfigInputs:
    """C2: MLP (64+t)-256-64 tanh fp32, Dopri5 x40 on [0,1], revolve:8 | store_all."""
    rng = np.random.default_rng(seed)
    widths = (65, 256, 64)
    theta = _round(xavier_uniform_mlp(rng, widths), "f32")
    u0 = _round(rng.standard_normal((batch, 64)), "f32")
    return ConfigInputs("C2", "f32", "mlp", widths, "tanh", True, "dopri5", 40, 0.0, 1.0,
                        policy, theta, u0)


def make_c3(batch=256, seed=3) -> ConfigInputs:
    """C3: conv ODE block fp32, state 16x16x64 (NHWC), RK4 x10, GAP+linear+CE head.

    f(u,t) = conv3x3(65->64)(cat(u, t)) -> relu -> conv3x3(64->64); padding 1,
    Kaiming-normal (fan_in, gain sqrt 2) weights, zero biases.  Head: linear
    64->10 Xavier-uniform, zero bias; labels uniform in 0..9.
    """
    rng = np.random.default_rng(seed)
    c = 64
    parts = []
    for cin in (c + 1, c):
        std = np.sqrt(2.0 / (cin * 9))
        parts.append(rng.standard_normal(c * 9 * cin) * std)
        parts.append(np.zeros(c))
    theta = _round(np.concatenate(parts), "f32")
    bound = np.sqrt(6.0 / (c + 10))
    head = _round(np.concatenate([rng.uniform(-bound, bound, 10 * c), np.zeros(10)]), "f32")
    labels = rng.integers(0, 10, size=batch).astype(np.int64)
    u0 = _round(rng.standard_normal((batch, 16, 16, c)), "f32")
    return ConfigInputs("C3", "f32", "conv", (c + 1, c, c), "relu", True, "rk4", 10, 0.0, 1.0,
                        "store_all", theta, u0, {"head": head, "labels": labels})


def make_c4(batch=1000, seed=4) -> ConfigInputs:
    """C4: CNF fp32, z in R^43, MLP (43+t)-860-860-43 softplus, Hutchinson with
    one Rademacher probe per sample, Dopri5 x20 on [0,1]."""
    rng = np.random.default_rng(seed)
    widths = (44, 860, 860, 43)
    theta = _round(xavier_uniform_mlp(rng, widths), "f32")
    eps = rng.integers(0, 2, size=(batch, 43)).astype(np.float64) * 2.0 - 1.0
    u0 = _round(rng.standard_normal((batch, 43)), "f32")
    return ConfigInputs("C4", "f32", "cnf", widths, "softplus", True, "dopri5", 20, 0.0, 1.0,
                        "store_all", theta, u0, {"eps": eps})


def make_c5(batch=256, seed=5) -> ConfigInputs:
    """C5: stiff f(u) = a*u + 0.1*MLP(u), a_i = -10^U(0,4), MLP 128-512-128 tanh,
    fp64, Crank-Nicolson x20, Newton 1e-10 + GMRES(30), gmres_maxit raised."""
    rng = np.random.default_rng(seed)
    widths = (128, 512, 128)
    theta = xavier_uniform_mlp(rng, widths)
    diag = -(10.0 ** rng.uniform(0.0, 4.0, size=128))
    u0 = rng.standard_normal((batch, 128))
    return ConfigInputs("C5", "f64", "stiff", widths, "tanh", False, "cn", 20, 0.0, 1.0,
                        "store_all", theta, u0,
                        {"diag": diag, "scale": 0.1,
                         "solver": dict(newton_tol=1e-10, newton_maxit=50, gmres_tol=1e-12,
                                        gmres_maxit=1000, gmres_restart=30)})


MAKERS = {"C1": make_c1, "C2": make_c2, "C3": make_c3, "C4": make_c4, "C5": make_c5}


def make_config(name: str, batch=None, **kw) -> ConfigInputs:
    maker = MAKERS[name]
    if batch is None:
        return maker(**kw)
    return maker(batch=batch, **kw)
