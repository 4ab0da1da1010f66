"""Vector fields on the device (reference Field protocol, integrators.py:53-141;
MLP model API, nn.py:38-112).

Every method is batched over a leading sample dimension: ``u`` is a CUDA
tensor [B, N]; ``eval`` returns f(u, t) [B, N]; ``jvp`` (df/du) w; ``vjp``
((df/du)^T v [B, N], sum_b (df/dtheta)^T v_b [Np]); ``vjp_u`` the state part
only.  Counters are mutated in place with the reference semantics (one call =
one evaluation per trajectory).  All compute goes through the C ABI.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .configs import ACT_IDS
from .controls import NfeCounters, raise_status

ACTIVATION_IDS = dict(ACT_IDS)
_TORCH_DTYPE = {"f32": torch.float32, "f64": torch.float64}


def _device():
    if not torch.cuda.is_available():
        raise RuntimeError("a CUDA device is required (the engine has no CPU path)")
    return torch.device("cuda", torch.cuda.current_device())


def to_device(x, dtype: torch.dtype) -> torch.Tensor:
    """Contiguous CUDA tensor of ``dtype`` (host arrays are copied H2D)."""
    if isinstance(x, torch.Tensor):
        t = x.to(device=_device(), dtype=dtype)
    else:
        t = torch.as_tensor(np.asarray(x), dtype=dtype).to(_device())
    return t.contiguous()


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


@dataclass(frozen=True)
class MlpSpec:
    """Architecture: layer widths, hidden activation, optional time input,
    compute dtype ("f64" like the reference, or "f32")."""

    layer_widths: tuple
    activation: str = "gelu"
    time_input: bool = False
    dtype: str = "f64"

    def __post_init__(self):
        widths = tuple(int(w) for w in self.layer_widths)
        object.__setattr__(self, "layer_widths", widths)
        if len(widths) < 2:
            raise ValueError("need at least input and output layer widths")
        if len(widths) - 1 > _lib.OB_MAX_LAYERS:
            raise ValueError(f"at most {_lib.OB_MAX_LAYERS} affine layers")
        if any(w <= 0 for w in widths):
            raise ValueError("layer widths must be positive")
        if self.activation not in ACTIVATION_IDS:
            raise ValueError(f"unknown activation {self.activation!r}")
        if self.dtype not in _TORCH_DTYPE:
            raise ValueError("dtype must be 'f32' or 'f64'")
        expected = widths[-1] + (1 if self.time_input else 0)
        if widths[0] != expected:
            raise ValueError(f"input width {widths[0]} inconsistent with state dim "
                             f"{widths[-1]} and time_input={self.time_input}")

    @property
    def state_dim(self) -> int:
        return self.layer_widths[-1]

    @property
    def n_params(self) -> int:
        ws = self.layer_widths
        return sum(ws[l + 1] * ws[l] + ws[l + 1] for l in range(len(ws) - 1))

    @property
    def act_id(self) -> int:
        return ACTIVATION_IDS[self.activation]

    @property
    def torch_dtype(self):
        return _TORCH_DTYPE[self.dtype]


def mlp_spec(state_dim, hidden, depth, activation="gelu", time_input=False, dtype="f64") -> MlpSpec:
    widths = (state_dim + (1 if time_input else 0),) + (hidden,) * depth + (state_dim,)
    return MlpSpec(widths, activation, time_input, dtype)


class MlpModel:
    """Flat parameter vector theta (per layer W row-major [out, in], then b;
    kernels.py:9-16) resident on the device in the spec's dtype."""

    def __init__(self, spec: MlpSpec, theta):
        self.spec = spec
        th = to_device(theta, spec.torch_dtype).reshape(-1)
        if th.numel() != spec.n_params:
            raise ValueError(f"expected length {spec.n_params}, got {th.numel()}")
        if not bool(torch.isfinite(th).all()):
            raise ValueError("vector contains non-finite entries")
        self.theta = th

    @property
    def n(self) -> int:
        return self.spec.state_dim

    @property
    def n_params(self) -> int:
        return self.spec.n_params


def init_model(spec: MlpSpec, seed=0) -> MlpModel:
    """Uniform init in [-sqrt(1/fan_in), +sqrt(1/fan_in)] per layer, seeded
    (same draw order as nn.py:102-112)."""
    rng = np.random.default_rng(seed)
    parts = []
    ws = spec.layer_widths
    for l in range(len(ws) - 1):
        bound = np.sqrt(1.0 / ws[l])
        parts.append(rng.uniform(-bound, bound, size=ws[l + 1] * ws[l]))
        parts.append(rng.uniform(-bound, bound, size=ws[l + 1]))
    return MlpModel(spec, np.concatenate(parts))


class Field:
    """Device field base: subclasses provide ``desc()`` and ``aux()``."""

    kind = _lib.OB_FIELD_MLP
    n_params = 0

    def desc(self) -> _lib.FieldDesc:
        raise NotImplementedError

    def aux(self):
        return None

    @property
    def torch_dtype(self):
        raise NotImplementedError

    @property
    def n(self) -> int:
        raise NotImplementedError

    def _prep(self, u):
        u = to_device(u, self.torch_dtype)
        if u.dim() == 1:
            u = u.unsqueeze(0)
        if u.dim() != 2 or u.shape[1] != self.n:
            raise ValueError(f"expected [B, {self.n}] states, got {tuple(u.shape)}")
        return u

    def _call(self, fn, u, t, w=None, want_ptv=False):
        lib = _lib.load()
        u = self._prep(u)
        out = torch.empty_like(u)
        aux = self.aux()
        aux_p = aux.data_ptr() if aux is not None else None
        d = self.desc()
        args = [C.byref(d), u.shape[0], self.theta_tensor().data_ptr(), aux_p, u.data_ptr(), float(t)]
        if w is not None:
            w = self._prep(w)
            if w.shape != u.shape:
                raise ValueError("tangent/cotangent shape mismatch")
            args.append(w.data_ptr())
        args.append(out.data_ptr())
        ptv = None
        if want_ptv:
            ptv = torch.empty(self.n_params, dtype=self.torch_dtype, device=u.device)
            args.append(ptv.data_ptr())
        args.append(stream_ptr())
        raise_status(fn(*args), _lib.last_error())
        return out, ptv

    def eval(self, u, t, counters: NfeCounters = None):
        if counters is not None:
            counters.nfe_forward += 1
        return self._call(_lib.load().ob_field_eval, u, t)[0]

    def jvp(self, u, t, w, counters: NfeCounters = None):
        # one linearization pass; counted like a forward evaluation (integrators.py:88-92)
        if counters is not None:
            counters.nfe_forward += 1
        return self._call(_lib.load().ob_field_jvp, u, t, w)[0]

    def vjp(self, u, t, v, counters: NfeCounters = None):
        if counters is not None:
            counters.nfe_backward += 1
        return self._call(_lib.load().ob_field_vjp, u, t, v, want_ptv=True)

    def vjp_u(self, u, t, v, counters: NfeCounters = None):
        if counters is not None:
            counters.nfe_backward += 1
        return self._call(_lib.load().ob_field_vjp_u, u, t, v)[0]


class MlpField(Field):
    """The neural-network right-hand side f(u, theta, t) (integrators.py:76-102)."""

    kind = _lib.OB_FIELD_MLP

    def __init__(self, model: MlpModel):
        self.model = model
        self.n_params = model.n_params

    @property
    def torch_dtype(self):
        return self.model.spec.torch_dtype

    @property
    def n(self):
        return self.model.n

    def theta_tensor(self):
        return self.model.theta

    def desc(self) -> _lib.FieldDesc:
        sp = self.model.spec
        d = _lib.FieldDesc()
        d.kind = self.kind
        d.dtype = _lib.OB_F32 if sp.dtype == "f32" else _lib.OB_F64
        d.n_layers = len(sp.layer_widths) - 1
        for i, w in enumerate(sp.layer_widths):
            d.widths[i] = w
        d.activation = sp.act_id
        d.time_input = int(sp.time_input)
        d.out_scale = 1.0
        d.n_params = sp.n_params
        return d


class StiffMlpField(MlpField):
    """f(u) = a*u + s*MLP(u) with diagonal a (config C5).  The reference builds
    this as a CallableField from nn.py products; here it is
    a native field kind sharing the MLP kernels."""

    kind = _lib.OB_FIELD_STIFF

    def __init__(self, model: MlpModel, diag, scale: float):
        if model.spec.time_input:
            raise ValueError("stiff field is autonomous")
        super().__init__(model)
        self.diag = to_device(diag, model.spec.torch_dtype).reshape(-1)
        if self.diag.numel() != model.n:
            raise ValueError("diag length must equal the state dimension")
        self.scale = float(scale)

    def aux(self):
        return self.diag

    def desc(self):
        d = super().desc()
        d.out_scale = self.scale
        return d


class CnfField(MlpField):
    """Continuous normalizing flow with a Hutchinson trace estimator (config C4).

    State [z (D), Delta]; f_aug = [f(z, t), -eps^T (df/dz) eps] with f an MLP
    taking time as its last input and one fixed probe eps per sample
    ([B, D], e.g. Rademacher).  The probes bind the field to a batch.  No
    reference counterpart; restated oracle in
    oracle/fields_ext.py.
    """

    kind = _lib.OB_FIELD_CNF

    def __init__(self, model: MlpModel, eps):
        if not model.spec.time_input:
            raise ValueError("CNF field takes time as an input")
        if model.spec.dtype != "f32":
            raise NotImplementedError("CNF kernels are built for fp32")
        super().__init__(model)
        self.eps = to_device(eps, model.spec.torch_dtype)
        if self.eps.dim() != 2 or self.eps.shape[1] != model.n:
            raise ValueError("eps must be [B, D]")

    @property
    def n(self):
        return self.model.n + 1

    def aux(self):
        return self.eps


class ConvField(Field):
    """Image-classifier ODE block (config C3): state = 16x16x64 NHWC image
    flattened to [B, 16384]; f(u, t) = conv3x3(65 -> 64)(cat(u, t)) -> relu ->
    conv3x3(64 -> 64), padding 1.  theta = [W1 (64 x 3 x 3 x 65), b1,
    W2 (64 x 3 x 3 x 64), b2].  No reference counterpart;
    restated oracle in oracle/fields_ext.py."""

    kind = _lib.OB_FIELD_CONV
    C = 64
    widths = (65, 64, 64)

    def __init__(self, theta, dtype="f32"):
        if dtype != "f32":
            raise NotImplementedError("conv kernels are built for fp32")
        self.n_params = 64 * 9 * 65 + 64 + 64 * 9 * 64 + 64
        self.theta = to_device(theta, torch.float32).reshape(-1)
        if self.theta.numel() != self.n_params:
            raise ValueError(f"expected length {self.n_params}, got {self.theta.numel()}")

    @property
    def torch_dtype(self):
        return torch.float32

    @property
    def n(self):
        return 16 * 16 * self.C

    def theta_tensor(self):
        return self.theta

    def desc(self) -> _lib.FieldDesc:
        d = _lib.FieldDesc()
        d.kind = self.kind
        d.dtype = _lib.OB_F32
        d.n_layers = 2
        for i, w in enumerate(self.widths):
            d.widths[i] = w
        d.activation = ACTIVATION_IDS["relu"]
        d.time_input = 1
        d.out_scale = 1.0
        d.n_params = self.n_params
        return d
