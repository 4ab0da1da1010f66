"""BASELINE workloads (configs C1..C5) assembled on the device API.

``field_from_config`` builds the device field for a seeded ConfigInputs
(paper_2206_01298_b200.configs); ``run_config`` runs one ``grad`` on it.
"""

from __future__ import annotations

import numpy as np

from .configs import ConfigInputs
from .controls import FixedController, SolverConfig
from .engine import grad
from .fields import CnfField, ConvField, MlpField, MlpModel, MlpSpec, StiffMlpField
from .losses import terminal_loss
from .policies import CheckpointPolicy
from .schemes import tableau_catalog


def field_from_config(ci: ConfigInputs, rows=None):
    """Device field of a config; ``rows`` selects a batch shard's per-sample field data
    (the CNF probes) -- a rank's field must carry its own rows."""
    if ci.kind == "conv":
        return ConvField(ci.theta)
    spec = MlpSpec(tuple(ci.widths), ci.activation, ci.time_input, ci.dtype)
    model = MlpModel(spec, ci.theta)
    if ci.kind == "mlp":
        return MlpField(model)
    if ci.kind == "stiff":
        return StiffMlpField(model, ci.extras["diag"], ci.extras["scale"])
    if ci.kind == "cnf":
        eps = ci.extras["eps"] if rows is None else ci.extras["eps"][rows]
        return CnfField(model, eps)
    raise NotImplementedError(f"config kind {ci.kind!r} is not built yet")


def solver_from_config(ci: ConfigInputs):
    s = ci.extras.get("solver")
    return SolverConfig(**s) if s else SolverConfig()


def initial_state(ci: ConfigInputs):
    """Integration state at t0 (CNF: [z0, Delta = 0])."""
    if ci.kind == "cnf":
        return np.concatenate([ci.u0, np.zeros((ci.batch, 1))], axis=1)
    if ci.kind == "conv":
        return ci.u0.reshape(ci.batch, -1)
    return ci.u0


def loss_kind(ci: ConfigInputs) -> str:
    return {"cnf": "cnf_nll", "conv": "ce_head"}.get(ci.kind, "half_sqnorm")


def loss_for(ci: ConfigInputs, rows=slice(None)):
    kind = loss_kind(ci)
    if kind == "ce_head":
        return terminal_loss(kind, ci.tF, (ci.extras["head"], ci.extras["labels"][rows]))
    return terminal_loss(kind, ci.tF)


def run_config(ci: ConfigInputs, policy: str = None, field=None, u0=None, **kw):
    field = field if field is not None else field_from_config(ci)
    pol = CheckpointPolicy.parse(policy or ci.policy)
    return grad(field, tableau_catalog(ci.scheme), loss_for(ci),
                initial_state(ci) if u0 is None else u0, ci.t0, ci.tF,
                FixedController(ci.n_steps), pol, solver_from_config(ci), **kw)
