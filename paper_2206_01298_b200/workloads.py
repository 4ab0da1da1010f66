"""BASELINE workloads (configs C1..C5) assembled on the device API.

``field_from_config`` builds the device field for a seeded ConfigInputs
(paper_2206_01298_b200.configs); ``run_config`` runs one ``grad`` on it.
"""

from __future__ import annotations

from .configs import ConfigInputs
from .controls import FixedController, SolverConfig
from .engine import grad
from .fields import MlpField, MlpModel, MlpSpec, StiffMlpField
from .losses import terminal_loss
from .policies import CheckpointPolicy
from .schemes import tableau_catalog


def field_from_config(ci: ConfigInputs):
    spec = MlpSpec(tuple(ci.widths), ci.activation, ci.time_input, ci.dtype)
    model = MlpModel(spec, ci.theta)
    if ci.kind == "mlp":
        return MlpField(model)
    if ci.kind == "stiff":
        return StiffMlpField(model, ci.extras["diag"], ci.extras["scale"])
    raise NotImplementedError(f"config kind {ci.kind!r} is not built yet")


def solver_from_config(ci: ConfigInputs):
    s = ci.extras.get("solver")
    return SolverConfig(**s) if s else SolverConfig()


def run_config(ci: ConfigInputs, policy: str = None, field=None, u0=None, **kw):
    field = field if field is not None else field_from_config(ci)
    pol = CheckpointPolicy.parse(policy or ci.policy)
    return grad(field, tableau_catalog(ci.scheme), terminal_loss("half_sqnorm", ci.tF),
                ci.u0 if u0 is None else u0, ci.t0, ci.tF, FixedController(ci.n_steps), pol,
                solver_from_config(ci), **kw)
