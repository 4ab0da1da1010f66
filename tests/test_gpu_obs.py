"""GPU parity for the observation losses: the reference's
LossSpec mse/mae over K observation times with min-max scaling
(losses.py:10-107), states captured at step boundaries and seeds injected into
the adjoint (adjoint.py:143-279).  Pinned against tests/golden/obs_losses.npz,
produced by the reference's own grad() (tools/make_golden.py gen_obs).

Tolerances: fp64 rel_error <= 1e-10 (loss/predictions 1e-12); fp32 <= 1e-4
against the fp64 oracle on the same fp32-rounded inputs.
"""

import numpy as np
import pytest
import torch

from oracle import core as oc
from oracle import obs_losses as ol
from paper_2206_01298_b200 import (CheckpointPolicy, FixedController, MlpField, MlpModel,
                                   MlpSpec, SolverConfig, grad, tableau_catalog)
from paper_2206_01298_b200.losses import LossSpec, MinMaxScaling

pytestmark = pytest.mark.gpu

CASES = ("mse_rk4", "mae_dopri5", "mse_cn", "mae_rk4_tF")


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    from paper_2206_01298_b200 import _lib as L
    L.load()


def case(g, name, dtype="f64"):
    kind, sch, pol, tin = (str(x) for x in g[f"{name}/meta"])
    tin = tin == "1"
    U0 = g[f"{name}/u0"]
    N = U0.shape[1]
    theta = g[f"{name}/theta"]
    if dtype == "f32":
        theta = theta.astype(np.float32).astype(np.float64)
        U0 = U0.astype(np.float32).astype(np.float64)
    model = MlpModel(MlpSpec((N + int(tin), 8, 8, N), "tanh", time_input=tin, dtype=dtype), theta)
    vals = g[f"{name}/values"]
    times = tuple(float(t) for t in g[f"{name}/times"])
    scaling = MinMaxScaling(g[f"{name}/lo"], g[f"{name}/hi"]) if f"{name}/lo" in g else None
    loss = LossSpec(kind, times, tuple(vals), scaling)
    return model, sch, pol, loss, U0, theta


def run(model, sch, pol, loss, U0, cfg=None):
    return grad(MlpField(model), tableau_catalog(sch), loss, U0, 0.0, 1.0, FixedController(8),
                CheckpointPolicy.parse(pol), cfg)


# fp32 implicit steps: the default Newton 1e-10 / GMRES 1e-12 tolerances are
# below fp32 resolution, so the fp32 case (and its fp64 oracle) use 1e-5
F32_SOLVER = dict(newton_tol=1e-5, gmres_tol=1e-5)


@pytest.mark.parametrize("name", CASES)
def test_observation_losses_match_reference_golden(golden, name):
    g = golden("obs_losses.npz")
    model, sch, pol, loss, U0, _ = case(g, name)
    res = run(model, sch, pol, loss, U0)
    ref_loss = float(g[f"{name}/loss"])
    assert abs(res.loss - ref_loss) <= 1e-12 * max(1.0, abs(ref_loss))
    assert oc.rel_error(np.stack(res.predictions), g[f"{name}/predictions"]) <= 1e-12
    assert oc.rel_error(res.dtheta, g[f"{name}/dtheta"]) <= 1e-10
    assert oc.rel_error(res.du0, g[f"{name}/du0"]) <= 1e-10


@pytest.mark.parametrize("name", ("mse_rk4", "mae_dopri5", "mse_cn"))
def test_observation_losses_fp32_match_oracle(golden, name):
    g = golden("obs_losses.npz")
    model, sch, pol, loss, U0, theta = case(g, name, "f32")
    res = run(model, sch, pol, loss, U0, SolverConfig(**F32_SOLVER))
    mlp = oc.Mlp(model.spec.layer_widths, "tanh", theta, model.spec.time_input)
    vals = np.asarray(g[f"{name}/values"], np.float32).astype(np.float64)
    lo = hi = None
    if loss.scaling is not None:
        lo = loss.scaling.lo.astype(np.float32).astype(np.float64)
        hi = loss.scaling.hi.astype(np.float32).astype(np.float64)
    obs = ol.ObsLoss(loss.kind, ol.match_boundaries(loss.times, np.linspace(0, 1, 9)), vals,
                     ol.MinMax(lo, hi) if lo is not None else None)
    ref = oc.grad_terminal(oc.MlpField(mlp), sch, U0, 0.0, 1.0, 8, pol, obs=obs,
                           cfg=oc.SolverCfg(**F32_SOLVER))
    assert abs(res.loss - ref["loss"]) <= 1e-4 * abs(ref["loss"])
    assert oc.rel_error(res.dtheta, ref["dtheta"]) <= 1e-4
    assert oc.rel_error(res.du0, ref["du0"]) <= 1e-4


def test_observation_policies_bit_identical(golden):
    g = golden("obs_losses.npz")
    model, sch, _, loss, U0, _ = case(g, "mae_dopri5")
    outs = [run(model, sch, pol, loss, U0) for pol in ("store_all", "store_solutions", "revolve:3")]
    for r in outs[1:]:
        assert np.array_equal(r.dtheta, outs[0].dtheta) and np.array_equal(r.du0, outs[0].du0)
        assert r.loss == outs[0].loss


def _zero_field(n):
    return MlpField(MlpModel(MlpSpec((n, 4, n), "tanh"), np.zeros(4 * n + 4 + n * 4 + n)))


def test_known_answers_through_the_device():
    """Zero field: u(t) = u0, so the device loss/seeds are the reference's
    loss_and_grad_seed examples (test_losses.py) and du0 = sum of seeds."""
    rk4, ctrl = tableau_catalog("rk4"), FixedController(4)

    def go(kind, u0, times, obs):
        u0 = np.asarray(u0, float)[None]
        return grad(_zero_field(u0.shape[1]), rk4,
                    LossSpec(kind, times, tuple(np.asarray(o, float) for o in obs)),
                    u0, 0.0, 1.0, ctrl)

    r = go("mae", [1.0, 2.0], (1.0,), [[1.0, 3.0]])
    assert r.loss == 0.5 and np.array_equal(r.du0[0], [0.0, -0.5])
    r = go("mse", [2.0], (1.0,), [[0.0]])
    assert r.loss == 4.0 and r.du0[0, 0] == 4.0
    r = go("mae", [1.0, 5.0], (1.0,), [[1.0, 2.0]])
    assert r.du0[0, 0] == 0.0
    r = go("mse", [1.0], (0.5, 1.0), [[0.0], [0.0]])          # two observations of u = 1
    assert r.loss == 1.0 and r.du0[0, 0] == 2.0
    r = go("mse", [3.0], (0.0, 1.0), [[1.0], [3.0]])           # observation at t0 (boundary 0)
    assert r.loss == 2.0 and r.du0[0, 0] == 2.0


def test_observation_errors():
    fld = _zero_field(2)
    rk4, ctrl = tableau_catalog("rk4"), FixedController(4)
    u0 = np.ones((3, 2))
    with pytest.raises(ValueError):      # not on a step boundary (adjoint.py:213-221)
        grad(fld, rk4, LossSpec("mse", (0.3,), (np.zeros(2),)), u0, 0.0, 1.0, ctrl)
    with pytest.raises(ValueError):      # past the final time (adjoint.py:264-265)
        grad(fld, rk4, LossSpec("mse", (1.5,), (np.zeros(2),)), u0, 0.0, 1.0, ctrl)
    with pytest.raises(ValueError):      # wrong observation shape
        grad(fld, rk4, LossSpec("mse", (1.0,), (np.zeros((2, 2)),)), u0, 0.0, 1.0, ctrl)
