"""GPU parity for adaptive stepping: per-sample
error-controlled Dopri5 / Bosh3 steps (integrators.py:294-349), one
integration per observation interval (adjoint.py:162-186), and the discrete
adjoint over each sample's frozen grid.  Pinned against
tests/golden/adaptive.npz from the reference's own grad() (tools/make_golden.py
gen_adaptive).

Step-count parity is exact (accepted, rejected, NFE).  The embedded error
estimate cancels ~8 digits, so ulp-level differences in the field evaluation
move the step sizes at the 1e-11 level (the oracle and the reference differ by
the same amount): grids are compared at 1e-9 and gradients at 1e-9 relative.
The frozen-grid identity (adaptive == FixedGridController on the returned grid)
holds at 1e-12.
"""

import numpy as np
import pytest
import torch

from oracle import adaptive as oa
from oracle import core as oc
from oracle import obs_losses as ol
from paper_2206_01298_b200 import (AdaptiveController, CheckpointPolicy, FixedGridController,
                                   IntegrationError, MlpField, MlpModel, MlpSpec, StiffnessError,
                                   grad, tableau_catalog)
from paper_2206_01298_b200.losses import LossSpec, MinMaxScaling

pytestmark = pytest.mark.gpu

CASES = ("dopri5_term", "bosh3_obs", "dopri5_obs0")


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    from paper_2206_01298_b200 import _lib as L
    L.load()


def case(g, name, dtype="f64"):
    sch, kind, pol = (str(x) for x in g[f"{name}/meta"])
    tol, _, h0 = (float(x) for x in g[f"{name}/ctrl"])
    U0 = g[f"{name}/u0"]
    theta = g[f"{name}/theta"]
    if dtype == "f32":
        theta = theta.astype(np.float32).astype(np.float64)
        U0 = U0.astype(np.float32).astype(np.float64)
    N = U0.shape[1]
    model = MlpModel(MlpSpec((N + 1, 16, 16, N), "tanh", time_input=True, dtype=dtype), theta)
    times = tuple(float(t) for t in g[f"{name}/times"])
    scaling = MinMaxScaling(g[f"{name}/lo"], g[f"{name}/hi"]) if f"{name}/lo" in g else None
    loss = LossSpec(kind, times, tuple(g[f"{name}/values"]), scaling)
    ctrl = AdaptiveController(abstol=tol, reltol=tol, h_init=h0)
    return model, sch, pol, loss, ctrl, U0, theta


def run(model, sch, pol, loss, ctrl, U0):
    return grad(MlpField(model), tableau_catalog(sch), loss, U0, 0.0, 1.0, ctrl,
                CheckpointPolicy.parse(pol))


@pytest.mark.parametrize("name", CASES)
def test_adaptive_matches_reference_golden(golden, name):
    g = golden("adaptive.npz")
    model, sch, pol, loss, ctrl, U0, _ = case(g, name)
    res = run(model, sch, pol, loss, ctrl, U0)
    sc = res.sample_counters
    for k in ("nfe_forward", "nfe_backward", "steps_recomputed"):
        assert list(sc[k]) == list(g[f"{name}/{k}"]), k
    assert list(sc["steps_accepted"]) == list(g[f"{name}/accepted"])
    assert list(sc["steps_rejected"]) == list(g[f"{name}/rejected"])
    for b, grid in enumerate(res.grids):
        ref = g[f"{name}/grids"][b]
        ref = ref[~np.isnan(ref)]
        assert len(grid) == len(ref) and np.max(np.abs(grid - ref)) <= 1e-9
    ref_loss = float(g[f"{name}/loss"])
    assert abs(res.loss - ref_loss) <= 1e-9 * abs(ref_loss)
    assert oc.rel_error(np.stack(res.predictions), g[f"{name}/predictions"]) <= 1e-9
    assert oc.rel_error(res.dtheta, g[f"{name}/dtheta"]) <= 1e-9
    assert oc.rel_error(res.du0, g[f"{name}/du0"]) <= 1e-9


@pytest.mark.parametrize("name", ("dopri5_term", "bosh3_obs"))
def test_adaptive_equals_frozen_grid(golden, name):
    """test_adjoint.py:342-369: step sizes are data in the reverse pass."""
    g = golden("adaptive.npz")
    model, sch, pol, loss, ctrl, U0, _ = case(g, name)
    res = run(model, sch, pol, loss, ctrl, U0)
    B = U0.shape[0]
    dth = np.zeros_like(res.dtheta)
    for b in range(B):
        lb = LossSpec(loss.kind, loss.times, tuple(v[b:b + 1] for v in loss.values), loss.scaling)
        fr = grad(MlpField(model), tableau_catalog(sch), lb, U0[b:b + 1], 0.0, 1.0,
                  FixedGridController(tuple(res.grids[b])), CheckpointPolicy.parse(pol))
        dth += fr.dtheta / B
        assert oc.rel_error(res.du0[b], fr.du0[0] / B) <= 1e-12
    assert oc.rel_error(res.dtheta, dth) <= 1e-12


def test_adaptive_policies_bit_identical(golden):
    g = golden("adaptive.npz")
    model, sch, _, loss, ctrl, U0, _ = case(g, "dopri5_obs0")
    a = run(model, sch, "store_all", loss, ctrl, U0)
    b = run(model, sch, "store_solutions", loss, ctrl, U0)
    assert np.array_equal(a.dtheta, b.dtheta) and np.array_equal(a.du0, b.du0)
    assert a.loss == b.loss


@pytest.mark.parametrize("name", ("dopri5_term", "bosh3_obs"))
def test_adaptive_fp32_matches_oracle(golden, name):
    g = golden("adaptive.npz")
    model, sch, pol, loss, ctrl, U0, theta = case(g, name, "f32")
    res = run(model, sch, pol, loss, ctrl, U0)
    mlp = oc.Mlp(model.spec.layer_widths, "tanh", theta, True)
    vals = np.asarray(g[f"{name}/values"], np.float32).astype(np.float64)
    sc = None
    if loss.scaling is not None:
        sc = ol.MinMax(loss.scaling.lo.astype(np.float32).astype(np.float64),
                       loss.scaling.hi.astype(np.float32).astype(np.float64))
    obs = ol.ObsLoss(loss.kind, range(len(loss.times)), vals, sc)
    ref = oa.grad_adaptive(oc.MlpField(mlp), sch, U0, 0.0, 1.0,
                           oa.AdaptiveCtrl(abstol=ctrl.abstol, reltol=ctrl.reltol, h_init=ctrl.h_init),
                           pol, obs=obs, obs_times=loss.times)
    assert abs(res.loss - ref["loss"]) <= 1e-4 * abs(ref["loss"])
    assert oc.rel_error(res.dtheta, ref["dtheta"]) <= 1e-4
    assert oc.rel_error(res.du0, ref["du0"]) <= 1e-4


def test_adaptive_errors(golden):
    g = golden("adaptive.npz")
    model, sch, _, loss, ctrl, U0, _ = case(g, "dopri5_term")
    fld = MlpField(model)
    dop = tableau_catalog("dopri5")
    with pytest.raises(ValueError):          # checkpointing.py:218-220
        grad(fld, dop, loss, U0, 0.0, 1.0, ctrl, CheckpointPolicy("revolve", 2))
    with pytest.raises(IntegrationError):    # integrators.py:297-299
        grad(fld, tableau_catalog("rk4"), loss, U0, 0.0, 1.0, ctrl)
    with pytest.raises(StiffnessError):      # max_steps per integrate call (:309-311)
        grad(fld, dop, loss, U0, 0.0, 1.0, AdaptiveController(1e-8, 1e-8, h_init=0.01, max_steps=5))
    with pytest.raises(StiffnessError):      # h underflow (:342-343)
        grad(fld, dop, loss, U0, 0.0, 1.0,
             AdaptiveController(1e-12, 1e-12, h_init=0.5, h_min=0.5, h_max=0.5))
    with pytest.raises(NotImplementedError):  # per-sample record capacity of this build
        grad(fld, dop, loss, U0, 0.0, 1.0, AdaptiveController(1e-8, 1e-8, h_init=0.5, max_accepted=3))
    with pytest.raises(ValueError):
        AdaptiveController(abstol=0.0)
