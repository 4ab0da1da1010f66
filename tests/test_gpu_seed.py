"""GPU tests of the split sweep with caller-formed seeds:
forward_pass + backward_sweep with an arbitrary terminal AdjointState
(adjoint.py:47-52, :151-253), injections at observation boundaries
(inject_observation, :135-140), loss_value (:282-291), the torch.autograd
ODEBlock, and the device-side GradientExplosionError (AdjointState.check_finite,
:42-44).
"""

import numpy as np
import pytest
import torch

from oracle import core as oc
from paper_2206_01298_b200 import (AdjointState, CheckpointPolicy, FixedController, GradientExplosionError,
                                   MlpField, MlpModel, MlpSpec, ODEBlock, adjoint_terminal, backward_sweep,
                                   forward_pass, grad, loss_value, tableau_catalog, terminal_loss)
from paper_2206_01298_b200.configs import make_config
from paper_2206_01298_b200.losses import LossSpec
from paper_2206_01298_b200.workloads import field_from_config, initial_state, loss_for, run_config

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    from paper_2206_01298_b200 import _lib as L
    L.load()


def np_(x):
    return x.detach().cpu().numpy().astype(np.float64) if isinstance(x, torch.Tensor) else np.asarray(x)


@pytest.mark.parametrize("name,pol", [("C1", "revolve:3"), ("C2", "revolve:8"), ("C5", "store_all")])
def test_split_sweep_with_grad_seed_equals_grad(name, pol):
    """forward_pass + backward_sweep seeded with the loss's own terminal seed u/B
    reproduces grad() bit for bit (the same kernels, the seed formed by the caller)."""
    ci = make_config(name).subset(8 if name == "C5" else 64)
    fld = field_from_config(ci)
    u0 = torch.as_tensor(ci.u0, dtype=fld.torch_dtype, device="cuda")
    ref = run_config(ci, pol, field=fld, u0=u0)
    scheme = tableau_catalog(ci.scheme)
    pol_ = CheckpointPolicy.parse(pol)
    from paper_2206_01298_b200.workloads import solver_from_config
    scfg = solver_from_config(ci)
    fwd = forward_pass(fld, scheme, u0, ci.t0, ci.tF, FixedController(ci.n_steps), pol_, scfg)
    assert torch.equal(fwd.u_final, ref.u_final)
    seed = fwd.u_final / u0.shape[0]
    adj = backward_sweep(fld, scheme, fwd, adjoint_terminal(seed), solver_cfg=scfg)
    assert torch.equal(adj.lam, ref.du0)
    assert torch.equal(adj.mu, ref.dtheta)


def test_terminal_mu_and_injections_match_oracle():
    """mu_N = dphi/dtheta is carried into mu_0; injections at observation boundaries
    are added to lambda before the step ending there is reversed."""
    ci = make_config("C1").subset(16)
    fld = field_from_config(ci)
    scheme = tableau_catalog("rk4")
    rng = np.random.default_rng(5)
    fwd = forward_pass(fld, scheme, ci.u0, 0.0, 1.0, FixedController(10),
                       CheckpointPolicy("store_solutions"), obs_times=(0.3, 0.6))
    assert len(fwd.obs_states) == 2
    lamN = rng.standard_normal((16, 64))
    muN = rng.standard_normal(fld.n_params)
    inj = {3: rng.standard_normal((16, 64)), 6: rng.standard_normal((16, 64))}
    adj = backward_sweep(fld, scheme, fwd, AdjointState(lamN, muN), injections=inj)
    # oracle: the same sweep with the same seeds (per-step reverse records)
    mlp = oc.Mlp(ci.widths, ci.activation, ci.theta, ci.time_input)
    ref = oc.sweep_with_seeds(oc.MlpField(mlp), "rk4", ci.u0, 0.0, 1.0, 10, lamN, muN, inj)
    assert oc.rel_error(adj.lam, ref["lam"]) <= 1e-12
    assert oc.rel_error(adj.mu, ref["mu"]) <= 1e-12
    obs_ref = ref["states"]
    assert oc.rel_error(fwd.obs_states[0], obs_ref[3]) <= 1e-13
    assert oc.rel_error(fwd.obs_states[1], obs_ref[6]) <= 1e-13
    with pytest.raises(ValueError):
        backward_sweep(fld, scheme, fwd, AdjointState(lamN, None), injections={4: lamN})


def test_loss_value_equals_grad_loss():
    ci = make_config("C2").subset(64)
    fld = field_from_config(ci)
    g = run_config(ci, "revolve:8", field=fld)
    lv = loss_value(fld, tableau_catalog("dopri5"), terminal_loss("half_sqnorm", 1.0), ci.u0, 0.0, 1.0,
                    FixedController(40))
    assert lv == g.loss


def test_ode_block_autograd_c3_head_in_torch_matches_fused_head():
    """The C3 classifier with the ODE block inside a torch graph: GAP + linear + CE in
    torch, the ODE block's backward by the discrete adjoint.  Equals the fused
    OB_LOSS_CE_HEAD path of grad() (same seed, formed by torch autograd)."""
    ci = make_config("C3").subset(4)
    fld = field_from_config(ci)
    fused = run_config(ci, "store_all", field=fld)
    block = ODEBlock(fld, tableau_catalog("rk4"), 0.0, 1.0, FixedController(10))
    head = torch.as_tensor(ci.extras["head"], dtype=torch.float32, device="cuda")
    Wh = head[:640].reshape(10, 64).clone().requires_grad_(True)
    bh = head[640:].clone().requires_grad_(True)
    labels = torch.as_tensor(ci.extras["labels"], device="cuda")
    u0 = torch.as_tensor(initial_state(ci), dtype=torch.float32, device="cuda").requires_grad_(True)
    uT = block(u0)
    gap = uT.reshape(4, 256, 64).double().mean(dim=1)
    logits = gap @ Wh.double().t() + bh.double()
    loss = torch.nn.functional.cross_entropy(logits, labels)
    loss.backward()
    assert abs(loss.item() - fused.loss) <= 1e-6 * abs(fused.loss)
    assert oc.rel_error(np_(u0.grad), np_(fused.du0)) <= 1e-5
    assert oc.rel_error(np_(block.theta.grad), np_(fused.dtheta)) <= 1e-5
    dh = np.concatenate([np_(Wh.grad).reshape(-1), np_(bh.grad)])
    assert oc.rel_error(dh, np_(fused.dtheta_head)) <= 1e-5


def test_ode_block_autograd_matches_oracle_mlp():
    """A small network: linear -> ODE block (C2 field, tcgen05 tile) -> loss."""
    ci = make_config("C2").subset(32)
    fld = field_from_config(ci)
    block = ODEBlock(fld, tableau_catalog("dopri5"), 0.0, 1.0, FixedController(40),
                     CheckpointPolicy.parse("revolve:8"))
    u0 = torch.as_tensor(ci.u0, dtype=torch.float32, device="cuda").requires_grad_(True)
    uT = block(u0)
    loss = 0.5 * (uT.double() ** 2).sum(dim=1).mean()
    loss.backward()
    mlp = oc.Mlp(ci.widths, ci.activation, ci.theta, ci.time_input)
    ref = oc.grad_terminal(oc.MlpField(mlp), ci.scheme, ci.u0, ci.t0, ci.tF, ci.n_steps, "store_all")
    assert oc.rel_error(np_(u0.grad), ref["du0"]) <= 1e-4
    assert oc.rel_error(np_(block.theta.grad), ref["dtheta"]) <= 1e-4


@pytest.mark.parametrize("tc", [False, True])
def test_device_gradient_explosion_raises(tc):
    """Forward finite, adjoint overflows: f(u) = c^2 u (identity MLP) in fp32; the
    forward grows by ~2.5e20 and the reverse sweep multiplies lambda_N = u_N / B by the
    same factor again, past fp32's range -> the reverse kernel's finiteness check
    (AdjointState.check_finite) raises GradientExplosionError.  tc: the tcgen05 tile's
    reverse_step check (a 16-128-16 field), else the SIMT tile."""
    D, H = (16, 128) if tc else (3, 8)
    spec = MlpSpec((D, H, D), "identity", dtype="f32")
    c = np.sqrt(60.0)
    W1 = np.zeros((H, D))
    W1[:D, :D] = c * np.eye(D)
    W2 = np.zeros((D, H))
    W2[:D, :D] = c * np.eye(D)
    theta = np.concatenate([W1.ravel(), np.zeros(H), W2.ravel(), np.zeros(D)])
    fld = MlpField(MlpModel(spec, theta))
    u0 = np.ones((4, D))
    fwd = forward_pass(fld, tableau_catalog("euler"), u0, 0.0, 1.0, FixedController(100),
                       tensor_cores=tc)
    assert np.all(np.isfinite(fwd.u_final))
    with pytest.raises(GradientExplosionError):
        grad(fld, tableau_catalog("euler"), terminal_loss("half_sqnorm", 1.0), u0, 0.0, 1.0,
             FixedController(100), tensor_cores=tc)
    with pytest.raises(GradientExplosionError):      # host-side check of the terminal state
        backward_sweep(fld, tableau_catalog("euler"), fwd, AdjointState(np.full((4, D), np.inf), None))
