"""GPU tests of the cluster-resident-weights theta kernels (csrc/theta_cluster.cuh): the
fp64 weights of a two-layer MLP / stiff field split over the 8 CTAs of a thread-block
cluster (hidden-unit slices in shared memory, all-gather / reduce-scatter through
distributed shared memory) against the single-CTA theta kernels (theta_impl.cuh, selected
with tensor_cores=False, which keeps every specialised tile off) and the oracle.

Same per-sample algorithm (Newton, GMRES(30) with modified Gram-Schmidt, transposed adjoint
solve); only the operator products are summed in a different order (eight hidden-slice
partials added in rank order), so values agree to fp64 rounding and iteration counts within
a few operator calls.
"""

import dataclasses

import numpy as np
import pytest
import torch

from oracle import core as oc
from paper_2206_01298_b200 import IntegrationError
from paper_2206_01298_b200.configs import make_config
from paper_2206_01298_b200.workloads import field_from_config, run_config

pytestmark = pytest.mark.gpu

TOL64 = 1e-10


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    from paper_2206_01298_b200 import _lib as L
    L.load()


def np_(x):
    return x.detach().cpu().numpy().astype(np.float64) if isinstance(x, torch.Tensor) else np.asarray(x)


@pytest.mark.parametrize("n,tiles,rows", [(16, 8, 2), (37, 24, 2), (250, (120, 128), (3, 2))])
def test_cluster_kernels_match_single_cta_kernels(n, tiles, rows):
    """16 rows = one full cluster; 37 = three clusters of 13 / 12 / 12 rows (CTAs with 2 and 1
    rows); 250 = the one-wave geometry of the C5 bench (15 resident clusters, 16-17 rows
    each, up to 3 per CTA).  Against the single-CTA kernels on the same inputs."""
    ci = make_config("C5").subset(n)
    fld = field_from_config(ci)
    cl = run_config(ci, "store_all", field=fld)
    base = run_config(ci, "store_all", field=fld, tensor_cores=False)
    # (250 rows: 15 resident clusters of 8 on this pool's B200s -> 120 CTAs x 3 rows; 16 -> 128 x 2)
    geo = (cl.device["tiles"], cl.device["tile_rows"])
    assert geo in (list(zip(tiles, rows)) if isinstance(tiles, tuple) else [(tiles, rows)])
    assert base.device["tiles"] * base.device["tile_rows"] >= n and base.device["tiles"] != geo[0]
    for k in ("u_final", "du0", "dtheta"):
        assert oc.rel_error(np_(getattr(cl, k)), np_(getattr(base, k))) <= TOL64, k
    assert abs(cl.loss - base.loss) <= TOL64 * abs(base.loss)
    a, b = cl.sample_counters, base.sample_counters
    for key in ("newton_iters", "steps_accepted"):
        if key in a:
            assert list(a[key]) == list(b[key]), key
    assert np.max(np.abs(np.asarray(a["nfe_forward"]) - np.asarray(b["nfe_forward"]))) <= 8
    assert np.max(np.abs(np.asarray(a["nfe_backward"]) - np.asarray(b["nfe_backward"]))) <= 8


def test_cluster_kernels_match_oracle_and_policies_agree():
    from oracle.problems import run_oracle
    ci = make_config("C5").subset(24)
    fld = field_from_config(ci)
    res = run_config(ci, "store_all", field=fld)
    assert res.device["tiles"] == 16
    ref = run_oracle(ci, "store_all")
    for k in ("u_final", "du0", "dtheta"):
        assert oc.rel_error(np_(getattr(res, k)), ref[k]) <= TOL64, k
    for pol in ("store_solutions", "revolve:4"):
        other = run_config(ci, pol, field=fld)
        assert other.device["tiles"] == 16
        for k in ("u_final", "du0", "dtheta"):
            assert np.array_equal(np_(getattr(other, k)), np_(getattr(res, k))), (pol, k)


def test_backward_euler_and_plain_mlp_field():
    """theta = 1 (no explicit half step in the adjoint) and a plain MlpField (no stiff
    diagonal) go through the same cluster kernels."""
    from paper_2206_01298_b200 import MlpField, MlpModel, MlpSpec
    from paper_2206_01298_b200.workloads import loss_for
    from paper_2206_01298_b200 import grad, tableau_catalog, FixedController, CheckpointPolicy, SolverConfig
    ci = dataclasses.replace(make_config("C5").subset(20), scheme="beuler", n_steps=5)
    fld = field_from_config(ci)
    cl = run_config(ci, "store_all", field=fld)
    base = run_config(ci, "store_all", field=fld, tensor_cores=False)
    assert cl.device["tiles"] == 16
    for k in ("u_final", "du0", "dtheta"):
        assert oc.rel_error(np_(getattr(cl, k)), np_(getattr(base, k))) <= TOL64, k
    rng = np.random.default_rng(3)
    spec = MlpSpec((32, 256, 32), "tanh", False, "f64")
    model = MlpModel(spec, 0.3 * rng.standard_normal(32 * 256 + 256 + 256 * 32 + 32))
    mf = MlpField(model)
    u0 = rng.standard_normal((19, 32))
    from paper_2206_01298_b200.losses import terminal_loss
    args = (mf, tableau_catalog("cn"), terminal_loss("half_sqnorm", 0.5), u0, 0.0, 0.5, FixedController(4),
            CheckpointPolicy.parse("store_all"), SolverConfig())
    a = grad(*args)
    b = grad(*args, tensor_cores=False)
    assert a.device["tiles"] == 16 and b.device["tiles"] != 16
    for k in ("u_final", "du0", "dtheta"):
        assert oc.rel_error(np_(getattr(a, k)), np_(getattr(b, k))) <= TOL64, k


@pytest.mark.timeout(120)
def test_errors_leave_the_cluster_together():
    """A non-finite input row and a Newton solve that cannot converge are voted across the
    cluster: every CTA returns (no CTA is left waiting on a cluster barrier) and the host
    raises the reference's exceptions."""
    from paper_2206_01298_b200 import SolverConfig
    ci = make_config("C5").subset(32)
    fld = field_from_config(ci)
    u0 = ci.u0.copy()
    u0[21, 5] = np.inf
    with pytest.raises(ValueError):
        run_config(ci, "store_all", field=fld, u0=u0)
    ci2 = make_config("C5").subset(32)
    ci2.extras["solver"] = dict(ci2.extras.get("solver") or {}, newton_maxit=1, gmres_maxit=2, gmres_restart=2)
    with pytest.raises(IntegrationError):
        run_config(ci2, "store_all", field=field_from_config(ci2))
    ok = run_config(ci, "store_all", field=fld)     # the device is fine afterwards
    assert np.isfinite(ok.loss)


@pytest.mark.timeout(300)
def test_full_batch_repeated_runs_identical():
    ci = make_config("C5")
    fld = field_from_config(ci)
    first = run_config(ci, "store_all", field=fld)
    assert (first.device["tiles"], first.device["tile_rows"]) in ((120, 3), (128, 2))
    again = run_config(ci, "store_all", field=fld)
    assert again.loss == first.loss
    for k in ("u_final", "du0", "dtheta"):
        assert np.array_equal(np_(getattr(again, k)), np_(getattr(first, k))), k


# ------------------------------------------------------------------ explicit RK on the cluster MLP
@pytest.mark.parametrize("scheme,policy", [("rk4", "store_all"), ("dopri5", "revolve:3"), ("midpoint", "store_solutions")])
def test_explicit_rk_on_cluster_matches_single_cta_kernels(scheme, policy):
    """C1's field (fp64 64-256-64 tanh MLP, no time input) on explicit schemes: the generic RK
    kernels with the cluster MLP adapter (weights resident across a cluster -- two CTAs for this
    shape, parameter cotangents in registers -- rows per CTA sized to one wave of resident
    clusters) against the single-CTA SIMT tile and the oracle."""
    ci = dataclasses.replace(make_config("C1"), scheme=scheme, n_steps=6)
    fld = field_from_config(ci)
    cl = run_config(ci, policy, field=fld)
    base = run_config(ci, policy, field=fld, tensor_cores=False)
    # 64 clusters x 2 CTAs x 4 rows (74 clusters of two are resident)
    assert (cl.device["tiles"], cl.device["tile_rows"]) == (128, 4)
    assert base.device["tile_rows"] == 4 and base.device["tiles"] == 128 and base.device["tensor_cores"] == 0
    assert cl.device["tensor_cores"] == 2
    for k in ("u_final", "du0", "dtheta"):
        assert oc.rel_error(np_(getattr(cl, k)), np_(getattr(base, k))) <= 1e-12, k
    assert abs(cl.loss - base.loss) <= 1e-12 * abs(base.loss)
    assert cl.counters.nfe_forward == base.counters.nfe_forward
    mlp = oc.Mlp(ci.widths, ci.activation, ci.theta, ci.time_input)
    ref = oc.grad_terminal(oc.MlpField(mlp), ci.scheme, ci.u0, ci.t0, ci.tF, ci.n_steps, "store_all")
    for k in ("u_final", "du0", "dtheta"):
        assert oc.rel_error(np_(getattr(cl, k)), ref[k]) <= TOL64, k


def test_explicit_rk_cluster_two_row_tiles_per_cluster():
    """A batch past one wave at 4 rows per CTA: 6 rows per CTA, 12 per cluster of two -- the
    products run over two MMA row tiles (the second half empty) and the register cotangent
    tiles take three k-steps."""
    ci = make_config("C1", batch=800)
    fld = field_from_config(ci)
    cl = run_config(ci, "store_all", field=fld)
    base = run_config(ci, "store_all", field=fld, tensor_cores=False)
    assert cl.device["tensor_cores"] == 2 and cl.device["tile_rows"] == 6
    for k in ("u_final", "du0", "dtheta"):
        assert oc.rel_error(np_(getattr(cl, k)), np_(getattr(base, k))) <= 1e-12, k
    mlp = oc.Mlp(ci.widths, ci.activation, ci.theta, ci.time_input)
    ref = oc.grad_terminal(oc.MlpField(mlp), ci.scheme, ci.u0, ci.t0, ci.tF, ci.n_steps, "store_all")
    for k in ("u_final", "du0", "dtheta"):
        assert oc.rel_error(np_(getattr(cl, k)), ref[k]) <= TOL64, k
    assert abs(cl.loss - ref["loss"]) <= TOL64 * abs(ref["loss"])


@pytest.mark.parametrize("activation", ["relu", "identity"])
def test_explicit_rk_cluster_other_activations_and_uneven_grid(activation):
    """The other activations the cluster MLP accepts, on an uneven step grid (the step size that
    scales the register cotangent tiles changes from step to step), against the SIMT tile."""
    from paper_2206_01298_b200.controls import FixedGridController
    from paper_2206_01298_b200.engine import grad
    from paper_2206_01298_b200.policies import CheckpointPolicy
    from paper_2206_01298_b200.schemes import tableau_catalog
    from paper_2206_01298_b200.workloads import initial_state, loss_for, solver_from_config
    ci = dataclasses.replace(make_config("C1").subset(300), activation=activation)
    fld = field_from_config(ci)
    ctrl = FixedGridController((0.0, 0.07, 0.2, 0.26, 0.55, 0.8, 1.0))
    args = (fld, tableau_catalog("bosh3"), loss_for(ci), initial_state(ci), ci.t0, ci.tF, ctrl,
            CheckpointPolicy.parse("store_all"), solver_from_config(ci))
    cl = grad(*args)
    base = grad(*args, tensor_cores=False)
    assert cl.device["tensor_cores"] == 2 and base.device["tensor_cores"] == 0
    for k in ("u_final", "du0", "dtheta"):
        assert oc.rel_error(np_(getattr(cl, k)), np_(getattr(base, k))) <= 1e-12, k
    assert abs(cl.loss - base.loss) <= 1e-12 * abs(base.loss)


def test_explicit_rk_on_clusters_of_eight():
    """A hidden layer too wide for two CTAs (64-512-64: half of the weights is 256 KB) runs on
    clusters of eight with the parameter cotangents accumulated in the mu slot."""
    import dataclasses as dc
    from paper_2206_01298_b200.configs import xavier_uniform_mlp
    rng = np.random.default_rng(21)
    widths = (64, 512, 64)
    ci = dc.replace(make_config("C1").subset(200), widths=widths, theta=xavier_uniform_mlp(rng, widths), n_steps=4)
    fld = field_from_config(ci)
    cl = run_config(ci, "store_all", field=fld)
    base = run_config(ci, "store_all", field=fld, tensor_cores=False)
    assert cl.device["tensor_cores"] == 2 and cl.device["tiles"] % 8 == 0 and base.device["tensor_cores"] == 0
    for k in ("u_final", "du0", "dtheta"):
        assert oc.rel_error(np_(getattr(cl, k)), np_(getattr(base, k))) <= 1e-12, k
    mlp = oc.Mlp(ci.widths, ci.activation, ci.theta, ci.time_input)
    ref = oc.grad_terminal(oc.MlpField(mlp), ci.scheme, ci.u0, ci.t0, ci.tF, ci.n_steps, "store_all")
    for k in ("u_final", "du0", "dtheta"):
        assert oc.rel_error(np_(getattr(cl, k)), ref[k]) <= TOL64, k


def test_explicit_rk_cluster_ragged_batch_and_bits():
    """A batch that leaves the last cluster partly empty (padding tiles), twice: identical bits."""
    ci = make_config("C1").subset(77)
    fld = field_from_config(ci)
    a = run_config(ci, "store_all", field=fld)
    b = run_config(ci, "store_all", field=fld)
    base = run_config(ci, "store_all", field=fld, tensor_cores=False)
    assert a.device["tiles"] % 2 == 0 and a.device["tiles"] * a.device["tile_rows"] >= 77
    assert a.loss == b.loss
    for k in ("u_final", "du0", "dtheta"):
        assert np.array_equal(np_(getattr(a, k)), np_(getattr(b, k))), k
        assert oc.rel_error(np_(getattr(a, k)), np_(getattr(base, k))) <= 1e-12, k
