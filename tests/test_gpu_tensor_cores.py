"""GPU parity of the tcgen05 tensor-core MLP tile (csrc/tc_mlp.cuh).

fp32 two-layer MLP fields on explicit fixed-step schemes run their
contractions on the 5th-gen tensor cores as a 3-pass bf16 split (A_hi B_hi +
A_hi B_lo + A_lo B_hi, fp32 accumulation in TMEM).  The bar is the fp32 one of
north_star: rel_error <= 1e-4 (inf-norm relative, adjoint.py:368-373) against
the fp64 oracle fed the same fp32-rounded inputs, for every shape, activation,
scheme and checkpoint policy the tile accepts, with ragged and single-sample
batches; the SIMT tile (tensor_cores=False) is held to the same bar, and
shapes the tile does not take must fall back to the SIMT tile.  ReLU stays on
the SIMT tile: its derivative jumps at 0, and the split products move
pre-activations near 0 across the jump often enough to cost ~4e-4 on du0.
"""

import numpy as np
import pytest
import torch

from oracle import core as oc
from paper_2206_01298_b200 import (CheckpointPolicy, FixedController, MlpField, MlpModel, MlpSpec,
                                   grad, tableau_catalog, terminal_loss)
from paper_2206_01298_b200.configs import make_config
from paper_2206_01298_b200.workloads import field_from_config, run_config

pytestmark = pytest.mark.gpu
TOL32 = 1e-4


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    from paper_2206_01298_b200 import _lib as L
    L.load()


def np_(x):
    return x.detach().cpu().numpy().astype(np.float64) if isinstance(x, torch.Tensor) else x


def f32(x):
    return np.asarray(x, np.float32).astype(np.float64)


def make_mlp(rng, n, hidden, act, time_input):
    widths = (n + int(time_input), hidden, n)
    parts = []
    for l in range(2):
        b = np.sqrt(6.0 / (widths[l] + widths[l + 1]))
        parts += [rng.uniform(-b, b, widths[l + 1] * widths[l]), rng.normal(0, 0.1, widths[l + 1])]
    return widths, f32(np.concatenate(parts))


def run_both(widths, act, time_input, theta, u0, scheme, n_steps, policy, tc=True):
    model = MlpModel(MlpSpec(widths, act, time_input=time_input, dtype="f32"), theta)
    fld = MlpField(model)
    res = grad(fld, tableau_catalog(scheme), terminal_loss("half_sqnorm", 1.0),
               torch.as_tensor(u0, dtype=torch.float32, device="cuda"), 0.0, 1.0,
               FixedController(n_steps), CheckpointPolicy.parse(policy), tensor_cores=tc)
    ref = oc.grad_terminal(oc.MlpField(oc.Mlp(widths, act, theta, time_input)), scheme, u0, 0.0, 1.0,
                           n_steps, policy)
    return res, ref


def errs(res, ref):
    e = {k: oc.rel_error(np_(getattr(res, k)), ref[k]) for k in ("u_final", "du0", "dtheta")}
    e["loss"] = abs(res.loss - ref["loss"]) / abs(ref["loss"])
    return e


def test_c2_full_batch_on_tensor_cores_matches_oracle_and_simt():
    ci = make_config("C2")
    fld = field_from_config(ci)
    u0 = torch.as_tensor(ci.u0, dtype=torch.float32, device="cuda")
    tc = run_config(ci, "revolve:8", field=fld, u0=u0)
    simt = run_config(ci, "revolve:8", field=fld, u0=u0, tensor_cores=False)
    assert tc.device["tensor_cores"] == 1 and simt.device["tensor_cores"] == 0
    mlp = oc.Mlp(ci.widths, ci.activation, ci.theta, ci.time_input)
    ref = oc.grad_terminal(oc.MlpField(mlp), ci.scheme, ci.u0, ci.t0, ci.tF, ci.n_steps, "store_all")
    e_tc, e_simt = errs(tc, ref), errs(simt, ref)
    assert max(e_tc.values()) <= TOL32, e_tc
    assert max(e_simt.values()) <= TOL32, e_simt
    assert tc.counters.nfe_forward == 241 + 31 * 7 and tc.counters.nfe_backward == 280


def test_c2_policies_bit_identical_on_tensor_cores():
    ci = make_config("C2", batch=600)
    fld = field_from_config(ci)
    u0 = torch.as_tensor(ci.u0, dtype=torch.float32, device="cuda")
    runs = [run_config(ci, pol, field=fld, u0=u0) for pol in ("revolve:8", "store_all",
                                                               "store_solutions", "revolve:8")]
    for r in runs[1:]:
        assert r.device["tensor_cores"] == 1
        assert torch.equal(r.dtheta, runs[0].dtheta)
        assert torch.equal(r.du0, runs[0].du0)
        assert r.loss == runs[0].loss


@pytest.mark.parametrize("n,hidden,act,time_input", [
    (64, 256, "tanh", True), (64, 128, "tanh", False), (32, 256, "tanh", True),
    (16, 128, "identity", True), (48, 256, "tanh", False)])
@pytest.mark.parametrize("batch", [1, 37, 333])
def test_shapes_activations_ragged_batches(n, hidden, act, time_input, batch):
    rng = np.random.default_rng(1000 + n + hidden + batch)
    widths, theta = make_mlp(rng, n, hidden, act, time_input)
    u0 = f32(rng.normal(size=(batch, n)))
    res, ref = run_both(widths, act, time_input, theta, u0, "dopri5", 6, "store_all")
    assert res.device["tensor_cores"] == 1
    e = errs(res, ref)
    assert max(e.values()) <= TOL32, e


@pytest.mark.parametrize("scheme", ["euler", "midpoint", "bosh3", "rk4", "dopri5"])
@pytest.mark.parametrize("policy", ["store_all", "store_solutions", "revolve:3"])
def test_schemes_and_policies_on_tensor_cores(scheme, policy):
    rng = np.random.default_rng(7)
    widths, theta = make_mlp(rng, 64, 256, "tanh", True)
    u0 = f32(rng.normal(size=(300, 64)))
    res, ref = run_both(widths, "tanh", True, theta, u0, scheme, 9, policy)
    assert res.device["tensor_cores"] == 1
    e = errs(res, ref)
    assert max(e.values()) <= TOL32, e
    assert res.counters.nfe_forward == ref["counters"].nfe_forward
    assert res.counters.nfe_backward == ref["counters"].nfe_backward


def test_ineligible_shapes_fall_back_to_simt():
    rng = np.random.default_rng(3)
    for n, hidden, act in ((64, 256, "gelu"), (64, 256, "relu"), (64, 200, "tanh"), (100, 256, "tanh")):
        widths, theta = make_mlp(rng, n, hidden, act, True)
        u0 = f32(rng.normal(size=(40, n)))
        res, ref = run_both(widths, act, True, theta, u0, "rk4", 4, "store_all")
        assert res.device["tensor_cores"] == 0, (n, hidden, act)
        e = errs(res, ref)
        assert max(e.values()) <= TOL32, e


@pytest.mark.parametrize("kind,scaled", [("mse", False), ("mae", True)])
def test_observation_losses_on_tensor_cores(kind, scaled):
    """Observation seeds injected between reversed steps (adjoint.py:235-253) with the
    tensor-core tile's h-prescaled VJP and TMEM-resident parameter cotangent."""
    from oracle import obs_losses as ol
    from paper_2206_01298_b200.losses import LossSpec, MinMaxScaling
    rng = np.random.default_rng(11)
    widths, theta = make_mlp(rng, 64, 256, "tanh", True)
    B, n_steps = 200, 8
    u0 = f32(rng.normal(size=(B, 64)))
    times = (0.25, 0.5, 1.0)
    vals = [f32(rng.normal(size=(B, 64))) for _ in times]
    lo = hi = None
    if scaled:
        lo, hi = f32(rng.uniform(-2, -1, 64)), f32(rng.uniform(1, 2, 64))
        hi[3] = lo[3]   # a degenerate component passes through (losses.py:27-33)
    loss = LossSpec(kind, times, tuple(vals), MinMaxScaling(lo, hi) if scaled else None)
    model = MlpModel(MlpSpec(widths, "tanh", time_input=True, dtype="f32"), theta)
    res = grad(MlpField(model), tableau_catalog("dopri5"), loss,
               torch.as_tensor(u0, dtype=torch.float32, device="cuda"), 0.0, 1.0,
               FixedController(n_steps), CheckpointPolicy.parse("revolve:3"))
    assert res.device["tensor_cores"] == 1
    obs = ol.ObsLoss(kind, ol.match_boundaries(times, np.linspace(0, 1, n_steps + 1)),
                     np.stack(vals), ol.MinMax(lo, hi) if scaled else None)
    ref = oc.grad_terminal(oc.MlpField(oc.Mlp(widths, "tanh", theta, True)), "dopri5", u0, 0.0, 1.0,
                           n_steps, "revolve:3", obs=obs)
    assert abs(res.loss - ref["loss"]) <= 1e-4 * abs(ref["loss"])
    assert oc.rel_error(np_(res.dtheta), ref["dtheta"]) <= TOL32
    assert oc.rel_error(np_(res.du0), ref["du0"]) <= TOL32
    assert oc.rel_error(np.stack([np_(p) for p in res.predictions]), np.stack(ref["predictions"])) <= TOL32


def test_mse_target_loss_on_tensor_cores():
    rng = np.random.default_rng(5)
    widths, theta = make_mlp(rng, 32, 128, "tanh", False)
    u0 = f32(rng.normal(size=(150, 32)))
    target = f32(rng.normal(size=(150, 32)))
    model = MlpModel(MlpSpec(widths, "tanh", time_input=False, dtype="f32"), theta)
    res = grad(MlpField(model), tableau_catalog("rk4"), terminal_loss("mse", 1.0, target),
               torch.as_tensor(u0, dtype=torch.float32, device="cuda"), 0.0, 1.0,
               FixedController(10), CheckpointPolicy.parse("store_all"))
    res64 = grad(MlpField(MlpModel(MlpSpec(widths, "tanh", time_input=False), theta)),
                 tableau_catalog("rk4"), terminal_loss("mse", 1.0, target), u0, 0.0, 1.0,
                 FixedController(10), CheckpointPolicy.parse("store_all"))
    assert res.device["tensor_cores"] == 1 and res64.device["tensor_cores"] != 1   # (fp64: SIMT or cluster MLP)
    assert abs(res.loss - res64.loss) <= 1e-4 * abs(res64.loss)
    assert oc.rel_error(np_(res.dtheta), np_(res64.dtheta)) <= TOL32
    assert oc.rel_error(np_(res.du0), np_(res64.du0)) <= TOL32


@pytest.mark.parametrize("scheme,n_steps", [("dopri5", 1), ("bosh3", 1), ("dopri5", 2)])
def test_fsal_edges_on_tensor_cores(scheme, n_steps):
    """FSAL carry and the skipped unused last stage at the sweep's edges (one and two
    steps), revolve with a single slot."""
    rng = np.random.default_rng(21 + n_steps)
    widths, theta = make_mlp(rng, 64, 256, "tanh", True)
    u0 = f32(rng.normal(size=(90, 64)))
    for pol in ("store_all", "revolve:1"):
        res, ref = run_both(widths, "tanh", True, theta, u0, scheme, n_steps, pol)
        assert res.device["tensor_cores"] == 1
        e = errs(res, ref)
        assert max(e.values()) <= TOL32, (pol, e)
        assert res.counters.nfe_forward == ref["counters"].nfe_forward


def test_nonuniform_grid_on_tensor_cores():
    from paper_2206_01298_b200 import FixedGridController
    rng = np.random.default_rng(8)
    widths, theta = make_mlp(rng, 48, 128, "tanh", True)
    u0 = f32(rng.normal(size=(120, 48)))
    times = (0.0, 0.05, 0.2, 0.3, 0.65, 1.0)
    model = MlpModel(MlpSpec(widths, "tanh", time_input=True, dtype="f32"), theta)
    res = grad(MlpField(model), tableau_catalog("dopri5"), terminal_loss("half_sqnorm", 1.0),
               torch.as_tensor(u0, dtype=torch.float32, device="cuda"), 0.0, 1.0,
               FixedGridController(times), CheckpointPolicy.parse("revolve:2"))
    assert res.device["tensor_cores"] == 1
    ref = oc.grad_terminal(oc.MlpField(oc.Mlp(widths, "tanh", theta, True)), "dopri5", u0, 0.0, 1.0,
                           len(times) - 1, "revolve:2", times=np.array(times))
    e = errs(res, ref)
    assert max(e.values()) <= TOL32, e


def test_batch_shards_sum_to_full_batch_on_tensor_cores():
    """Data-parallel contract on the tensor-core tile: shards with batch_global = B sum to
    the full call (deterministic per-CTA slots, fixed-order reduction)."""
    ci = make_config("C2", batch=700)
    fld = field_from_config(ci)
    full = run_config(ci, "revolve:8", field=fld)
    a = run_config(ci, "revolve:8", field=fld, u0=ci.u0[:300], batch_global=ci.batch)
    b = run_config(ci, "revolve:8", field=fld, u0=ci.u0[300:], batch_global=ci.batch)
    assert full.device["tensor_cores"] == 1 and a.device["tensor_cores"] == 1
    assert oc.rel_error(np_(a.dtheta) + np_(b.dtheta), np_(full.dtheta)) <= 1e-5
    assert abs(a.loss + b.loss - full.loss) <= 1e-6 * abs(full.loss)
    assert oc.rel_error(np.concatenate([np_(a.du0), np_(b.du0)]), np_(full.du0)) <= 1e-6


def test_overflow_and_bad_input_on_tensor_cores():
    from paper_2206_01298_b200 import IntegrationError
    rng = np.random.default_rng(9)
    widths, theta = make_mlp(rng, 64, 256, "identity", True)
    model = MlpModel(MlpSpec(widths, "identity", time_input=True, dtype="f32"), theta * 40.0)
    u0 = f32(rng.normal(size=(50, 64)))
    with pytest.raises(IntegrationError):
        grad(MlpField(model), tableau_catalog("rk4"), terminal_loss("half_sqnorm", 1.0),
             torch.as_tensor(u0, dtype=torch.float32, device="cuda"), 0.0, 1.0, FixedController(30),
             CheckpointPolicy.parse("store_all"))
    bad = u0.copy()
    bad[3, 5] = np.nan
    model = MlpModel(MlpSpec(widths, "identity", time_input=True, dtype="f32"), theta)
    with pytest.raises(ValueError):
        grad(MlpField(model), tableau_catalog("rk4"), terminal_loss("half_sqnorm", 1.0),
             torch.as_tensor(bad, dtype=torch.float32, device="cuda"), 0.0, 1.0, FixedController(3),
             CheckpointPolicy.parse("store_all"))


def test_plan_cache_distinguishes_problems():
    """The host plan is reused only for an identical problem (struct and host arrays):
    alternating grids / batches / policies must reproduce fresh results exactly."""
    from paper_2206_01298_b200 import FixedGridController
    rng = np.random.default_rng(13)
    widths, theta = make_mlp(rng, 64, 256, "tanh", True)
    model = MlpModel(MlpSpec(widths, "tanh", time_input=True, dtype="f32"), theta)
    fld = MlpField(model)
    u0 = torch.as_tensor(f32(rng.normal(size=(64, 64))), dtype=torch.float32, device="cuda")

    def run(times, pol, rows):
        return grad(fld, tableau_catalog("dopri5"), terminal_loss("half_sqnorm", 1.0), u0[:rows],
                    0.0, 1.0, FixedGridController(times), CheckpointPolicy.parse(pol))

    ga, gb = (0.0, 0.25, 0.5, 1.0), (0.0, 0.5, 0.75, 1.0)   # same step count, other times
    first = [run(ga, "store_all", 64), run(gb, "store_all", 64), run(ga, "revolve:1", 40)]
    again = [run(ga, "revolve:1", 40), run(gb, "store_all", 64), run(ga, "store_all", 64)][::-1]
    for x, y in zip(first, again):
        assert torch.equal(x.dtheta, y.dtheta) and torch.equal(x.du0, y.du0) and x.loss == y.loss
    assert not torch.equal(first[0].dtheta, first[1].dtheta)
