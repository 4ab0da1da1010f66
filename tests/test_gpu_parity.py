"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle and the
reference-generated golden fixtures.

Tolerances (north_star): rel_error <= 1e-10 for fp64 configs, <= 1e-4 for fp32
configs (inf-norm relative error, adjoint.py:368-373); the fp32 GPU path is
compared with the fp64 oracle fed the same fp32-rounded inputs.  Checkpoint
policies must agree bit-for-bit on the GPU and the loss must be bit-identical
across runs.
"""

import numpy as np
import pytest
import torch

from oracle import core as oc
from paper_2206_01298_b200 import (CheckpointPolicy, FixedController, GradientExplosionError,
                                   IntegrationError, MlpField, MlpModel, MlpSpec, grad,
                                   tableau_catalog, terminal_loss)
from paper_2206_01298_b200.configs import make_config
from paper_2206_01298_b200.workloads import field_from_config, run_config

pytestmark = pytest.mark.gpu

TOL64 = 1e-10
TOL32 = 1e-4


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    from paper_2206_01298_b200 import _lib as L
    L.load()      # the prebuilt in-tree library; a missing one fails loudly


def oracle_run(ci, policy=None):
    mlp = oc.Mlp(ci.widths, ci.activation, ci.theta, ci.time_input)
    if ci.kind == "stiff":
        fld = oc.StiffField(mlp, ci.extras["diag"], ci.extras["scale"])
        cfg = oc.SolverCfg(**ci.extras["solver"])
    else:
        fld = oc.MlpField(mlp)
        cfg = oc.SolverCfg()
    return oc.grad_terminal(fld, ci.scheme, ci.u0, ci.t0, ci.tF, ci.n_steps,
                            policy or ci.policy, cfg=cfg)


def np_(x):
    return x.detach().cpu().numpy().astype(np.float64) if isinstance(x, torch.Tensor) else x


def assert_close(res, ref, tol):
    errs = {k: oc.rel_error(np_(getattr(res, k)), ref[k]) for k in ("u_final", "du0", "dtheta")}
    errs["loss"] = abs(res.loss - ref["loss"]) / abs(ref["loss"])
    assert max(errs.values()) <= tol, errs
    return errs


# ------------------------------------------------------------------ C1 fp64
def test_c1_full_batch_matches_oracle():
    ci = make_config("C1")
    res = run_config(ci)
    ref = oracle_run(ci)
    assert_close(res, ref, TOL64)
    assert res.counters.nfe_forward == 40 and res.counters.nfe_backward == 40
    assert res.store_counters.stored_states == 9
    assert res.store_counters.stored_stage_vectors == 36


@pytest.mark.parametrize("pol", ["store_solutions", "revolve:3", "revolve:1"])
def test_c1_policies_bit_identical_on_gpu(pol):
    ci = make_config("C1")
    fld = field_from_config(ci)
    u0 = torch.as_tensor(ci.u0, device="cuda")
    base = run_config(ci, "store_all", field=fld, u0=u0)
    other = run_config(ci, pol, field=fld, u0=u0)
    assert torch.equal(base.dtheta, other.dtheta)
    assert torch.equal(base.du0, other.du0)
    assert torch.equal(base.u_final, other.u_final)
    assert base.loss == other.loss


def test_c1_subset_matches_reference_golden(golden):
    g = golden("c1_sub.npz")
    ci = make_config("C1").subset(4)
    for pol in ("store_all", "store_solutions", "revolve:3"):
        res = run_config(ci, pol)
        for k in ("u_final", "du0", "dtheta"):
            assert oc.rel_error(np_(getattr(res, k)), g[f"{pol}/{k}"]) <= TOL64, (pol, k)
        assert res.store_counters.stored_states == g[f"{pol}/stored_states"]
        assert res.store_counters.max_live_slots == g[f"{pol}/max_live_slots"]
        assert res.store_counters.recomputed_steps == g[f"{pol}/recomputed_steps"]
        assert res.counters.nfe_forward == g[f"{pol}/nfe_forward"][0]
        assert res.counters.nfe_backward == g[f"{pol}/nfe_backward"][0]


# ------------------------------------------------------------------ C2 fp32
@pytest.mark.parametrize("pol", ["store_all", "revolve:8"])
def test_c2_subset_matches_reference_golden(golden, pol):
    g = golden("c2_sub.npz")
    ci = make_config("C2").subset(3)
    res = run_config(ci, pol)
    for k in ("u_final", "du0", "dtheta"):
        assert oc.rel_error(np_(getattr(res, k)), g[f"{pol}/{k}"]) <= TOL32, (pol, k)
    assert res.counters.nfe_forward == g[f"{pol}/nfe_forward"][0]
    assert res.counters.nfe_backward == g[f"{pol}/nfe_backward"][0]
    assert res.counters.steps_recomputed == g[f"{pol}/steps_recomputed"][0]
    assert res.store_counters.max_live_slots == g[f"{pol}/max_live_slots"]


def test_c2_full_batch_matches_oracle_and_policies_agree():
    ci = make_config("C2")
    fld = field_from_config(ci)
    u0 = torch.as_tensor(ci.u0, dtype=torch.float32, device="cuda")
    rev = run_config(ci, "revolve:8", field=fld, u0=u0)
    alls = run_config(ci, "store_all", field=fld, u0=u0)
    sol = run_config(ci, "store_solutions", field=fld, u0=u0)
    for other in (alls, sol):
        assert torch.equal(rev.dtheta, other.dtheta)
        assert torch.equal(rev.du0, other.du0)
        assert rev.loss == other.loss
    ref = oracle_run(ci, "store_all")
    assert_close(rev, ref, TOL32)
    assert rev.counters.nfe_forward == 241 + 31 * 7
    assert rev.store_counters.max_live_slots <= 8


def test_loss_bit_reproducible_across_runs():
    ci = make_config("C2", batch=1024)
    fld = field_from_config(ci)
    u0 = torch.as_tensor(ci.u0, dtype=torch.float32, device="cuda")
    runs = [run_config(ci, "revolve:8", field=fld, u0=u0) for _ in range(3)]
    for r in runs[1:]:
        assert r.loss == runs[0].loss
        assert torch.equal(r.dtheta, runs[0].dtheta)
        assert torch.equal(r.du0, runs[0].du0)


def test_batch_shards_sum_to_full_batch():
    """Data-parallel contract: shards with batch_global=B sum to the full call."""
    ci = make_config("C1")
    fld = field_from_config(ci)
    full = run_config(ci, field=fld)
    a = run_config(ci, field=fld, u0=ci.u0[:200], batch_global=ci.batch)
    b = run_config(ci, field=fld, u0=ci.u0[200:], batch_global=ci.batch)
    assert oc.rel_error(a.dtheta + b.dtheta, full.dtheta) <= 1e-13
    assert abs(a.loss + b.loss - full.loss) <= 1e-13 * full.loss
    assert np.array_equal(np.concatenate([a.du0, b.du0]), full.du0)


# ------------------------------------------------------------------ C5 fp64
def test_c5_subset_matches_reference_golden(golden):
    """Stiff Crank-Nicolson, Newton 1e-10 + GMRES(30): values to 1e-10 against
    both reference kernel paths; per-sample NFE within rounding-boundary GMRES
    stops of the reference (whose own numba and numpy paths differ by 1)."""
    g, gn = golden("c5_sub.npz"), golden("c5_sub_numpy.npz")
    ci = make_config("C5").subset(2)
    res = run_config(ci)
    for ref in (g, gn):
        for k in ("u_final", "du0", "dtheta"):
            assert oc.rel_error(np_(getattr(res, k)), ref["store_all/" + k]) <= TOL64, k
        sc = res.sample_counters
        assert np.max(np.abs(sc["nfe_forward"] - ref["store_all/nfe_forward"])) <= 6
        assert np.max(np.abs(sc["nfe_backward"] - ref["store_all/nfe_backward"])) <= 6


def test_c5_batch_matches_oracle_and_policies_agree():
    ci = make_config("C5").subset(8)
    fld = field_from_config(ci)
    u0 = torch.as_tensor(ci.u0, device="cuda")
    base = run_config(ci, "store_all", field=fld, u0=u0)
    for pol in ("revolve:4", "store_solutions"):
        other = run_config(ci, pol, field=fld, u0=u0)
        assert torch.equal(base.dtheta, other.dtheta)
        assert torch.equal(base.du0, other.du0)
        assert base.loss == other.loss
    ref = oracle_run(ci, "store_all")
    assert_close(base, ref, TOL64)
    nf = np.array([s.nfe_forward for s in ref["sample_counters"]])
    nb = np.array([s.nfe_backward for s in ref["sample_counters"]])
    assert np.max(np.abs(base.sample_counters["nfe_forward"] - nf)) <= 6
    assert np.max(np.abs(base.sample_counters["nfe_backward"] - nb)) <= 6
    assert np.all(base.sample_counters["newton_iters"] >= 20)


# ------------------------------------------------------------------ C4 fp32 CNF
def _cnf_oracle(ci, policy="store_all"):
    from oracle.problems import run_oracle
    return run_oracle(ci, policy)


def test_c4_field_protocol_matches_restated_oracle():
    from oracle import fields_ext as ox
    from paper_2206_01298_b200.workloads import initial_state
    ci = make_config("C4").subset(12)
    fld = field_from_config(ci)
    ofl = ox.CnfField(oc.Mlp(ci.widths, ci.activation, ci.theta, True), ci.extras["eps"])
    rng = np.random.default_rng(3)
    Y = initial_state(ci).astype(np.float32).astype(np.float64)
    Y[:, -1] = rng.standard_normal(ci.batch)
    V = rng.standard_normal(Y.shape).astype(np.float32).astype(np.float64)
    f_ref = ofl.eval(Y, 0.4, oc.Counters())
    j_ref, p_ref = ofl.vjp(Y, 0.4, V, oc.Counters())
    f = np_(fld.eval(Y, 0.4))
    j, p = fld.vjp(Y, 0.4, V)
    assert oc.rel_error(f, f_ref) <= TOL32
    assert oc.rel_error(np_(j), j_ref) <= TOL32
    assert oc.rel_error(np_(p), p_ref) <= TOL32


def test_c4_subset_matches_restated_oracle_and_policies_agree():
    ci = make_config("C4").subset(24)
    fld = field_from_config(ci)
    base = run_config(ci, "store_all", field=fld)
    rev = run_config(ci, "revolve:5", field=fld)
    assert np.array_equal(base.dtheta, rev.dtheta) and base.loss == rev.loss
    ref = _cnf_oracle(ci)
    errs = {k: oc.rel_error(np_(getattr(base, k)), ref[k]) for k in ("u_final", "du0", "dtheta")}
    assert max(errs.values()) <= TOL32, errs
    assert abs(base.loss - ref["loss"]) <= TOL32 * abs(ref["loss"])
    assert base.counters.nfe_forward == 121 and base.counters.nfe_backward == 140


# ------------------------------------------------------------------ C3 fp32 conv
def test_c3_field_protocol_matches_restated_oracle():
    from oracle import fields_ext as ox
    ci = make_config("C3").subset(3)
    fld = field_from_config(ci)
    ofl = ox.ConvField(ci.theta)
    rng = np.random.default_rng(9)
    U = ci.u0.reshape(3, -1)
    V = rng.standard_normal(U.shape).astype(np.float32).astype(np.float64)
    f_ref = ofl.eval(U, 0.35, oc.Counters())
    j_ref, p_ref = ofl.vjp(U, 0.35, V, oc.Counters())
    assert oc.rel_error(np_(fld.eval(U, 0.35)), f_ref) <= TOL32
    j, p = fld.vjp(U, 0.35, V)
    assert oc.rel_error(np_(j), j_ref) <= TOL32
    assert oc.rel_error(np_(p), p_ref) <= TOL32


@pytest.mark.parametrize("tensor_cores", [True, False])
def test_c3_subset_matches_restated_oracle_and_policies_agree(tensor_cores):
    """Six images on the tcgen05 conv tile and on the SIMT tile: store_all and revolve:3
    bit-identical; u_final, dtheta, head gradient and loss at the fp32 bar; du0 per image
    at the bar or at a demonstrated ReLU kink of the oracle (tests/_kinks.py)."""
    from _kinks import check_du0_with_kinks
    from oracle import fields_ext as ox
    from oracle.problems import run_oracle
    ci = make_config("C3").subset(6)
    fld = field_from_config(ci)
    base = run_config(ci, "store_all", field=fld, tensor_cores=tensor_cores)
    rev = run_config(ci, "revolve:3", field=fld, tensor_cores=tensor_cores)
    assert base.device["tensor_cores"] == int(tensor_cores)
    assert np.array_equal(base.dtheta, rev.dtheta) and base.loss == rev.loss
    assert np.array_equal(np_(base.du0), np_(rev.du0))
    ref = run_oracle(ci, "store_all")
    errs = {k: oc.rel_error(np_(getattr(base, k)), ref[k]) for k in ("u_final", "dtheta")}
    assert max(errs.values()) <= TOL32, errs
    assert abs(base.loss - ref["loss"]) <= TOL32 * abs(ref["loss"])
    check_du0_with_kinks(lambda: make_config("C3").subset(6), np_(base.du0), ref["du0"], TOL32, max_over=1)
    dhead = ox.head_loss(ref["u_final"], ci.extras["head"], ci.extras["labels"])[2]
    assert oc.rel_error(np_(base.dtheta_head), dhead) <= TOL32
    assert base.counters.nfe_forward == 40 and base.counters.nfe_backward == 40


# ------------------------------------------------- all schemes, policies
EXPLICIT = ("euler", "midpoint", "bosh3", "rk4", "dopri5")
THETA = ("beuler", "cn")


@pytest.mark.parametrize("name", EXPLICIT + THETA)
@pytest.mark.parametrize("pol", ["store_all", "store_solutions", "revolve:3"])
def test_small_schemes_match_reference_golden(golden, name, pol):
    g = golden("small_schemes.npz")
    model = MlpModel(MlpSpec((3, 8, 8, 3), "tanh"), g[f"{name}/theta"])
    res = grad(MlpField(model), tableau_catalog(name), terminal_loss("half_sqnorm", 1.0),
               g[f"{name}/u0"], 0.0, 1.0, FixedController(7), CheckpointPolicy.parse(pol))
    pre = f"{name}/{pol}/"
    # implicit steps: Newton stops at |F| <= 1e-10, so the solution itself is
    # only defined to that level; the GPU must still agree to 1e-9
    tol = TOL64 if name in EXPLICIT else 1e-9
    for k in ("u_final", "du0", "dtheta"):
        assert oc.rel_error(res.__dict__[k], g[pre + k]) <= tol, k
    assert abs(res.loss - float(g[pre + "loss"])) <= 1e-9
    if name in EXPLICIT:
        assert res.counters.nfe_forward == g[pre + "nfe_forward"][0]
        assert res.counters.nfe_backward == g[pre + "nfe_backward"][0]
    else:   # data-dependent: per-sample counts within a rounding-boundary GMRES stop
        sc = res.sample_counters
        assert np.max(np.abs(sc["nfe_forward"] - g[pre + "nfe_forward"])) <= 4
        assert np.max(np.abs(sc["nfe_backward"] - g[pre + "nfe_backward"])) <= 4
    assert res.store_counters.stored_states == g[pre + "stored_states"]
    assert res.store_counters.stored_stage_vectors == g[pre + "stored_stage_vectors"]
    assert res.store_counters.max_live_slots == g[pre + "max_live_slots"]


@pytest.mark.parametrize("act", ["identity", "relu", "tanh", "gelu"])
def test_time_input_activations_match_reference_golden(golden, act):
    g = golden("small_schemes.npz")
    model = MlpModel(MlpSpec((5, 6, 6, 4), act, time_input=True), g[f"act_{act}/theta"])
    res = grad(MlpField(model), tableau_catalog("dopri5"), terminal_loss("half_sqnorm", 1.0),
               g[f"act_{act}/u0"], 0.0, 1.0, FixedController(5))
    for k in ("u_final", "du0", "dtheta"):
        assert oc.rel_error(res.__dict__[k], g[f"act_{act}/{k}"]) <= TOL64, k


@pytest.mark.parametrize("act", ["identity", "relu", "tanh", "gelu"])
def test_field_protocol_matches_reference_kernels(golden, act):
    g = golden("mlp_kernels.npz")
    fld = MlpField(MlpModel(MlpSpec((6, 7, 7, 5), act, time_input=True), g[f"{act}/theta"]))
    for b in range(4):
        U = g[f"{act}/U"][b:b + 1]
        t = float(g[f"{act}/t"][b])
        f = np_(fld.eval(U, t))[0]
        jtv, ptv = fld.vjp(U, t, g[f"{act}/V"][b:b + 1])
        jv = np_(fld.jvp(U, t, g[f"{act}/W"][b:b + 1]))[0]
        ju = np_(fld.vjp_u(U, t, g[f"{act}/V"][b:b + 1]))[0]
        assert np.max(np.abs(f - g[f"{act}/f"][b])) <= 1e-13
        assert np.max(np.abs(np_(jtv)[0] - g[f"{act}/jtv"][b])) <= 1e-13
        assert np.max(np.abs(ju - g[f"{act}/jtv"][b])) <= 1e-13
        assert np.max(np.abs(np_(ptv) - g[f"{act}/ptv"][b])) <= 1e-13
        assert np.max(np.abs(jv - g[f"{act}/jv"][b])) <= 1e-13


def test_adjoint_identity_on_device():
    """<v, J w> == <J^T v, w> per sample (test_acceptance.py:242-256)."""
    ci = make_config("C1", batch=64)
    fld = field_from_config(ci)
    rng = np.random.default_rng(0)
    V = rng.standard_normal((64, 64))
    W = rng.standard_normal((64, 64))
    jw = np_(fld.jvp(ci.u0, 0.3, W))
    jtv = np_(fld.vjp_u(ci.u0, 0.3, V))
    lhs = np.sum(V * jw, axis=1)
    rhs = np.sum(jtv * W, axis=1)
    assert np.max(np.abs(lhs - rhs) / np.maximum(1.0, np.abs(lhs))) <= 1e-12


# ------------------------------------------------------------- errors
def test_non_finite_input_raises_value_error():
    ci = make_config("C1", batch=8)
    u0 = ci.u0.copy()
    u0[3, 5] = np.nan
    with pytest.raises(ValueError):
        run_config(ci, u0=u0)


def test_overflow_raises_integration_error():
    spec = MlpSpec((2, 4, 2), "identity", dtype="f32")
    theta = np.full(spec.n_params, 1e3)
    with pytest.raises(IntegrationError, match="overflowed"):
        grad(MlpField(MlpModel(spec, theta)), tableau_catalog("euler"),
             terminal_loss("half_sqnorm", 10.0), np.ones((3, 2)), 0.0, 10.0, FixedController(10))


def test_gradient_explosion_error_class_exists():
    assert issubclass(GradientExplosionError, RuntimeError)
