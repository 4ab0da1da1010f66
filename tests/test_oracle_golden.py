"""Pin the CPU oracle (oracle/) against the reference's own outputs.

The fixtures in tests/golden/ were produced by running the reference odegrad
package itself (tools/make_golden.py); the known-answer values below are the
reference test-suite's own (pkg/tests/*.py, cited per test).
"""

import numpy as np
import pytest

from oracle import core as oc
from oracle import revolve as orv
from paper_2206_01298_b200 import configs

TOL = 1e-12   # batching changes BLAS blocking / batch-sum order only


def test_revolve_counts_match_reference(golden):
    g = golden("revolve.npz")
    for nt in range(1, 61):
        for nc in range(1, 21):
            assert orv.revolve_count(nt, nc) == g["counts"][nt, nc]
            assert orv.dp_optimal_count(nt, nc) == g["counts"][nt, nc]


def test_revolve_schedules_match_reference(golden):
    g = golden("revolve.npz")
    kinds = {"advance": 0, "store": 1, "restore": 2, "reverse": 3}
    for key, arr in g.items():
        if not key.startswith("sched_"):
            continue
        _, nt, nc = key.split("_")
        acts = orv.revolve_schedule(int(nt), int(nc))
        mine = np.array([[kinds[k], s, a, b] for k, s, a, b in acts], np.int64)
        assert np.array_equal(mine, arr), key


def test_revolve_spot_values_and_audit():
    # pkg/tests/test_checkpointing.py:24-33, test_acceptance.py:110-128
    assert orv.revolve_count(10, 3) == 6
    assert orv.revolve_count(4, 1) == 3
    assert orv.revolve_count(5, 4) == 0
    for nt in range(1, 30):
        for nc in range(1, 10):
            extra, live = orv.audit(nt, nc)
            assert extra == orv.revolve_count(nt, nc)
            assert live <= nc


def test_mlp_kernels_match_reference(golden):
    g = golden("mlp_kernels.npz")
    for act in ("identity", "relu", "tanh", "gelu"):
        mlp = oc.Mlp((6, 7, 7, 5), act, g[f"{act}/theta"], time_input=True)
        fld = oc.MlpField(mlp)
        c = oc.Counters()
        for b in range(4):
            U = g[f"{act}/U"][b:b + 1]
            t = g[f"{act}/t"][b]
            f = fld.eval(U, t, c)
            jtv, ptv = fld.vjp(U, t, g[f"{act}/V"][b:b + 1], c)
            jv = fld.jvp(U, t, g[f"{act}/W"][b:b + 1], c)
            assert np.max(np.abs(f[0] - g[f"{act}/f"][b])) <= 1e-14
            assert np.max(np.abs(jtv[0] - g[f"{act}/jtv"][b])) <= 1e-14
            assert np.max(np.abs(ptv - g[f"{act}/ptv"][b])) <= 1e-14
            assert np.max(np.abs(jv[0] - g[f"{act}/jv"][b])) <= 1e-14


def _check(res, g, prefix, tol=TOL):
    assert oc.rel_error(res["u_final"], g[prefix + "u_final"]) <= tol
    assert oc.rel_error(res["du0"], g[prefix + "du0"]) <= tol
    assert oc.rel_error(res["dtheta"], g[prefix + "dtheta"]) <= tol
    assert abs(res["loss"] - float(g[prefix + "loss"])) <= tol * max(1.0, abs(res["loss"]))
    nf = [s.nfe_forward for s in res["sample_counters"]]
    nb = [s.nfe_backward for s in res["sample_counters"]]
    assert nf == list(g[prefix + "nfe_forward"])
    assert nb == list(g[prefix + "nfe_backward"])
    assert res["store"].stored_states == g[prefix + "stored_states"]
    assert res["store"].stored_stage_vectors == g[prefix + "stored_stage_vectors"]
    assert res["store"].max_live_slots == g[prefix + "max_live_slots"]
    assert res["store"].recomputed_steps == g[prefix + "recomputed_steps"]


SCHEMES = ("euler", "midpoint", "bosh3", "rk4", "dopri5", "beuler", "cn")


@pytest.mark.parametrize("name", SCHEMES)
@pytest.mark.parametrize("pol", ["store_all", "store_solutions", "revolve:3"])
def test_small_schemes_match_reference(golden, name, pol):
    g = golden("small_schemes.npz")
    mlp = oc.Mlp((3, 8, 8, 3), "tanh", g[f"{name}/theta"])
    res = oc.grad_terminal(oc.MlpField(mlp), name, g[f"{name}/u0"], 0.0, 1.0, 7, pol)
    _check(res, g, f"{name}/{pol}/", tol=1e-11 if name in ("beuler", "cn") else TOL)


@pytest.mark.parametrize("act", ["identity", "relu", "tanh", "gelu"])
def test_time_input_activations_match_reference(golden, act):
    g = golden("small_schemes.npz")
    mlp = oc.Mlp((5, 6, 6, 4), act, g[f"act_{act}/theta"], time_input=True)
    res = oc.grad_terminal(oc.MlpField(mlp), "dopri5", g[f"act_{act}/u0"], 0.0, 1.0, 5)
    _check(res, g, f"act_{act}/")


@pytest.mark.parametrize("pol", ["store_all", "store_solutions", "revolve:3"])
def test_c1_subset_matches_reference(golden, pol):
    g = golden("c1_sub.npz")
    ci = configs.make_config("C1").subset(4)
    assert np.array_equal(ci.u0, g["u0"])
    assert float(np.sum(ci.theta * np.arange(1, ci.theta.size + 1))) == float(g["theta_checksum"])
    fld = oc.MlpField(oc.Mlp(ci.widths, ci.activation, ci.theta, ci.time_input))
    res = oc.grad_terminal(fld, ci.scheme, ci.u0, ci.t0, ci.tF, ci.n_steps, pol)
    _check(res, g, f"{pol}/")


@pytest.mark.parametrize("pol", ["store_all", "revolve:8"])
def test_c2_subset_matches_reference(golden, pol):
    g = golden("c2_sub.npz")
    ci = configs.make_config("C2").subset(3)
    assert np.array_equal(ci.u0, g["u0"])
    fld = oc.MlpField(oc.Mlp(ci.widths, ci.activation, ci.theta, ci.time_input))
    res = oc.grad_terminal(fld, ci.scheme, ci.u0, ci.t0, ci.tF, ci.n_steps, pol)
    _check(res, g, f"{pol}/")


def test_c5_subset_matches_reference(golden):
    """Values match both reference kernel paths to 1e-10.  Counters match the
    reference's numpy path exactly (same ufuncs); against its numba path they
    may differ by a rounding-boundary GMRES stop (+-1 per solve), exactly as the
    reference's two paths differ from each other."""
    g = golden("c5_sub_numpy.npz")
    gn = golden("c5_sub.npz")
    ci = configs.make_config("C5").subset(2)
    assert np.array_equal(ci.u0, g["u0"])
    fld = oc.StiffField(oc.Mlp(ci.widths, ci.activation, ci.theta), ci.extras["diag"],
                        ci.extras["scale"])
    res = oc.grad_terminal(fld, ci.scheme, ci.u0, ci.t0, ci.tF, ci.n_steps, "store_all",
                           cfg=oc.SolverCfg(**ci.extras["solver"]))
    _check(res, g, "store_all/", tol=1e-10)
    for k in ("u_final", "du0", "dtheta"):
        assert oc.rel_error(res[k], gn["store_all/" + k]) <= 1e-10
    nf = np.array([s.nfe_forward for s in res["sample_counters"]])
    assert np.max(np.abs(nf - gn["store_all/nfe_forward"])) <= 2


# --- reference known-answer tests restated against the oracle -------------

class _Lin:
    """u' = k*u field with closed-form products (pkg/tests/test_integrators.py:19-21)."""

    def __init__(self, k):
        self.k = k
        self.n_params = 0

    def eval(self, U, t, c):
        c.nfe_forward += 1
        return self.k * U

    def jvp(self, U, t, W, c):
        c.nfe_forward += 1
        return self.k * W

    def vjp(self, U, t, V, c):
        c.nfe_backward += 1
        return self.k * V, np.zeros(0)

    def vjp_u(self, U, t, V, c):
        c.nfe_backward += 1
        return self.k * V


def test_kat_single_steps():
    # pkg/tests/test_integrators.py:24-64
    c = oc.Counters()
    rec, _ = oc.rk_step(oc.explicit_tableau("euler"), _Lin(1.0), np.array([[1.0]]), 0.0, 0.1, c)
    assert abs(rec.u_next[0, 0] - 1.1) <= 1e-15
    rec, _ = oc.rk_step(oc.explicit_tableau("rk4"), _Lin(1.0), np.array([[1.0]]), 0.0, 0.1, c)
    assert abs(rec.u_next[0, 0] - 1.1051708333) <= 1e-10
    rec = oc.theta_step(1.0, _Lin(1.0), np.array([[1.0]]), 0.0, 0.5, oc.SolverCfg(), c)
    assert abs(rec.u_next[0, 0] - 2.0) <= 1e-9
    rec = oc.theta_step(0.5, _Lin(-1000.0), np.array([[1.0]]), 0.0, 0.1, oc.SolverCfg(), c)
    assert abs(rec.u_next[0, 0] - (-49.0 / 51.0)) <= 1e-9


def test_kat_fsal_counts():
    # pkg/tests/test_integrators.py:96-108
    for name, per, extra in (("dopri5", 6, 1), ("rk4", 4, 0), ("bosh3", 3, 1)):
        res = oc.grad_terminal(_Lin(1.0), name, np.array([[1.0]]), 0.0, 1.0, 10)
        assert res["counters"].nfe_forward == per * 10 + extra


def test_kat_rk4_global_error():
    # pkg/tests/test_integrators.py:86-93
    res = oc.grad_terminal(_Lin(1.0), "rk4", np.array([[1.0]]), 0.0, 1.0, 20)
    err = abs(res["u_final"][0, 0] - np.e)
    assert abs(err - 1.358e-7) <= 0.01e-7


def test_kat_transpose_dense_all_schemes():
    # pkg/tests/test_acceptance.py:242-291: forward step matrix == adjoint^T
    rng = np.random.default_rng(123)
    A = rng.standard_normal((3, 3)) * 0.5

    class LinA:
        n_params = 0

        def eval(self, U, t, c):
            c.nfe_forward += 1
            return U @ A.T

        def jvp(self, U, t, W, c):
            c.nfe_forward += 1
            return W @ A.T

        def vjp(self, U, t, V, c):
            c.nfe_backward += 1
            return V @ A, np.zeros(0)

        def vjp_u(self, U, t, V, c):
            c.nfe_backward += 1
            return V @ A

    cfg = oc.SolverCfg(newton_tol=1e-14, gmres_tol=5e-16, newton_maxit=100)
    for name in SCHEMES:
        sch = oc.scheme(name)
        E = np.eye(3)
        c = oc.Counters()
        if sch.kind == "rk":
            fwd = oc.rk_step(sch.tab, LinA(), E, 0.0, 0.2, c)[0].u_next.T
            rec0 = oc.rk_step(sch.tab, LinA(), np.zeros((3, 3)), 0.0, 0.2, c)[0]
            adj, _ = oc.rk_adjoint_step(sch.tab, LinA(), rec0, E, np.zeros(0), c)
        else:
            fwd = oc.theta_step(sch.theta, LinA(), E, 0.0, 0.2, cfg, c).u_next.T
            rec0 = oc.theta_step(sch.theta, LinA(), np.zeros((3, 3)), 0.0, 0.2, cfg, c)
            adj, _ = oc.theta_adjoint_step(sch.theta, LinA(), rec0, E, np.zeros(0), cfg, c)
        assert np.max(np.abs(adj.T - fwd.T)) <= 1e-12, name


def test_kat_gmres():
    # pkg/tests/test_linalg.py:7-62
    cfg = oc.SolverCfg()
    x, it = oc.gmres(lambda v: v, np.array([1.0, -2.0, 3.0]), cfg)
    assert np.allclose(x, [1.0, -2.0, 3.0], atol=1e-14) and it <= 1
    x, it = oc.gmres(lambda v: 2 * v, np.zeros(4), cfg)
    assert it == 0 and not np.any(x)
    rng = np.random.default_rng(3)
    m = rng.standard_normal((40, 40))
    a = m @ m.T + 0.05 * np.eye(40)
    with pytest.raises(oc.ConvergenceError):
        oc.gmres(lambda v: a @ v, rng.standard_normal(40),
                 oc.SolverCfg(gmres_maxit=2, gmres_restart=2))


OBS_CASES = ("mse_rk4", "mae_dopri5", "mse_cn", "mae_rk4_tF")


def obs_case(g, name):
    """Oracle ObsLoss + field for one obs_losses.npz case (reference grad() per sample)."""
    from oracle import obs_losses as ol
    kind, sch, pol, tin = (str(x) for x in g[f"{name}/meta"])
    tin = tin == "1"
    N = g[f"{name}/u0"].shape[1]
    mlp = oc.Mlp((N + int(tin), 8, 8, N), "tanh", g[f"{name}/theta"], time_input=tin)
    ts = np.linspace(0.0, 1.0, 9)
    steps = ol.match_boundaries(g[f"{name}/times"], ts)
    scaling = ol.MinMax(g[f"{name}/lo"], g[f"{name}/hi"]) if f"{name}/lo" in g else None
    return mlp, sch, pol, ol.ObsLoss(kind, steps, g[f"{name}/values"], scaling)


@pytest.mark.parametrize("name", OBS_CASES)
def test_observation_losses_match_reference(golden, name):
    g = golden("obs_losses.npz")
    mlp, sch, pol, obs = obs_case(g, name)
    res = oc.grad_terminal(oc.MlpField(mlp), sch, g[f"{name}/u0"], 0.0, 1.0, 8, pol, obs=obs)
    assert abs(res["loss"] - float(g[f"{name}/loss"])) <= 1e-12 * max(1.0, abs(float(g[f"{name}/loss"])))
    assert oc.rel_error(res["predictions"], g[f"{name}/predictions"]) < 1e-12
    assert oc.rel_error(res["dtheta"], g[f"{name}/dtheta"]) < 1e-10
    assert oc.rel_error(res["du0"], g[f"{name}/du0"]) < 1e-10


def test_observation_alignment_and_scaling_rules():
    from oracle import obs_losses as ol
    ts = np.linspace(0.0, 1.0, 5)
    assert ol.match_boundaries([0.0, 0.5, 1.0], ts) == [0, 2, 4]
    with pytest.raises(ValueError):
        ol.match_boundaries([0.3], ts)
    sc = ol.MinMax([0.0, 1.0], [2.0, 1.0])        # second component degenerate
    np.testing.assert_allclose(sc.apply(np.array([1.0, 5.0])), [0.5, 5.0])
    np.testing.assert_allclose(sc.chain(np.array([1.0, 1.0])), [0.5, 1.0])


ADAPTIVE_CASES = ("dopri5_term", "bosh3_obs", "dopri5_obs0")


def adaptive_case(g, name):
    """Oracle field / ctrl / ObsLoss for one adaptive.npz case (reference grad per sample)."""
    from oracle import adaptive as oa
    from oracle import obs_losses as ol
    sch, kind, pol = (str(x) for x in g[f"{name}/meta"])
    tol, _, h0 = (float(x) for x in g[f"{name}/ctrl"])
    N = g[f"{name}/u0"].shape[1]
    mlp = oc.Mlp((N + 1, 16, 16, N), "tanh", g[f"{name}/theta"], time_input=True)
    scaling = ol.MinMax(g[f"{name}/lo"], g[f"{name}/hi"]) if f"{name}/lo" in g else None
    times = tuple(float(t) for t in g[f"{name}/times"])
    obs = ol.ObsLoss(kind, range(len(times)), g[f"{name}/values"], scaling)
    return mlp, sch, pol, oa.AdaptiveCtrl(abstol=tol, reltol=tol, h_init=h0), obs, times


@pytest.mark.parametrize("name", ADAPTIVE_CASES)
def test_adaptive_stepping_matches_reference(golden, name):
    from oracle import adaptive as oa
    g = golden("adaptive.npz")
    mlp, sch, pol, ctrl, obs, times = adaptive_case(g, name)
    res = oa.grad_adaptive(oc.MlpField(mlp), sch, g[f"{name}/u0"], 0.0, 1.0, ctrl, pol,
                           obs=obs, obs_times=times)
    for k in ("accepted", "rejected", "nfe_forward", "nfe_backward", "steps_recomputed"):
        assert list(res[k]) == list(g[f"{name}/{k}"]), k
    for b, grid in enumerate(res["grids"]):
        ref = g[f"{name}/grids"][b]
        ref = ref[~np.isnan(ref)]
        # the embedded error estimate cancels ~8 digits (err ~ 1e-9 from O(1) stages),
        # so ulp-level field differences move the step sizes at the 1e-11 level
        assert len(grid) == len(ref) and np.max(np.abs(grid - ref)) <= 1e-9
    assert abs(res["loss"] - float(g[f"{name}/loss"])) <= 1e-12 * abs(float(g[f"{name}/loss"]))
    assert oc.rel_error(res["predictions"], g[f"{name}/predictions"]) <= 1e-12
    assert oc.rel_error(res["dtheta"], g[f"{name}/dtheta"]) <= 1e-10
    assert oc.rel_error(res["du0"], g[f"{name}/du0"]) <= 1e-10


def test_adaptive_rules():
    from oracle import adaptive as oa
    mlp = oc.Mlp((3, 4, 2), "tanh", np.zeros(4 * 3 + 4 + 2 * 4 + 2), time_input=True)
    with pytest.raises(ValueError):
        oa.grad_adaptive(oc.MlpField(mlp), "dopri5", np.ones((1, 2)), 0.0, 1.0, oa.AdaptiveCtrl(),
                         "revolve:2")
    with pytest.raises(oc.IntegrationError):
        oa.grad_adaptive(oc.MlpField(mlp), "rk4", np.ones((1, 2)), 0.0, 1.0, oa.AdaptiveCtrl())


def test_adamw_restatement_matches_reference(golden):
    from oracle import training as otr
    g = golden("training.npz")
    theta, m, v, t = g["adamw/theta0"], np.zeros(50), np.zeros(50), 0
    for k in range(4):
        theta, m, v, t = otr.adamw_step(theta, g[f"adamw/g{k}"], m, v, t, lr=0.01, weight_decay=0.1)
        assert np.array_equal(theta, g[f"adamw/theta{k + 1}"])
        assert np.array_equal(m, g[f"adamw/m{k + 1}"]) and np.array_equal(v, g[f"adamw/v{k + 1}"])


def test_dataset_formats_roundtrip(tmp_path, golden):
    from paper_2206_01298_b200.formats import read_dataset_csv, write_dataset_csv
    from paper_2206_01298_b200.training import Dataset, geometric_grid, minmax_normalize
    g = golden("training.npz")
    ds = Dataset(g["data/times"], list(g["data/obs"]))
    p = tmp_path / "d.csv"
    write_dataset_csv(ds, p)
    back = read_dataset_csv(p)
    assert np.array_equal(back.times, ds.times) and np.array_equal(back.matrix(), ds.matrix())
    assert open(p).readline().strip() == "t,u1,u2,u3"
    grid = geometric_grid(ds.times, 3)
    assert len(grid) == 3 * (len(ds.times) - 1) + 1
    assert all(np.min(np.abs(grid - t)) <= 1e-9 * t for t in ds.times)
    nd = minmax_normalize(ds)
    assert np.allclose(nd.matrix().min(axis=0), 0.0) and np.allclose(nd.matrix().max(axis=0), 1.0)
    with pytest.raises(ValueError):
        Dataset([0.0, 0.0], [np.zeros(2), np.zeros(2)])


@pytest.mark.parametrize("sch", ["euler", "rk4", "dopri5"])
def test_continuous_adjoint_matches_reference(golden, sch):
    from oracle import cadj
    g = golden("cadj.npz")
    n_steps, tin = (int(x) for x in g[f"{sch}/meta"])
    mlp = oc.Mlp((3 + tin, 8, 8, 3), "tanh", g[f"{sch}/theta"], time_input=bool(tin))
    uf = g[f"{sch}/u_final"]
    lam0, mu0 = cadj.continuous_adjoint_solve(oc.MlpField(mlp), sch, uf / uf.shape[0], uf, 0.0, 1.0,
                                              n_steps)
    assert oc.rel_error(lam0, g[f"{sch}/lam0"]) <= 1e-12
    assert oc.rel_error(mu0, g[f"{sch}/mu0"]) <= 1e-12
