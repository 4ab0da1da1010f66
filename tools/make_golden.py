"""Generate golden fixtures by running the REFERENCE (odegrad) itself.

Run in the build container only (needs /root/reference, read-only):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tools/make_golden.py
    ODEGRAD_NO_NUMBA=1 python tools/make_golden.py     # C5 numpy-path variant

Writes ``tests/golden/*.npz``.  Inputs come from the package's seeded config
generator (``paper_2206_01298_b200.configs``); the reference is driven through
its own public API: ``forward_pass`` + ``backward_sweep`` with the BASELINE
terminal seed lam_N = u_b(T)/B (the pattern of
``pkg/tests/test_acceptance.py:188-193``), per sample, summing mu_b in sample
order.  Nothing here is imported at test time; the fixtures are data.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, REF)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import odegrad as og  # noqa: E402
from odegrad import nn as ognn  # noqa: E402

from paper_2206_01298_b200 import configs  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def ref_batch_grad(field, scheme_name, U0, t0, tF, n_steps, policy, cfg=None):
    """Per-sample reference forward_pass + backward_sweep, batch seed u/B."""
    scheme = og.tableau_catalog(scheme_name)
    cfg = cfg or og.SolverConfig()
    pol = og.CheckpointPolicy.parse(policy)
    B = U0.shape[0]
    uf, du0, mus, nfe_f, nfe_b, recomp = [], [], [], [], [], []
    store = None
    for b in range(B):
        c = og.NfeCounters()
        fwd = og.adjoint.forward_pass(field, scheme, U0[b], t0, tF, og.FixedController(n_steps),
                                      pol, cfg, c, obs_times=())
        lamN = fwd.u_final / B
        adj = og.adjoint.backward_sweep(field, scheme, fwd,
                                        og.AdjointState(lamN, np.zeros(field.n_params)),
                                        {}, cfg, c)
        uf.append(fwd.u_final)
        du0.append(adj.lam)
        mus.append(adj.mu)
        nfe_f.append(c.nfe_forward)
        nfe_b.append(c.nfe_backward)
        recomp.append(c.steps_recomputed)
        store = fwd.store.counters
    uf = np.array(uf)
    dth = np.zeros(field.n_params)
    for m in mus:
        dth = dth + m
    loss = float(np.mean(0.5 * np.sum(uf * uf, axis=1)))
    return dict(u_final=uf, du0=np.array(du0), dtheta=dth, loss=np.float64(loss),
                nfe_forward=np.array(nfe_f), nfe_backward=np.array(nfe_b),
                steps_recomputed=np.array(recomp),
                stored_states=np.int64(store.stored_states),
                stored_stage_vectors=np.int64(store.stored_stage_vectors),
                max_live_slots=np.int64(store.max_live_slots),
                recomputed_steps=np.int64(store.recomputed_steps))


def mlp_field(cfg_in):
    spec = og.MlpSpec(tuple(cfg_in.widths), cfg_in.activation, cfg_in.time_input)
    return og.MlpField(og.MlpModel(spec, cfg_in.theta.copy()))


def stiff_field(cfg_in):
    spec = og.MlpSpec(tuple(cfg_in.widths), cfg_in.activation, False)
    model = og.MlpModel(spec, cfg_in.theta.copy())
    a = cfg_in.extras["diag"]
    s = cfg_in.extras["scale"]

    def f(u, t):
        return a * u + s * ognn.mlp_forward(model, u)[0]

    def jvp(u, t, w):
        return a * w + s * ognn.jvp_input(model, ognn.mlp_forward(model, u)[1], w)

    def vjp_u(u, t, v):
        return a * v + s * ognn.vjp_input(model, ognn.mlp_forward(model, u)[1], v)

    def vjp_theta(u, t, v):
        return s * ognn.vjp_params(model, ognn.mlp_forward(model, u)[1], v)

    return og.CallableField(f, jvp, vjp_u, vjp_theta, model.n_params)


def save(name, **arrays):
    path = os.path.join(OUT, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.1f} KiB)")


def gen_small():
    """All 7 schemes x 3 policies on a toy MLP, 3 samples, seed-fixed."""
    out = {}
    rng = np.random.default_rng(20260101)
    for si, name in enumerate(og.SCHEME_NAMES):
        model = og.init_model(og.mlp_spec(3, 8, 2, "tanh"), seed=si)
        U0 = rng.uniform(-1, 1, (3, 3))
        out[f"{name}/theta"] = model.theta
        out[f"{name}/u0"] = U0
        for pol in ("store_all", "store_solutions", "revolve:3"):
            r = ref_batch_grad(og.MlpField(model), name, U0, 0.0, 1.0, 7, pol)
            for k, v in r.items():
                out[f"{name}/{pol}/{k}"] = v
    # time-input + every activation on rk4 / dopri5 (kernel coverage)
    for act in ("identity", "relu", "tanh", "gelu"):
        spec = og.mlp_spec(4, 6, 2, act, time_input=True)
        model = og.init_model(spec, seed=11)
        U0 = rng.standard_normal((2, 4))
        out[f"act_{act}/theta"] = model.theta
        out[f"act_{act}/u0"] = U0
        r = ref_batch_grad(og.MlpField(model), "dopri5", U0, 0.0, 1.0, 5, "store_all")
        for k, v in r.items():
            out[f"act_{act}/{k}"] = v
    save("small_schemes.npz", **out)


def gen_kernels():
    """Per-sample reference kernel outputs (forward / vjp / jvp) for every activation."""
    out = {}
    rng = np.random.default_rng(7)
    for act in ("identity", "relu", "tanh", "gelu"):
        spec = og.mlp_spec(5, 7, 2, act, time_input=True)
        model = og.init_model(spec, seed=3)
        U = rng.standard_normal((4, 5))
        V = rng.standard_normal((4, 5))
        Wt = rng.standard_normal((4, 5))
        ts = rng.uniform(0, 1, 4)
        fs, jt, pt, jv = [], [], [], []
        for b in range(4):
            f, cache = ognn.mlp_forward(model, U[b], ts[b])
            d, p = ognn.vjp_pair(model, cache, V[b])
            fs.append(f)
            jt.append(d)
            pt.append(p)
            jv.append(ognn.jvp_input(model, cache, Wt[b]))
        out.update({f"{act}/theta": model.theta, f"{act}/U": U, f"{act}/V": V, f"{act}/W": Wt,
                    f"{act}/t": ts, f"{act}/f": np.array(fs), f"{act}/jtv": np.array(jt),
                    f"{act}/ptv": np.array(pt), f"{act}/jv": np.array(jv)})
    save("mlp_kernels.npz", **out)


def gen_config(name, nsub, policies, solver=None, suffix=""):
    cfg_in = configs.make_config(name).subset(nsub)
    out = {"theta_checksum": np.float64(np.sum(cfg_in.theta * np.arange(1, cfg_in.theta.size + 1))),
           "u0": cfg_in.u0}
    fld = stiff_field(cfg_in) if cfg_in.kind == "stiff" else mlp_field(cfg_in)
    scfg = og.SolverConfig(**solver) if solver else None
    for pol in policies:
        tic = time.time()
        r = ref_batch_grad(fld, cfg_in.scheme, cfg_in.u0, cfg_in.t0, cfg_in.tF, cfg_in.n_steps,
                           pol, scfg)
        print(f"  {name} {pol}: {time.time() - tic:.1f}s")
        for k, v in r.items():
            out[f"{pol}/{k}"] = v
    save(f"{name.lower()}_sub{suffix}.npz", **out)


def gen_obs():
    """Multi-observation MAE/MSE losses with min-max scaling (losses.py:10-107,
    adjoint.py:143-279) through the reference's own grad(), per sample; the batch
    result is the sample mean (loss, dtheta) and du0_b / B."""
    out = {}
    rng = np.random.default_rng(424242)
    cases = [
        ("mse_rk4", "mse", "rk4", "store_all", (0.25, 0.5, 1.0), False, False),
        ("mae_dopri5", "mae", "dopri5", "revolve:3", (0.0, 0.5, 0.75), True, True),
        ("mse_cn", "mse", "cn", "store_solutions", (0.5, 1.0), True, False),
        ("mae_rk4_tF", "mae", "rk4", "store_all", (1.0,), False, False),
    ]
    n_steps, B, N = 8, 3, 3
    for name, kind, sch, pol, times, scaled, tin in cases:
        model = og.init_model(og.mlp_spec(N, 8, 2, "tanh", time_input=tin), seed=5)
        U0 = rng.uniform(-1, 1, (B, N))
        vals = rng.uniform(-0.5, 0.5, (len(times), B, N))
        lo = hi = None
        scaling = None
        if scaled:
            lo = np.array([-1.0, 0.3, -2.0])
            hi = np.array([1.5, 0.3, 0.5])       # component 1 degenerate (hi <= lo)
            scaling = og.losses.MinMaxScaling(lo, hi)
        scheme = og.tableau_catalog(sch)
        ctrl = og.FixedController(n_steps)
        loss, dth, du0, preds = 0.0, np.zeros(model.n_params), [], []
        for b in range(B):
            spec = og.losses.LossSpec(kind, times, tuple(vals[:, b]), scaling)
            r = og.grad(og.MlpField(model), scheme, spec, U0[b], 0.0, 1.0, ctrl,
                        og.CheckpointPolicy.parse(pol))
            loss += r.loss / B
            dth = dth + r.dtheta / B
            du0.append(r.du0 / B)
            preds.append(np.array(r.predictions))
        pre = f"{name}/"
        out[pre + "theta"] = model.theta
        out[pre + "u0"] = U0
        out[pre + "values"] = vals
        out[pre + "times"] = np.array(times)
        out[pre + "meta"] = np.array([kind, sch, pol, str(int(tin))])
        if scaled:
            out[pre + "lo"] = lo
            out[pre + "hi"] = hi
        out[pre + "loss"] = np.float64(loss)
        out[pre + "dtheta"] = dth
        out[pre + "du0"] = np.array(du0)
        out[pre + "predictions"] = np.transpose(np.array(preds), (1, 0, 2))   # [K, B, N]
    save("obs_losses.npz", **out)


def gen_adaptive():
    """Adaptive Dopri5 / Bosh3 stepping (integrators.py:294-349, adjoint.py:162-186)
    through the reference's grad() per sample; batch = sample mean."""
    from odegrad.integrators import AdaptiveController
    out = {}
    rng = np.random.default_rng(777)
    cases = [
        ("dopri5_term", "dopri5", "mse", "store_all", (1.0,), False, 1e-8, 0.5),
        ("bosh3_obs", "bosh3", "mae", "store_solutions", (0.3, 0.7, 1.0), True, 1e-6, 0.3),
        ("dopri5_obs0", "dopri5", "mse", "store_all", (0.0, 0.5), False, 1e-9, 0.4),
    ]
    B, N = 3, 3
    for name, sch, kind, pol, times, scaled, tol, h0 in cases:
        model = og.init_model(og.mlp_spec(N, 16, 2, "tanh", time_input=True), seed=9)
        model = og.MlpModel(model.spec, 2.5 * model.theta)     # livelier dynamics
        U0 = rng.uniform(-1.5, 1.5, (B, N))
        vals = rng.uniform(-0.5, 0.5, (len(times), B, N))
        scaling = og.losses.MinMaxScaling(np.array([-1.0, 0.2, -2.0]),
                                          np.array([1.5, 0.2, 0.5])) if scaled else None
        ctrl = AdaptiveController(abstol=tol, reltol=tol, h_init=h0)
        loss, dth, du0, preds, grids = 0.0, np.zeros(model.n_params), [], [], []
        acc, rej, nff, nfb, rec = [], [], [], [], []
        for b in range(B):
            spec = og.losses.LossSpec(kind, times, tuple(vals[:, b]), scaling)
            c = og.NfeCounters()
            r = og.grad(og.MlpField(model), og.tableau_catalog(sch), spec, U0[b], 0.0, 1.0, ctrl,
                        og.CheckpointPolicy.parse(pol), counters=c)
            fwd = og.adjoint.forward_pass(og.MlpField(model), og.tableau_catalog(sch), U0[b], 0.0,
                                          1.0, ctrl, og.CheckpointPolicy.parse(pol),
                                          og.SolverConfig(), og.NfeCounters(), obs_times=times)
            loss += r.loss / B
            dth = dth + r.dtheta / B
            du0.append(r.du0 / B)
            preds.append(np.array(r.predictions))
            grids.append(np.array(fwd.boundary_times))
            acc.append(c.steps_accepted)
            rej.append(c.steps_rejected)
            nff.append(c.nfe_forward)
            nfb.append(c.nfe_backward)
            rec.append(c.steps_recomputed)
        L = max(len(g) for g in grids)
        pre = f"{name}/"
        out[pre + "theta"] = model.theta
        out[pre + "u0"] = U0
        out[pre + "values"] = vals
        out[pre + "times"] = np.array(times)
        out[pre + "meta"] = np.array([sch, kind, pol])
        out[pre + "ctrl"] = np.array([tol, tol, h0])
        if scaled:
            out[pre + "lo"] = scaling.lo
            out[pre + "hi"] = scaling.hi
        out[pre + "loss"] = np.float64(loss)
        out[pre + "dtheta"] = dth
        out[pre + "du0"] = np.array(du0)
        out[pre + "predictions"] = np.transpose(np.array(preds), (1, 0, 2))
        out[pre + "grids"] = np.array([np.pad(g, (0, L - len(g)), constant_values=np.nan) for g in grids])
        out[pre + "accepted"] = np.array(acc)
        out[pre + "rejected"] = np.array(rej)
        out[pre + "nfe_forward"] = np.array(nff)
        out[pre + "nfe_backward"] = np.array(nfb)
        out[pre + "steps_recomputed"] = np.array(rec)
    save("adaptive.npz", **out)


def gen_training():
    """AdamW steps (training.py:175-190), a reference Robertson dataset
    (training.py:86-129, minmax-normalised :132-137) and short train() runs
    (training.py:233-329): CN on the geometric grid and adaptive Dopri5; plus the
    reference's model JSON / dataset CSV text (nn.py:190-220, training.py:140-152)."""
    from odegrad import training as tr
    from odegrad import nn as rnn
    out = {}
    rng = np.random.default_rng(99)
    theta = rng.standard_normal(50)
    st = tr.OptimizerState.zeros(50)
    cfg = tr.AdamWConfig(lr=0.01, weight_decay=0.1)
    out["adamw/theta0"] = theta.copy()
    for k in range(4):
        g = rng.standard_normal(50) * (10.0 ** (k - 2))
        theta, st = tr.adamw_step(theta, g, st, cfg)
        out[f"adamw/g{k}"] = g
        out[f"adamw/theta{k + 1}"] = theta.copy()
        out[f"adamw/m{k + 1}"] = st.m.copy()
        out[f"adamw/v{k + 1}"] = st.v.copy()
    ds = tr.minmax_normalize(tr.generate_robertson_dataset(n_points=6, span=(1e-5, 1e-1), n_sub=12))
    out["data/times"] = ds.times
    out["data/obs"] = ds.matrix()
    model = og.init_model(og.mlp_spec(3, 8, 1, "tanh"), seed=3)
    out["model/theta"] = model.theta
    out["model/json"] = np.array(rnn.model_to_json(model))
    runs = [("cn", tr.TrainConfig(epochs=4, n_sub=3, loss_kind="mae",
                                  optimizer=tr.AdamWConfig(lr=0.01))),
            ("dopri5", tr.TrainConfig(epochs=3, loss_kind="mse", abstol=1e-6, reltol=1e-6,
                                      optimizer=tr.AdamWConfig(lr=0.02, weight_decay=0.01)))]
    for sch, tc in runs:
        trained, rec = tr.train(model, og.tableau_catalog(sch), ds, tc)
        pre = f"train_{sch}/"
        out[pre + "loss"] = np.array(rec.loss)
        out[pre + "grad_norm"] = np.array(rec.grad_norm)
        out[pre + "nfe_forward"] = np.array(rec.nfe_forward)
        out[pre + "nfe_backward"] = np.array(rec.nfe_backward)
        out[pre + "final_theta"] = rec.final_theta
    save("training.npz", **out)


def gen_cadj():
    """Continuous-adjoint baseline (adjoint.py:294-331) per sample: terminal state
    from the reference integrate, seed u(tF)/B; batch mu = sum over samples."""
    out = {}
    rng = np.random.default_rng(1234)
    B = 3
    for sch, n_steps, tin in (("euler", 12, False), ("rk4", 6, True), ("dopri5", 5, True)):
        model = og.init_model(og.mlp_spec(3, 8, 2, "tanh", time_input=tin), seed=21)
        U0 = rng.uniform(-1, 1, (B, 3))
        fld = og.MlpField(model)
        scheme = og.tableau_catalog(sch)
        lam0, mu0, uf, nff, nfb = [], np.zeros(model.n_params), [], [], []
        for b in range(B):
            u1, _ = og.integrators.integrate(scheme, fld, U0[b], 0.0, 1.0, og.FixedController(n_steps))
            c = og.NfeCounters()
            lam, mu, _ = og.adjoint.continuous_adjoint_solve(fld, scheme, u1 / B, u1, 0.0, 1.0,
                                                             n_steps, counters=c)
            lam0.append(lam)
            mu0 = mu0 + mu
            uf.append(u1)
            nff.append(c.nfe_forward)
            nfb.append(c.nfe_backward)
        pre = f"{sch}/"
        out[pre + "theta"] = model.theta
        out[pre + "u0"] = U0
        out[pre + "u_final"] = np.array(uf)
        out[pre + "lam0"] = np.array(lam0)
        out[pre + "mu0"] = mu0
        out[pre + "meta"] = np.array([n_steps, int(tin)])
        out[pre + "nfe"] = np.array([nff, nfb])
    save("cadj.npz", **out)


def gen_revolve():
    out = {}
    counts = np.zeros((61, 21), np.int64)
    for nt in range(1, 61):
        for nc in range(1, 21):
            counts[nt, nc] = og.revolve_count(nt, nc)
    out["counts"] = counts
    kinds = {"advance": 0, "store": 1, "restore": 2, "reverse": 3}
    for nt, nc in [(1, 1), (2, 1), (4, 1), (9, 2), (10, 3), (12, 11), (40, 8), (37, 5),
                   (60, 4), (25, 1), (40, 39)]:
        acts = og.revolve_schedule(nt, nc)
        out[f"sched_{nt}_{nc}"] = np.array([[kinds[a.kind], a.step, a.start, a.stop] for a in acts],
                                           np.int64)
    save("revolve.npz", **out)


def _c5_chunk(args):
    lo, hi = args
    cfg_in = configs.make_config("C5")
    fld = stiff_field(cfg_in)
    scfg = og.SolverConfig(**cfg_in.extras["solver"])
    B = cfg_in.batch
    scheme = og.tableau_catalog(cfg_in.scheme)
    pol = og.CheckpointPolicy.parse("store_all")
    out = []
    for b in range(lo, hi):
        c = og.NfeCounters()
        fwd = og.adjoint.forward_pass(fld, scheme, cfg_in.u0[b], cfg_in.t0, cfg_in.tF,
                                      og.FixedController(cfg_in.n_steps), pol, scfg, c, obs_times=())
        adj = og.adjoint.backward_sweep(fld, scheme, fwd,
                                        og.AdjointState(fwd.u_final / B, np.zeros(fld.n_params)),
                                        {}, scfg, c)
        out.append((b, fwd.u_final, adj.lam, adj.mu, c.nfe_forward, c.nfe_backward))
    return out


def gen_c5_full():
    """C5 at the full BASELINE batch (256 samples; the benchmarked 2-rows-per-CTA tile)
    through the reference per sample (forward_pass + backward_sweep, seed u/B), in a
    process pool; mu summed in sample order.  Also the first-16-sample sum (tile-geometry
    tests at 2 and 8 rows per CTA)."""
    import multiprocessing as mp
    B = configs.make_config("C5").batch
    nproc = len(os.sched_getaffinity(0))
    chunks = [(i, min(B, i + 4)) for i in range(0, B, 4)]
    tic = time.time()
    with mp.get_context("fork").Pool(nproc) as pool:
        rows = [r for part in pool.map(_c5_chunk, chunks) for r in part]
    rows.sort(key=lambda r: r[0])
    print(f"  C5 full: {time.time() - tic:.1f}s on {nproc} processes")
    uf = np.array([r[1] for r in rows])
    du0 = np.array([r[2] for r in rows])
    dth = np.zeros_like(rows[0][3])
    dth16 = None
    for i, r in enumerate(rows):
        dth = dth + r[3]
        if i == 15:
            dth16 = dth.copy()
    cfg_in = configs.make_config("C5")
    save("c5_full.npz", u0_checksum=np.float64(np.sum(cfg_in.u0)), u_final=uf, du0=du0, dtheta=dth,
         dtheta_first16=dth16, loss=np.float64(np.mean(0.5 * np.sum(uf * uf, axis=1))),
         nfe_forward=np.array([r[4] for r in rows]), nfe_backward=np.array([r[5] for r in rows]))


def gen_adaptive_rows():
    """Adaptive stepping with many samples per CTA tile: B = 12 samples whose
    controllers accept / reject on different trials (per-sample grids of different
    lengths), through the reference's grad() per sample; batch = sample mean."""
    from odegrad.integrators import AdaptiveController
    out = {}
    rng = np.random.default_rng(4242)
    cases = [
        ("dopri5_rows", "dopri5", "mse", "store_all", (1.0,), 1e-8, 0.5),
        ("bosh3_rows", "bosh3", "mae", "store_solutions", (0.4, 1.0), 1e-6, 0.3),
    ]
    B, N = 12, 3
    for name, sch, kind, pol, times, tol, h0 in cases:
        model = og.init_model(og.mlp_spec(N, 16, 2, "tanh", time_input=True), seed=11)
        model = og.MlpModel(model.spec, 2.5 * model.theta)
        # spread initial states so the per-sample step-size histories differ
        U0 = rng.uniform(-1.5, 1.5, (B, N)) * np.linspace(0.2, 2.5, B)[:, None]
        vals = rng.uniform(-0.5, 0.5, (len(times), B, N))
        ctrl = AdaptiveController(abstol=tol, reltol=tol, h_init=h0)
        loss, dth, du0, grids = 0.0, np.zeros(model.n_params), [], []
        acc, rej, nff, nfb = [], [], [], []
        for b in range(B):
            spec = og.losses.LossSpec(kind, times, tuple(vals[:, b]), None)
            c = og.NfeCounters()
            r = og.grad(og.MlpField(model), og.tableau_catalog(sch), spec, U0[b], 0.0, 1.0, ctrl,
                        og.CheckpointPolicy.parse(pol), counters=c)
            fwd = og.adjoint.forward_pass(og.MlpField(model), og.tableau_catalog(sch), U0[b], 0.0,
                                          1.0, ctrl, og.CheckpointPolicy.parse(pol),
                                          og.SolverConfig(), og.NfeCounters(), obs_times=times)
            loss += r.loss / B
            dth = dth + r.dtheta / B
            du0.append(r.du0 / B)
            grids.append(np.array(fwd.boundary_times))
            acc.append(c.steps_accepted)
            rej.append(c.steps_rejected)
            nff.append(c.nfe_forward)
            nfb.append(c.nfe_backward)
        L = max(len(g) for g in grids)
        pre = f"{name}/"
        out[pre + "theta"] = model.theta
        out[pre + "u0"] = U0
        out[pre + "values"] = vals
        out[pre + "times"] = np.array(times)
        out[pre + "meta"] = np.array([sch, kind, pol])
        out[pre + "ctrl"] = np.array([tol, tol, h0])
        out[pre + "loss"] = np.float64(loss)
        out[pre + "dtheta"] = dth
        out[pre + "du0"] = np.array(du0)
        out[pre + "grids"] = np.array([np.pad(g, (0, L - len(g)), constant_values=np.nan) for g in grids])
        out[pre + "accepted"] = np.array(acc)
        out[pre + "rejected"] = np.array(rej)
        out[pre + "nfe_forward"] = np.array(nff)
        out[pre + "nfe_backward"] = np.array(nfb)
        print(f"  {name}: accepted {acc}, rejected {rej}")
    save("adaptive_rows.npz", **out)


def gen_c5_rows_numpy():
    """Per-sample NFE counts of the first 16 C5 samples on the reference's numpy
    kernel path (ODEGRAD_NO_NUMBA=1): how far the reference's own two kernel paths
    disagree on data-dependent Newton / GMRES counts (rounding-boundary stops), the
    yardstick for the GPU's counts against c5_full.npz (numba path)."""
    import multiprocessing as mp
    with mp.get_context("fork").Pool(len(os.sched_getaffinity(0))) as pool:
        rows = [r for part in pool.map(_c5_chunk, [(i, i + 1) for i in range(16)]) for r in part]
    rows.sort(key=lambda r: r[0])
    save("c5_rows_numpy.npz", nfe_forward=np.array([r[4] for r in rows]),
         nfe_backward=np.array([r[5] for r in rows]),
         du0=np.array([r[2] for r in rows]))


if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    if not og.kernels.NUMBA_ENABLED:
        # the reference's own numpy kernel path (ODEGRAD_NO_NUMBA=1): its
        # ulp-level differences from the numba path flip GMRES stopping
        # decisions at rounding boundaries, so C5 iteration counts are pinned
        # against both paths ("iteration-count parity").
        if len(sys.argv) > 1 and sys.argv[1] == "c5_rows":
            gen_c5_rows_numpy()
            sys.exit(0)
        gen_config("C5", 2, ["store_all"], solver=configs.make_c5(batch=1).extras["solver"],
                   suffix="_numpy")
        gen_c5_rows_numpy()
        sys.exit(0)
    og.kernels.warmup()
    if len(sys.argv) > 1 and sys.argv[1] == "obs":
        gen_obs()
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "adaptive":
        gen_adaptive()
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "adaptive_rows":
        gen_adaptive_rows()
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "c5_full":
        gen_c5_full()
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "training":
        gen_training()
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "cadj":
        gen_cadj()
        sys.exit(0)
    gen_revolve()
    gen_kernels()
    gen_small()
    gen_obs()
    gen_adaptive()
    gen_training()
    gen_cadj()
    gen_config("C1", 4, ["store_all", "store_solutions", "revolve:3"])
    gen_config("C2", 3, ["store_all", "revolve:8"])
    gen_config("C5", 2, ["store_all"], solver=configs.make_c5(batch=1).extras["solver"])
    gen_adaptive_rows()
    gen_c5_full()
