"""TEST INFRASTRUCTURE ONLY -- the oracle side of each BASELINE config:
(field, initial state, terminal seed, solver config) for oracle.core.grad_terminal.
Used by tests/ and by bench.py's cpu_baseline / --impl reference legs."""

from __future__ import annotations

from . import core as oc
from . import fields_ext as ox


def oracle_problem(ci, batch_global=None):
    """Oracle field / y0 / seed_fn / SolverCfg for a ConfigInputs."""
    B = batch_global or ci.batch
    if ci.kind == "conv":
        mlp = None
    else:
        mlp = oc.Mlp(ci.widths, ci.activation, ci.theta, ci.time_input)
    if ci.kind == "stiff":
        return (oc.StiffField(mlp, ci.extras["diag"], ci.extras["scale"]), ci.u0, None,
                oc.SolverCfg(**ci.extras["solver"]))
    if ci.kind == "cnf":
        fld = ox.CnfField(mlp, ci.extras["eps"])
        return fld, ox.cnf_initial_state(ci.u0), ox.cnf_seed(fld.D, B), oc.SolverCfg()
    if ci.kind == "mlp":
        return oc.MlpField(mlp), ci.u0, None, oc.SolverCfg()
    if ci.kind == "conv":
        fld = ox.ConvField(ci.theta)
        head, labels = ci.extras["head"], ci.extras["labels"]

        def seed(uf):
            loss, lam, _ = ox.head_loss(uf, head, labels[:uf.shape[0]], batch_global=B)
            return loss, lam
        return fld, ci.u0.reshape(ci.batch, -1), seed, oc.SolverCfg()
    raise NotImplementedError(ci.kind)


def run_oracle(ci, policy=None, rows=None):
    """grad_terminal on the config (optionally a row slice, batch seed over the full batch)."""
    fld, y0, seed, cfg = oracle_problem(ci)
    if rows is not None:
        y0 = y0[rows]
        if hasattr(fld, "eps"):
            fld = type(fld)(fld.mlp, fld.eps[rows])
        if ci.kind == "conv":
            from . import fields_ext as ox2
            head, labels = ci.extras["head"], ci.extras["labels"][rows]

            def seed(uf):
                loss, lam, _ = ox2.head_loss(uf, head, labels, batch_global=ci.batch)
                return loss, lam
    return oc.grad_terminal(fld, ci.scheme, y0, ci.t0, ci.tF, ci.n_steps, policy or ci.policy,
                            seed_fn=seed, cfg=cfg)
