"""Toy-size gradient calls for compute-sanitizer (tools/sanitize.sh): every kernel
family of the library once -- tcgen05 MLP tile (C2 shape, 2 tiles), SIMT MLP tiles
fp32 / fp64, CNF, conv, theta-method Newton/GMRES, adaptive, field ops, optimizer."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2206_01298_b200 import (AdaptiveController, CheckpointPolicy, MlpField, MlpModel, MlpSpec,  # noqa: E402
                                   grad, tableau_catalog, terminal_loss)
from paper_2206_01298_b200.configs import make_config  # noqa: E402
from paper_2206_01298_b200.workloads import field_from_config, run_config  # noqa: E402
from paper_2206_01298_b200 import training as tr  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"


def case(name):
    return which in ("all", name)


if case("tc"):
    ci = make_config("C2").subset(40)
    r = run_config(ci, "revolve:3", tile_rows=20)
    assert r.device["tensor_cores"] == 1
    print("tc ok", r.loss)
if case("simt"):
    ci = make_config("C2").subset(6)
    print("simt32 ok", run_config(ci, "revolve:3", tensor_cores=False).loss)
    ci = make_config("C1").subset(6)
    print("simt64 ok", run_config(ci, "store_solutions").loss)
    fld = field_from_config(ci)
    fld.eval(ci.u0, 0.3)
    fld.jvp(ci.u0, 0.3, ci.u0)
    fld.vjp(ci.u0, 0.3, ci.u0)
if case("cnf"):
    ci = make_config("C4").subset(3)
    print("cnf ok", run_config(ci, "store_all").loss)
if case("conv"):
    ci = make_config("C3").subset(1)
    print("conv ok", run_config(ci, "store_all").loss)
if case("theta"):
    ci = make_config("C5").subset(2)
    print("theta ok", run_config(ci, "store_all").loss)
if case("adaptive"):
    spec = MlpSpec((4, 16, 16, 3), "tanh", time_input=True)
    model = MlpModel(spec, np.random.default_rng(1).uniform(-0.5, 0.5, spec.n_params))
    r = grad(MlpField(model), tableau_catalog("dopri5"), terminal_loss("half_sqnorm", 1.0),
             np.random.default_rng(2).standard_normal((3, 3)), 0.0, 1.0,
             AdaptiveController(1e-6, 1e-6, h_init=0.1))
    print("adaptive ok", r.loss)
if case("optim"):
    th = torch.ones(1000, dtype=torch.float64, device="cuda")
    st = tr.OptimizerState.zeros(1000)
    tr.adamw_step(th, torch.full_like(th, 0.5), st, tr.AdamWConfig())
    print("optim ok", tr.grad_norm(th))
torch.cuda.synchronize()
