"""GPU parity for the continuous-adjoint baseline (
continuous_adjoint_solve, adjoint.py:294-331) against the reference's own
results (tests/golden/cadj.npz): fp64 <= 1e-10, NFE counts exact; plus the
reference's known answers (zero terminal seed gives zero, test_adjoint.py:292-300)
and the O(h) gap to the discrete adjoint on a nonlinear field."""

import numpy as np
import pytest
import torch

from oracle import core as oc
from paper_2206_01298_b200 import (FixedController, MlpField, MlpModel, MlpSpec, NfeCounters,
                                   continuous_adjoint_solve, grad, tableau_catalog, terminal_loss)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    from paper_2206_01298_b200 import _lib as L
    L.load()


def _field(g, sch, dtype="f64"):
    n_steps, tin = (int(x) for x in g[f"{sch}/meta"])
    spec = MlpSpec((3 + tin, 8, 8, 3), "tanh", time_input=bool(tin), dtype=dtype)
    return MlpField(MlpModel(spec, g[f"{sch}/theta"])), n_steps


@pytest.mark.parametrize("sch", ["euler", "rk4", "dopri5"])
def test_continuous_adjoint_matches_reference(golden, sch):
    g = golden("cadj.npz")
    fld, n_steps = _field(g, sch)
    uf = g[f"{sch}/u_final"]
    c = NfeCounters()
    lam0, mu0, c = continuous_adjoint_solve(fld, tableau_catalog(sch), uf / uf.shape[0], uf,
                                            0.0, 1.0, n_steps, c)
    assert oc.rel_error(lam0, g[f"{sch}/lam0"]) <= 1e-10
    assert oc.rel_error(mu0, g[f"{sch}/mu0"]) <= 1e-10
    assert c.nfe_forward == int(g[f"{sch}/nfe"][0, 0]) and c.nfe_backward == int(g[f"{sch}/nfe"][1, 0])


def test_continuous_adjoint_zero_seed_and_gap(golden):
    g = golden("cadj.npz")
    fld, n_steps = _field(g, "rk4")
    uf = g["rk4/u_final"]
    lam0, mu0, _ = continuous_adjoint_solve(fld, tableau_catalog("rk4"), np.zeros_like(uf), uf,
                                            0.0, 1.0, n_steps)
    assert not np.any(lam0) and not np.any(mu0)
    # discrete vs continuous: agree to O(h^p) on a smooth field, not bit-for-bit
    u0 = g["rk4/u0"]
    res = grad(fld, tableau_catalog("rk4"), terminal_loss("half_sqnorm", 1.0), u0, 0.0, 1.0,
               FixedController(n_steps))
    lam_c, mu_c, _ = continuous_adjoint_solve(fld, tableau_catalog("rk4"), res.u_final / u0.shape[0],
                                              res.u_final, 0.0, 1.0, n_steps)
    gap = oc.rel_error(mu_c, res.dtheta)
    assert 0.0 < gap < 1e-3


def test_continuous_adjoint_fp32(golden):
    g = golden("cadj.npz")
    fld, n_steps = _field(g, "dopri5", "f32")
    uf = g["dopri5/u_final"]
    lam0, mu0, _ = continuous_adjoint_solve(fld, tableau_catalog("dopri5"), uf / 3, uf, 0.0, 1.0, n_steps)
    assert oc.rel_error(lam0, g["dopri5/lam0"]) <= 1e-4
    assert oc.rel_error(mu0, g["dopri5/mu0"]) <= 1e-4
