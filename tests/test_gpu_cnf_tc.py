"""GPU tests of the tcgen05 CNF tile (csrc/tc_cnf.cuh, config C4): the tensor-core
tile and the SIMT tile against the restated oracle, the cluster-padding tile (an
odd number of sample tiles is padded to whole clusters of two CTAs that share the
TMA weight stream), the input-only VJP (no parameter log), replays interleaved with
VJPs (revolve), and the field protocol at a tile that is not the bench's.

fp32 bar (north_star): 1e-4 inf-norm relative error against the fp64 oracle fed the
same fp32-rounded inputs.
"""

import numpy as np
import pytest
import torch

from oracle import core as oc
from oracle import fields_ext as ox
from paper_2206_01298_b200.configs import make_config
from paper_2206_01298_b200.workloads import field_from_config, initial_state, run_config

pytestmark = pytest.mark.gpu

TOL32 = 1e-4


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    from paper_2206_01298_b200 import _lib as L
    L.load()


def np_(x):
    return x.detach().cpu().numpy().astype(np.float64) if isinstance(x, torch.Tensor) else np.asarray(x)


def errs(res, ref):
    e = {k: oc.rel_error(np_(getattr(res, k)), ref[k]) for k in ("u_final", "du0", "dtheta")}
    e["loss"] = abs(res.loss - float(ref["loss"])) / abs(float(ref["loss"]))
    return e


@pytest.mark.parametrize("n,rows", [(63, 7), (5, 1), (40, 8)])
def test_tensor_core_and_simt_tiles_match_oracle(n, rows):
    """63 samples at 7 per tile = 9 tiles, padded to 10 (clusters of 2); 5 samples at 1
    per tile = 5 tiles + 1 padding tile; 40 at the widest tile (8 samples, N = 16)."""
    from oracle.problems import run_oracle
    ci = make_config("C4").subset(n)
    fld = field_from_config(ci)
    tc = run_config(ci, "store_all", field=fld, tile_rows=rows)
    si = run_config(ci, "store_all", field=fld, tile_rows=rows, tensor_cores=False)
    assert tc.device["tensor_cores"] == 1 and si.device["tensor_cores"] == 0
    assert tc.device["tiles"] % 2 == 0 and tc.device["tile_rows"] == rows
    ref = run_oracle(ci, "store_all")
    e_tc, e_si = errs(tc, ref), errs(si, ref)
    assert max(e_tc.values()) <= TOL32, e_tc
    assert max(e_si.values()) <= TOL32, e_si


def test_revolve_replays_bit_identical_to_store_all():
    """The reverse kernel interleaves replayed forward evaluations with VJPs (the weight
    stream's chunk ordinals and prefetch run across both); records and gradients must be
    bit-identical to store_all."""
    ci = make_config("C4").subset(21)
    fld = field_from_config(ci)
    u0 = torch.as_tensor(initial_state(ci), dtype=torch.float32, device="cuda")
    a = run_config(ci, "store_all", field=fld, u0=u0, tile_rows=3)
    b = run_config(ci, "revolve:3", field=fld, u0=u0, tile_rows=3)
    c = run_config(ci, "store_solutions", field=fld, u0=u0, tile_rows=3)
    assert b.device["steps_recomputed"] > 0
    for o in (b, c):
        assert torch.equal(a.dtheta, o.dtheta) and torch.equal(a.du0, o.du0) and a.loss == o.loss


def test_field_protocol_on_tensor_cores():
    """eval / vjp / vjp_u of the CNF field through ob_field_* (the tensor-core tile,
    one logged VJP per tile, finish() forms the parameter cotangent)."""
    ci = make_config("C4").subset(17)
    fld = field_from_config(ci)
    ofl = ox.CnfField(oc.Mlp(ci.widths, ci.activation, ci.theta, True), ci.extras["eps"])
    rng = np.random.default_rng(11)
    Y = initial_state(ci).astype(np.float32).astype(np.float64)
    Y[:, -1] = rng.standard_normal(ci.batch)
    V = rng.standard_normal(Y.shape).astype(np.float32).astype(np.float64)
    f_ref = ofl.eval(Y, 0.7, oc.Counters())
    j_ref, p_ref = ofl.vjp(Y, 0.7, V, oc.Counters())
    assert oc.rel_error(np_(fld.eval(Y, 0.7)), f_ref) <= TOL32
    j, p = fld.vjp(Y, 0.7, V)
    assert oc.rel_error(np_(j), j_ref) <= TOL32
    assert oc.rel_error(np_(p), p_ref) <= TOL32
    ju = fld.vjp_u(Y, 0.7, V)
    assert torch.equal(ju, j)


def test_bench_geometry_is_the_tensor_core_tile():
    ci = make_config("C4")
    res = run_config(ci, "store_all")
    assert res.device["tensor_cores"] == 1
    assert res.device["tile_rows"] == 7 and res.device["tiles"] == 144   # 143 + 1 padding tile
    assert np.isfinite(res.loss)
