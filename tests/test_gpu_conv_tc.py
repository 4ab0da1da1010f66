"""GPU tests of the tcgen05 conv tile (csrc/tc_conv.cuh): the C3 block's implicit-GEMM
convolutions on the tensor cores with an fp16 two-term split, one stencil tap per TMEM
partial (round-to-nearest sums in registers), against the restated fp64 oracle
(oracle/fields_ext.py ConvField) and the fp32 SIMT tile.

The accuracy claims the tile's design rests on are tested here, not only the 1e-4 bar:
the field value and VJP are at fp32-FMA-chain level (a few 1e-7), far below what a
single TMEM accumulation chain (3.7e-6, truncating adds) or a bf16 split (2^-16) gives.
"""

import numpy as np
import pytest
import torch

from oracle import core as oc
from oracle import fields_ext as ox
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
    return x.detach().cpu().numpy().astype(np.float64) if isinstance(x, torch.Tensor) else np.asarray(x)


def _blocks(v):
    """theta-shaped vector -> (W1 [64, 9, 65], b1, W2 [64, 9, 64], b2)."""
    n1, n2 = 64 * 9 * 65, 64 * 9 * 64
    return (v[:n1].reshape(64, 9, 65), v[n1:n1 + 64], v[n1 + 64:n1 + 64 + n2].reshape(64, 9, 64),
            v[n1 + 64 + n2:])


@pytest.mark.parametrize("t", [0.0, 0.35, 1.0])
def test_field_eval_and_vjp_at_fp32_level(t):
    """Field protocol through the tile (ob_field_eval / ob_field_vjp run it for conv
    fields): f, J^T v and every block of P^T v -- both convs' weights, both biases and
    the time channel, which the tile handles outside the MMAs (border-class bias forward,
    indicator product backward) -- within 2e-6 of the fp64 oracle."""
    ci = make_config("C3").subset(5)
    fld = field_from_config(ci)
    ofl = ox.ConvField(ci.theta)
    rng = np.random.default_rng(11)
    U = ci.u0.reshape(5, -1)
    V = rng.standard_normal(U.shape).astype(np.float32).astype(np.float64)
    f_ref = ofl.eval(U, t, oc.Counters())
    j_ref, p_ref = ofl.vjp(U, t, V, oc.Counters())
    assert oc.rel_error(np_(fld.eval(U, t)), f_ref) <= 1e-6
    j, p = fld.vjp(U, t, V)
    assert oc.rel_error(np_(j), j_ref) <= 2e-6
    for got, want, name in zip(_blocks(np_(p)), _blocks(p_ref), ("W1", "b1", "W2", "b2")):
        assert oc.rel_error(got, want) <= 2e-6, name
    if t != 0.0:
        assert oc.rel_error(_blocks(np_(p))[0][:, :, 64], _blocks(p_ref)[0][:, :, 64]) <= 2e-6   # time channel
    assert oc.rel_error(np_(fld.vjp_u(U, t, V)), j_ref) <= 2e-6


def test_field_wide_dynamic_range():
    """Per-tile power-of-two scaling: inputs and cotangents of very different magnitudes
    (1e-6 .. 1e3) keep their relative accuracy (fp16 has 5 exponent bits; the tile
    rescales every operand image to its own maximum)."""
    ci = make_config("C3").subset(4)
    fld = field_from_config(ci)
    ofl = ox.ConvField(ci.theta)
    rng = np.random.default_rng(5)
    U = ci.u0.reshape(4, -1).copy()
    V = rng.standard_normal(U.shape)
    for b, (su, sv) in enumerate(((1e-6, 1e3), (1e3, 1e-6), (1.0, 1e-9), (37.0, 1.0))):
        U[b] *= su
        V[b] *= sv
    U = U.astype(np.float32).astype(np.float64)
    V = V.astype(np.float32).astype(np.float64)
    f = np_(fld.eval(U, 0.5))
    j = np_(fld.vjp_u(U, 0.5, V))
    f_ref = ofl.eval(U, 0.5, oc.Counters())
    j_ref = ofl.vjp_u(U, 0.5, V, oc.Counters())
    for b in range(4):   # per image: each has its own scale
        assert oc.rel_error(f[b], f_ref[b]) <= 2e-6, b
        assert oc.rel_error(j[b], j_ref[b]) <= 2e-6, b


def test_tensor_core_tile_is_the_default_and_matches_simt():
    """grad() on a conv field runs the tcgen05 tile unless tensor_cores=False; both tiles
    agree with each other far inside the fp32 bar wherever no ReLU kink separates them
    (u_final, loss, dtheta), and the tile reports itself."""
    ci = make_config("C3").subset(8)
    fld = field_from_config(ci)
    tc = run_config(ci, "store_all", field=fld)
    si = run_config(ci, "store_all", field=fld, tensor_cores=False)
    assert tc.device["tensor_cores"] == 1 and si.device["tensor_cores"] == 0
    assert tc.device["tiles"] == 8 and tc.device["kernel_launches"] == 4
    assert oc.rel_error(np_(tc.u_final), np_(si.u_final)) <= 5e-6
    assert abs(tc.loss - si.loss) <= 5e-6 * abs(si.loss)
    assert oc.rel_error(np_(tc.dtheta), np_(si.dtheta)) <= TOL32
    assert tc.counters.nfe_forward == si.counters.nfe_forward == 40


def test_loss_and_gradients_bit_reproducible():
    """Fixed-order sums everywhere (per-CTA mu slots, register sums of the tap partials in
    tap order, tile-ordered reduction): two runs give identical bits."""
    ci = make_config("C3").subset(5)
    fld = field_from_config(ci)
    a = run_config(ci, "store_all", field=fld)
    b = run_config(ci, "store_all", field=fld)
    assert a.loss == b.loss
    for k in ("u_final", "du0", "dtheta", "dtheta_head"):
        assert np.array_equal(np_(getattr(a, k)), np_(getattr(b, k))), k


@pytest.mark.parametrize("scheme,policy", [("euler", "store_all"), ("midpoint", "store_solutions"),
                                           ("bosh3", "revolve:2"), ("dopri5", "revolve:3")])
def test_other_schemes_and_policies(scheme, policy):
    """The tile owns its RK steps (stage sums in registers, FSAL carry, skipped zero-cotangent
    stages): every explicit scheme / policy the generic kernels support, against the oracle
    and bit-identical to store_all."""
    from _kinks import check_du0_with_kinks
    from oracle.problems import run_oracle
    import dataclasses

    def make():
        c = make_config("C3").subset(3)
        return dataclasses.replace(c, scheme=scheme, n_steps=4)

    ci = make()
    assert ci.scheme == scheme
    fld = field_from_config(ci)
    res = run_config(ci, policy, field=fld)
    base = run_config(ci, "store_all", field=fld)
    assert res.device["tensor_cores"] == 1
    assert np.array_equal(np_(res.dtheta), np_(base.dtheta)) and res.loss == base.loss
    ref = run_oracle(ci, "store_all")
    for k in ("u_final", "dtheta"):
        assert oc.rel_error(np_(getattr(res, k)), ref[k]) <= TOL32, k
    check_du0_with_kinks(make, np_(res.du0), ref["du0"], TOL32, max_over=1)


@pytest.mark.timeout(300)
def test_full_batch_repeated_runs_identical():
    """Two waves of CTAs (256 images on 148 SMs), eight gradients in a row: identical bits
    every time.  The tile's six issuing warps, accumulator ring and weight ring synchronise
    through ~20 mbarriers; a protocol slip shows up here as differing bits or a hang (one
    did: a warp that skipped a weight phase read the next parity as complete)."""
    ci = make_config("C3")
    fld = field_from_config(ci)
    u0 = torch.as_tensor(ci.u0.reshape(ci.batch, -1), dtype=torch.float32, device="cuda")
    first = run_config(ci, "store_all", field=fld, u0=u0)
    for _ in range(7):
        r = run_config(ci, "store_all", field=fld, u0=u0)
        assert r.loss == first.loss
        assert torch.equal(r.dtheta, first.dtheta) and torch.equal(r.du0, first.du0)


def test_non_finite_input_raises():
    ci = make_config("C3").subset(2)
    fld = field_from_config(ci)
    u0 = ci.u0.reshape(2, -1).copy()
    u0[1, 77] = np.nan
    with pytest.raises(ValueError):
        run_config(ci, "store_all", field=fld, u0=u0)
