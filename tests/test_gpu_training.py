"""GPU parity for the training loop: the device AdamW update
(csrc/optim.cu, training.py:175-190) bit-identical to the reference in fp64,
the fixed-order gradient norm, short full-batch ``train`` runs (Crank-Nicolson
on the geometric grid; adaptive Dopri5) against the reference's own train() on
a reference-generated Robertson dataset (tests/golden/training.npz), and the
model JSON format (nn.py:190-220).

Tolerances: AdamW fp64 bit-exact; train() losses / gradient norms / final
parameters <= 1e-9 relative (each epoch's gradient is pinned at 1e-10 and the
optimizer is exact, so differences stay at rounding level); NFE counts exact.
"""

import numpy as np
import pytest
import torch

from oracle import core as oc
from paper_2206_01298_b200 import GradientExplosionError, MlpModel, MlpSpec, tableau_catalog
from paper_2206_01298_b200 import formats, training as tr

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    from paper_2206_01298_b200 import _lib as L
    L.load()


def dev(x, dt=torch.float64):
    return torch.as_tensor(np.asarray(x), dtype=dt, device="cuda").contiguous()


def test_adamw_bit_identical_to_reference(golden):
    g = golden("training.npz")
    theta = dev(g["adamw/theta0"])
    st = tr.OptimizerState.zeros(50)
    cfg = tr.AdamWConfig(lr=0.01, weight_decay=0.1)
    for k in range(4):
        theta, st = tr.adamw_step(theta, dev(g[f"adamw/g{k}"]), st, cfg)
        assert np.array_equal(theta.cpu().numpy(), g[f"adamw/theta{k + 1}"])
        assert np.array_equal(st.m.cpu().numpy(), g[f"adamw/m{k + 1}"])
        assert np.array_equal(st.v.cpu().numpy(), g[f"adamw/v{k + 1}"])
    assert st.step == 4


def test_adamw_fp32_and_nonfinite(golden):
    g = golden("training.npz")
    theta = dev(g["adamw/theta0"], torch.float32)
    st = tr.OptimizerState.zeros(50, torch.float32)
    theta, st = tr.adamw_step(theta, dev(g["adamw/g0"], torch.float32), st,
                              tr.AdamWConfig(lr=0.01, weight_decay=0.1))
    assert np.max(np.abs(theta.cpu().numpy() - g["adamw/theta1"])) <= 1e-6
    bad = dev(g["adamw/g1"])
    bad[7] = float("nan")
    th = dev(g["adamw/theta0"])
    st = tr.OptimizerState.zeros(50)
    before = th.clone()
    with pytest.raises(GradientExplosionError):
        tr.adamw_step(th, bad, st, tr.AdamWConfig())
    assert torch.equal(th, before) and st.step == 0 and not bool(st.m.any())


def test_grad_norm_fixed_order():
    rng = np.random.default_rng(4)
    x = rng.standard_normal(100_003)
    n1 = tr.grad_norm(dev(x))
    assert abs(n1 - np.linalg.norm(x)) <= 1e-13 * np.linalg.norm(x)
    assert n1 == tr.grad_norm(dev(x))            # deterministic
    x[5] = np.inf
    assert not np.isfinite(tr.grad_norm(dev(x)))


def _dataset(g):
    return tr.Dataset(g["data/times"], list(g["data/obs"]))


@pytest.mark.parametrize("sch", ["cn", "dopri5"])
def test_train_matches_reference(golden, sch):
    g = golden("training.npz")
    model = MlpModel(MlpSpec((3, 8, 3), "tanh"), g["model/theta"])
    if sch == "cn":
        cfg = tr.TrainConfig(epochs=4, n_sub=3, loss_kind="mae", optimizer=tr.AdamWConfig(lr=0.01))
    else:
        cfg = tr.TrainConfig(epochs=3, loss_kind="mse", abstol=1e-6, reltol=1e-6,
                             optimizer=tr.AdamWConfig(lr=0.02, weight_decay=0.01))
    _, rec = tr.train(model, tableau_catalog(sch), _dataset(g), cfg)
    pre = f"train_{sch}/"
    assert rec.aborted == ""
    assert oc.rel_error(rec.loss, g[pre + "loss"]) <= 1e-9
    assert oc.rel_error(rec.grad_norm, g[pre + "grad_norm"]) <= 1e-9
    assert list(rec.nfe_forward) == list(g[pre + "nfe_forward"])
    assert list(rec.nfe_backward) == list(g[pre + "nfe_backward"])
    assert oc.rel_error(rec.final_theta, g[pre + "final_theta"]) <= 1e-9


def test_train_explosion_and_zero_epochs(golden):
    g = golden("training.npz")
    model = MlpModel(MlpSpec((3, 8, 3), "tanh"), g["model/theta"])
    _, rec = tr.train(model, tableau_catalog("cn"), _dataset(g),
                      tr.TrainConfig(epochs=3, n_sub=3, explosion_threshold=1e-6))
    assert rec.aborted == "gradient_explosion" and rec.abort_epoch == 0
    assert np.array_equal(rec.final_theta, g["model/theta"])
    m2, rec = tr.train(model, tableau_catalog("cn"), _dataset(g), tr.TrainConfig(epochs=0, n_sub=3))
    assert len(rec.loss) == 1 and np.isfinite(rec.loss[0])


def test_model_json_matches_reference(golden, tmp_path):
    g = golden("training.npz")
    model = MlpModel(MlpSpec((3, 8, 3), "tanh"), g["model/theta"])
    assert formats.model_to_json(model) == str(g["model/json"])
    p = tmp_path / "m.json"
    formats.save_model(model, p)
    back = formats.load_model(p)
    assert back.spec == model.spec and torch.equal(back.theta, model.theta)
