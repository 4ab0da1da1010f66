"""Host-side loss semantics (reference tests/test_losses.py): LossSpec
validation and MinMaxScaling on the product's host mirror, and the oracle's
loss_and_grad_seed restatement on the reference's known-answer examples."""

import numpy as np
import pytest

from oracle import obs_losses as ol
from paper_2206_01298_b200.losses import LossSpec, MinMaxScaling, match_boundaries, terminal_loss


def _oracle(kind, preds, obs, scaling=None):
    """reference loss_and_grad_seed on one sample (B=1) through the oracle."""
    p = np.asarray(preds, float)[:, None, :]
    v = np.asarray(obs, float)[:, None, :]
    sc = ol.MinMax(scaling.lo, scaling.hi) if scaling is not None else None
    return ol.ObsLoss(kind, range(len(p)), v, sc).loss_and_seeds(p)


def test_known_answers_match_reference_examples():
    value, seeds = _oracle("mae", [[1.0, 2.0]], [[1.0, 3.0]])      # test_mae_example
    assert value == 0.5 and np.array_equal(seeds[0, 0], [0.0, -0.5])
    value, seeds = _oracle("mse", [[2.0]], [[0.0]])                  # test_mse_scalar_example
    assert value == 4.0 and seeds[0, 0, 0] == 4.0
    obs = [[0.1, -0.2, 0.3]]
    value, seeds = _oracle("mae", obs, obs)                          # zero loss, zero seeds
    assert value == 0.0 and np.array_equal(seeds[0, 0], np.zeros(3))
    _, seeds = _oracle("mae", [[1.0, 5.0]], [[1.0, 2.0]])            # subgradient at r = 0
    assert seeds[0, 0, 0] == 0.0
    value, seeds = _oracle("mse", [[1.0], [3.0]], [[0.0], [0.0]])    # multi-observation mean
    assert value == (1.0 + 9.0) / 2 and np.allclose(seeds[:, 0, 0], [1.0, 3.0])


def test_minmax_matches_reference_rules():
    s = MinMaxScaling(lo=np.array([0.0]), hi=np.array([4.0]))
    assert [s.apply(np.array([v]))[0] for v in (0.0, 2.0, 4.0)] == [0.0, 0.5, 1.0]
    s = MinMaxScaling(lo=np.array([2.0, 0.0]), hi=np.array([2.0, 1.0]))
    v = np.array([2.0, 0.5])
    assert np.array_equal(s.apply(v), v) and s.degenerate[0] and not s.degenerate[1]
    rng = np.random.default_rng(3)
    for _ in range(30):
        x = rng.uniform(-1e6, 1e6, rng.integers(3, 7))
        s = MinMaxScaling(lo=x.min() * np.ones(1), hi=x.max() * np.ones(1))
        span = max(1.0, float(x.max() - x.min()), float(np.max(np.abs(x))))
        for val in x:
            u = np.array([val])
            assert np.max(np.abs(s.invert(s.apply(u)) - u)) <= 1e-15 * span


def test_scaled_seed_matches_finite_differences():
    scaling = MinMaxScaling(lo=np.array([0.0, -1.0]), hi=np.array([2.0, 3.0]))
    obs = scaling.apply(np.array([1.5, 0.5]))
    pred = np.array([0.7, 1.2])
    _, seeds = _oracle("mse", [pred], [obs], scaling)
    eps = 1e-7
    for i in range(2):
        e = np.zeros(2)
        e[i] = eps
        fd = (_oracle("mse", [pred + e], [obs], scaling)[0]
              - _oracle("mse", [pred - e], [obs], scaling)[0]) / (2 * eps)
        assert abs(seeds[0, 0, i] - fd) <= 1e-7 * max(1.0, abs(fd))


def test_loss_spec_validation():
    with pytest.raises(ValueError):
        LossSpec("huber", (1.0,), (np.zeros(2),))
    with pytest.raises(ValueError):
        LossSpec("mae", (1.0, 0.5), (np.zeros(2), np.zeros(2)))
    with pytest.raises(ValueError):
        LossSpec("mae", (0.5, 1.0), (np.zeros(2), np.zeros(3)))
    with pytest.raises(ValueError):
        LossSpec("mse", (0.5, 1.0), (np.zeros(2),))
    with pytest.raises(ValueError):
        LossSpec("half_sqnorm", (0.5, 1.0))
    assert terminal_loss("mse", 1.0, np.zeros((4, 2))).n_obs == 1
    assert match_boundaries([0.0, 0.25, 1.0], np.linspace(0, 1, 5)) == [0, 1, 4]
    with pytest.raises(ValueError):
        match_boundaries([0.3], np.linspace(0, 1, 5))
