"""Pin the restated right-hand sides with no reference counterpart (C4 CNF,
C3 conv) by central finite differences and the adjoint identity, in the style
of the reference's own tests (pkg/tests/test_nn.py:112-201,
test_adjoint.py:248-261)."""

import numpy as np
import pytest

from oracle import core as oc
from oracle import fields_ext as ox


def _small_cnf(seed=0, D=5, H=7, B=3):
    rng = np.random.default_rng(seed)
    widths = (D + 1, H, H, D)
    from paper_2206_01298_b200.configs import xavier_uniform_mlp
    theta = xavier_uniform_mlp(rng, widths) + 0.1 * rng.standard_normal(
        sum(widths[l] * widths[l + 1] + widths[l + 1] for l in range(3)))
    mlp = oc.Mlp(widths, "softplus", theta, time_input=True)
    eps = rng.integers(0, 2, (B, D)) * 2.0 - 1.0
    Y = ox.cnf_initial_state(rng.standard_normal((B, D)))
    Y[:, D] = rng.standard_normal(B)
    return mlp, ox.CnfField(mlp, eps), Y, rng


def test_cnf_trace_term_matches_dense_jacobian():
    mlp, fld, Y, rng = _small_cnf()
    D = fld.D
    f = fld.eval(Y, 0.3, oc.Counters())
    for b in range(Y.shape[0]):
        J = np.zeros((D, D))
        for i in range(D):
            e = np.zeros((1, D + 1))
            e[0, i] = 1e-6
            fp = fld.eval(Y[b:b + 1] + e, 0.3, oc.Counters())[0, :D]
            fm = fld.eval(Y[b:b + 1] - e, 0.3, oc.Counters())[0, :D]
            J[:, i] = (fp - fm) / 2e-6
        eps = fld.eps[b]
        assert abs(f[b, D] - (-eps @ J @ eps)) <= 1e-7 * max(1.0, abs(f[b, D]))


def test_cnf_vjp_matches_finite_differences():
    mlp, fld, Y, rng = _small_cnf(seed=1)
    V = rng.standard_normal(Y.shape)
    t = 0.7
    jtv, ptv = fld.vjp(Y, t, V, oc.Counters())

    def phi_y(y):
        return float(np.sum(V * fld.eval(y, t, oc.Counters())))

    g = np.zeros_like(Y)
    for idx in np.ndindex(*Y.shape):
        e = np.zeros_like(Y)
        e[idx] = 1e-6
        g[idx] = (phi_y(Y + e) - phi_y(Y - e)) / 2e-6
    assert oc.rel_error(jtv, g) <= 1e-7

    def phi_th(th):
        f2 = ox.CnfField(oc.Mlp(mlp.widths, "softplus", th, True), fld.eps)
        return float(np.sum(V * f2.eval(Y, t, oc.Counters())))

    gt = np.zeros(mlp.n_params)
    for i in range(mlp.n_params):
        e = np.zeros(mlp.n_params)
        e[i] = 1e-6
        gt[i] = (phi_th(mlp.theta + e) - phi_th(mlp.theta - e)) / 2e-6
    assert oc.rel_error(ptv, gt) <= 1e-7


def test_cnf_full_gradient_matches_finite_differences():
    """Discrete adjoint through Dopri5 with the CNF field == FD of the loss."""
    mlp, fld, Y, rng = _small_cnf(seed=2, D=3, H=5, B=2)
    D, B = fld.D, Y.shape[0]
    seed = ox.cnf_seed(D, B)
    res = oc.grad_terminal(fld, "dopri5", Y, 0.0, 1.0, 4, seed_fn=seed)

    def loss_of(th=None, y0=None):
        f2 = fld if th is None else ox.CnfField(oc.Mlp(mlp.widths, "softplus", th, True), fld.eps)
        r = oc.grad_terminal(f2, "dopri5", Y if y0 is None else y0, 0.0, 1.0, 4, seed_fn=seed)
        return r["loss"]

    gt = np.array([(loss_of(th=mlp.theta + e) - loss_of(th=mlp.theta - e)) / 2e-6
                   for e in np.eye(mlp.n_params) * 1e-6])
    assert oc.rel_error(res["dtheta"], gt) <= 1e-6
    gy = np.zeros_like(Y)
    for idx in np.ndindex(*Y.shape):
        e = np.zeros_like(Y)
        e[idx] = 1e-6
        gy[idx] = (loss_of(y0=Y + e) - loss_of(y0=Y - e)) / 2e-6
    assert oc.rel_error(res["du0"], gy) <= 1e-6


def test_conv_vjp_matches_finite_differences():
    rng = np.random.default_rng(5)
    C, H = 3, 4
    n1, n2 = C * 9 * (C + 1), C * 9 * C
    theta = rng.standard_normal(n1 + n2 + 2 * C) * 0.3
    fld = ox.ConvField(theta, C=C, H=H, W=H)
    U = rng.standard_normal((2, H * H * C))
    V = rng.standard_normal(U.shape)
    jtv, ptv = fld.vjp(U, 0.6, V, oc.Counters())

    def phi(u=U, th=theta):
        f2 = ox.ConvField(th, C=C, H=H, W=H)
        return float(np.sum(V * f2.eval(u, 0.6, oc.Counters())))

    g = np.array([(phi(u=U + e.reshape(U.shape)) - phi(u=U - e.reshape(U.shape))) / 2e-6
                  for e in np.eye(U.size) * 1e-6]).reshape(U.shape)
    assert oc.rel_error(jtv, g) <= 1e-7
    gt = np.array([(phi(th=theta + e) - phi(th=theta - e)) / 2e-6 for e in np.eye(theta.size) * 1e-6])
    assert oc.rel_error(ptv, gt) <= 1e-7


def test_conv_head_loss_gradients_match_finite_differences():
    rng = np.random.default_rng(6)
    C, H, K = 3, 4, 5
    Uf = rng.standard_normal((3, H * H * C))
    head = rng.standard_normal(K * C + K)
    labels = rng.integers(0, K, 3)
    loss, lam, dhead = ox.head_loss(Uf, head, labels, C=C, H=H, W=H, n_classes=K)
    f = lambda u, h: ox.head_loss(u, h, labels, C=C, H=H, W=H, n_classes=K)[0]   # noqa: E731
    g = np.array([(f(Uf + e.reshape(Uf.shape), head) - f(Uf - e.reshape(Uf.shape), head)) / 2e-6
                  for e in np.eye(Uf.size) * 1e-6]).reshape(Uf.shape)
    assert oc.rel_error(lam, g) <= 1e-7
    gh = np.array([(f(Uf, head + e) - f(Uf, head - e)) / 2e-6 for e in np.eye(head.size) * 1e-6])
    assert oc.rel_error(dhead, gh) <= 1e-7
