"""TEST INFRASTRUCTURE ONLY -- restated right-hand sides with no reference
counterpart (C3 conv block, C4 CNF), in float64, with the batched Field
protocol of oracle/core.py so the restated reference integrator / adjoint
(core.grad_terminal) drives them unchanged (the reference's
CallableField plugin, integrators.py:105-141).

Parity for these is "restated RHS": nothing in the reference pins them; they
are pinned here by central finite differences and the adjoint identity
(tests/test_oracle_ext.py), in the style of pkg/tests/test_nn.py:112-201.
"""

from __future__ import annotations

import numpy as np

from .core import Mlp, act, act_prime, act_second

LOG2PI = float(np.log(2.0 * np.pi))


class CnfField:
    """Continuous normalizing flow with a Hutchinson trace estimator.

    State y = [z (D), Delta]; f_aug(y, t) = [f(z, t), -eps^T (df/dz) eps] with a
    fixed Rademacher probe eps per sample and f an MLP with time appended to
    its input.  The VJP needs the second-order terms of eps^T J eps
    (forward-over-reverse through the tangent chain).
    """

    def __init__(self, mlp: Mlp, eps):
        assert mlp.time_input
        self.mlp = mlp
        self.eps = np.asarray(eps, dtype=np.float64)   # [B, D]
        self.D = mlp.widths[-1]
        self.n = self.D + 1
        self.n_params = mlp.n_params

    def _chains(self, Z, t, eps):
        """Forward (z_l, a_l) and tangent (s_l raw, u_l) chains of every layer."""
        m = self.mlp
        B = Z.shape[0]
        a = np.concatenate([Z, np.full((B, 1), float(t))], axis=1)
        u = np.concatenate([eps, np.zeros((B, 1))], axis=1)
        A, U, Zs, S = [a], [u], [], []
        L = len(m.layers)
        for l in range(L):
            W, b = m.W(l), m.b(l)
            z = a @ W.T + b
            s = u @ W.T
            Zs.append(z)
            S.append(s)
            if l < L - 1:
                a = act(z, m.activation)
                u = act_prime(z, m.activation) * s
                A.append(a)
                U.append(u)
        return A, U, Zs, S

    def _eps(self, B):
        return self.eps[:B] if self.eps.shape[0] != B else self.eps

    def eval(self, Y, t, c):
        c.nfe_forward += 1
        Z = Y[:, :self.D]
        eps = self._eps(Y.shape[0])
        _, _, Zs, S = self._chains(Z, t, eps)
        f = Zs[-1]
        g = -np.sum(eps * S[-1], axis=1, keepdims=True)
        return np.concatenate([f, g], axis=1)

    def vjp(self, Y, t, V, c, want_theta=True):
        c.nfe_backward += 1
        m = self.mlp
        Z = Y[:, :self.D]
        eps = self._eps(Y.shape[0])
        A, U, Zs, S = self._chains(Z, t, eps)
        vz = V[:, :self.D]
        vd = V[:, self.D:self.D + 1]
        L = len(m.layers)
        dth = np.zeros(m.n_params)
        zbar = vz                      # cotangent of the last layer's output z_L
        sbar = -vd * eps               # cotangent of its tangent output s_L
        for l in range(L - 1, -1, -1):
            o, ob, nin, nout = m.layers[l]
            W = m.W(l)
            if want_theta:
                dth[o:ob] = (zbar.T @ A[l] + sbar.T @ U[l]).ravel()
                dth[ob:ob + nout] = zbar.sum(axis=0)
            abar = zbar @ W
            ubar = sbar @ W
            if l > 0:
                z, s = Zs[l - 1], S[l - 1]
                sp = act_prime(z, m.activation)
                spp = act_second(z, m.activation)
                sbar = sp * ubar
                zbar = spp * s * ubar + sp * abar
            else:
                jz = abar[:, :self.D]
        jtv = np.concatenate([jz, np.zeros((Y.shape[0], 1))], axis=1)
        return jtv, dth

    def vjp_u(self, Y, t, V, c):
        return self.vjp(Y, t, V, c, want_theta=False)[0]


def cnf_seed(D, B):
    """NLL = 0.5||z(1)||^2 + D/2 log(2 pi) + Delta(1) per sample, batch mean:
    (loss, lambda_N) with lambda_N = [z/B, 1/B]."""
    def seed(Y):
        z = Y[:, :D]
        nll = 0.5 * np.sum(z * z, axis=1) + 0.5 * D * LOG2PI + Y[:, D]
        lam = np.concatenate([z / B, np.full((Y.shape[0], 1), 1.0 / B)], axis=1)
        return float(np.mean(nll)) if Y.shape[0] == B else float(np.sum(nll) / B), lam
    return seed


def cnf_initial_state(z0):
    """[z0, Delta=0]."""
    z0 = np.asarray(z0, dtype=np.float64)
    return np.concatenate([z0, np.zeros((z0.shape[0], 1))], axis=1)


# --------------------------------------------------------------------- C3 conv
def _im2col(X):
    """[B, H, W, C] -> [B, H*W, 9*C] patches of a 3x3 stencil with zero padding 1,
    patch order (kh, kw, c) matching weights stored [Cout][kh][kw][Cin]."""
    B, H, W, C = X.shape
    Xp = np.zeros((B, H + 2, W + 2, C))
    Xp[:, 1:-1, 1:-1] = X
    cols = [Xp[:, kh:kh + H, kw:kw + W, :] for kh in range(3) for kw in range(3)]
    return np.concatenate(cols, axis=3).reshape(B, H * W, 9 * C)


def _col2im(G, H, W, C):
    """Adjoint of _im2col: [B, H*W, 9*C] -> [B, H, W, C]."""
    B = G.shape[0]
    G = G.reshape(B, H, W, 9, C)
    Xp = np.zeros((B, H + 2, W + 2, C))
    s = 0
    for kh in range(3):
        for kw in range(3):
            Xp[:, kh:kh + H, kw:kw + W, :] += G[:, :, :, s, :]
            s += 1
    return Xp[:, 1:-1, 1:-1]


class ConvField:
    """C3 ODE block: f(u, t) = conv3x3(C+1 -> C)(cat(u, t)) -> relu -> conv3x3(C -> C),
    padding 1, NHWC state flattened to [B, H*W*C].  theta = [W1 (C x 3 x 3 x (C+1)),
    b1, W2 (C x 3 x 3 x C), b2] (paper_2206_01298_b200/configs.py make_c3)."""

    def __init__(self, theta, C=64, H=16, W=16):
        self.C, self.H, self.W = C, H, W
        th = np.asarray(theta, dtype=np.float64)
        n1 = C * 9 * (C + 1)
        n2 = C * 9 * C
        self.W1 = th[:n1].reshape(C, 9 * (C + 1))
        self.b1 = th[n1:n1 + C]
        self.W2 = th[n1 + C:n1 + C + n2].reshape(C, 9 * C)
        self.b2 = th[n1 + C + n2:n1 + 2 * C + n2]
        self.n_params = th.size
        self.n = H * W * C

    def _fwd(self, U, t):
        B = U.shape[0]
        X = np.concatenate([U.reshape(B, self.H, self.W, self.C),
                            np.full((B, self.H, self.W, 1), float(t))], axis=3)
        P1 = _im2col(X)
        Z1 = P1 @ self.W1.T + self.b1
        Hh = np.maximum(Z1, 0.0)
        P2 = _im2col(Hh.reshape(B, self.H, self.W, self.C))
        F = P2 @ self.W2.T + self.b2
        return P1, Z1, P2, F

    def eval(self, U, t, c):
        c.nfe_forward += 1
        return self._fwd(U, t)[3].reshape(U.shape[0], -1)

    def vjp(self, U, t, V, c, want_theta=True):
        c.nfe_backward += 1
        B, C = U.shape[0], self.C
        P1, Z1, P2, _ = self._fwd(U, t)
        Vr = V.reshape(B, self.H * self.W, C)
        dH = _col2im(Vr @ self.W2, self.H, self.W, C).reshape(B, self.H * self.W, C)
        dZ1 = dH * (Z1 > 0.0)
        dX = _col2im(dZ1 @ self.W1, self.H, self.W, C + 1)[..., :C]
        dth = None
        if want_theta:
            dW1 = np.einsum("bpo,bpk->ok", dZ1, P1)
            dW2 = np.einsum("bpo,bpk->ok", Vr, P2)
            dth = np.concatenate([dW1.ravel(), dZ1.sum(axis=(0, 1)), dW2.ravel(),
                                  Vr.sum(axis=(0, 1))])
        return dX.reshape(B, -1), dth

    def vjp_u(self, U, t, V, c):
        return self.vjp(U, t, V, c, want_theta=False)[0]


def head_loss(Uf, head, labels, C=64, H=16, W=16, n_classes=10, batch_global=None):
    """Global-average-pool + linear C -> n_classes + cross-entropy, batch mean.
    Returns (loss, lambda_N [B, H*W*C], dhead [n_classes*C + n_classes])."""
    B = Uf.shape[0]
    Bg = batch_global or B
    Wh = head[:n_classes * C].reshape(n_classes, C)
    bh = head[n_classes * C:]
    gap = Uf.reshape(B, H * W, C).mean(axis=1)
    logits = gap @ Wh.T + bh
    m = logits.max(axis=1, keepdims=True)
    ex = np.exp(logits - m)
    lse = m[:, 0] + np.log(ex.sum(axis=1))
    loss = float(np.sum(lse - logits[np.arange(B), labels]) / Bg)
    dlog = ex / ex.sum(axis=1, keepdims=True)
    dlog[np.arange(B), labels] -= 1.0
    dlog /= Bg
    dgap = dlog @ Wh
    lam = np.repeat(dgap[:, None, :] / (H * W), H * W, axis=1).reshape(B, -1)
    dhead = np.concatenate([(dlog.T @ gap).ravel(), dlog.sum(axis=0)])
    return loss, lam, dhead
