"""AdamW for the oracle (TEST INFRASTRUCTURE ONLY -- imported by tests/, never
by the product): restates adamw_step (training.py:175-190) in numpy with the
reference's evaluation order."""

import numpy as np


def adamw_step(theta, g, m, v, step, lr=0.005, beta1=0.9, beta2=0.999, eps=1e-8,
               weight_decay=0.0):
    """One decoupled-weight-decay Adam update; returns (theta', m', v', step')."""
    g = np.asarray(g, dtype=np.float64)
    if not np.all(np.isfinite(g)):
        raise FloatingPointError("non-finite gradient passed to the optimizer")
    t = step + 1
    theta = theta * (1.0 - lr * weight_decay)
    m = beta1 * m + (1.0 - beta1) * g
    v = beta2 * v + (1.0 - beta2) * g * g
    m_hat = m / (1.0 - beta1 ** t)
    v_hat = v / (1.0 - beta2 ** t)
    theta = theta - lr * m_hat / (np.sqrt(v_hat) + eps)
    return theta, m, v, t
