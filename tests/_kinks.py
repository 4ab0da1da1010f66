"""Shared check for the C3 block's ReLU kinks (test helper, not a test module).

The discrete adjoint of conv -> relu -> conv is discontinuous where a pre-activation
crosses zero: a value within rounding of 0 flips ReLU' between an fp32 device run and
the fp64 oracle and moves lambda locally by O(|W| h |lambda|).  du0 therefore meets the
fp32 bar on every image except a few; for each of those the check shows that the
ORACLE ITSELF jumps by a comparable amount when that image's input is perturbed at
fp32-rounding size (2^-20 relative), i.e. the difference is the problem's conditioning
at the kink, not an arithmetic error of the device path.
"""

import numpy as np


def check_du0_with_kinks(make_ci, du0, ref_du0, tol, max_over, median_tol=2e-6, seed=0):
    """make_ci() -> a fresh ConfigInputs of the batch; du0 / ref_du0: [B, N].
    Returns (per-image error, indices over the bar)."""
    from oracle.problems import run_oracle

    du0 = np.asarray(du0, dtype=np.float64)
    scale = np.max(np.abs(ref_du0))
    per = np.max(np.abs(du0 - ref_du0), axis=1) / scale
    assert np.median(per) <= median_tol, float(np.median(per))
    over = np.nonzero(per > tol)[0]
    assert len(over) <= max_over, per[over]
    rng = np.random.default_rng(seed)
    for b in over:
        base = run_oracle(make_ci(), "store_all", rows=slice(b, b + 1))["du0"][0]
        jump = 0.0
        for _ in range(12):
            c2 = make_ci()
            c2.u0[b] = c2.u0[b] * (1 + rng.uniform(-1, 1, size=c2.u0[b].shape) * 2.0 ** -20)
            p = run_oracle(c2, "store_all", rows=slice(b, b + 1))["du0"][0]
            jump = max(jump, np.max(np.abs(p - base)) / scale)
            if jump >= 0.3 * per[b]:
                break
        assert jump >= 0.3 * per[b], (int(b), float(per[b]), float(jump))
    return per, over
