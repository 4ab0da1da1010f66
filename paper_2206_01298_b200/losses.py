"""Terminal losses (reference LossSpec / terminal_loss, losses.py:40-107).

Batched semantics: the loss is the mean over samples of a per-sample terminal
loss, so the seed is lambda_N,b = grad ell(u_b(T)) / B.
  * ``half_sqnorm``: ell(u) = 0.5 ||u||^2 (the BASELINE configs' loss).
  * ``mse``: ell(u) = sum((u - y)^2) / N with per-sample targets y, i.e. the
    reference's K=1 MSE (seed 2 r / N, losses.py:100-107), averaged over B.
  * ``ce_head``: for ConvField states: global-average-pool + linear 64 -> 10
    + softmax cross-entropy; values = (head params [10*64 + 10], labels [B]);
    the head gradient comes back as GradResult.dtheta_head.
  * ``cnf_nll``: for CnfField states [z, Delta]: -log p(x) = 0.5||z||^2 +
    D/2 log(2 pi) + Delta (standard-normal base, log p(x) = log N(z(1)) - Delta(1)).
Multi-observation losses, MAE and min-max scaling are the next component
 and raise NotImplementedError.
"""

from __future__ import annotations

from dataclasses import dataclass

KINDS = ("half_sqnorm", "mse", "cnf_nll", "ce_head")


@dataclass(frozen=True)
class LossSpec:
    kind: str
    times: tuple
    values: object = None      # mse: targets [B, N] (host or device)
    scaling: object = None

    def __post_init__(self):
        if self.kind not in KINDS:
            raise NotImplementedError(f"loss kind {self.kind!r} is not built (SURVEY 8f row 3)")
        ts = tuple(float(t) for t in self.times)
        object.__setattr__(self, "times", ts)
        if len(ts) != 1:
            raise NotImplementedError("multi-observation losses are not built (SURVEY 8f row 3)")
        if self.scaling is not None:
            raise NotImplementedError("min-max scaling is not built (SURVEY 8f row 3)")
        if self.kind == "mse" and self.values is None:
            raise ValueError("mse needs observed targets")
        if self.kind == "ce_head" and (self.values is None or len(self.values) != 2):
            raise ValueError("ce_head needs (head parameters, labels)")

    @property
    def n_obs(self) -> int:
        return len(self.times)


def terminal_loss(kind, t_final, observed=None, scaling=None) -> LossSpec:
    return LossSpec(kind, (t_final,), observed, scaling)
