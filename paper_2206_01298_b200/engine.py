"""grad(): forward integration + checkpoints + discrete adjoint on the device
(reference adjoint.py:224-279: forward_pass :151-210, loss_and_grad_seed
losses.py:78-107, backward_sweep :235-253), batched over samples.

One call = one ``ob_grad`` into the native engine: two persistent kernels
(forward sweep, reverse program) plus weight packing and a fixed-order
reduction.  Host inputs (numpy arrays / CPU tensors) are copied to the device
and results copied back; device inputs stay on the device.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field as dc_field

import numpy as np
import torch

from . import _lib
from .controls import (AdaptiveController, NfeCounters, SolverConfig, StoreCounters, boundary_times,
                       raise_status)
from .fields import Field, stream_ptr, to_device
from .losses import OBSERVATION_KINDS, LossSpec, match_boundaries
from .policies import CheckpointPolicy
from .schemes import Scheme, to_desc


@dataclass
class GradResult:
    dtheta: object
    du0: object
    loss: float
    counters: NfeCounters
    predictions: list
    u_final: object
    store_counters: StoreCounters = None
    device: dict = dc_field(default_factory=dict)
    # per-sample reference counters (numpy int arrays over the batch): nfe_forward,
    # nfe_backward, newton_iters, gmres_iters_forward, gmres_iters_adjoint
    # (implicit schemes; explicit ones repeat the schedule-fixed counts)
    sample_counters: dict = None
    dtheta_head: object = None      # ce_head loss: gradient of the classification head
    # adaptive stepping: per-sample boundary times (t0, t_n + h_n; adjoint.py:171-173)
    grids: list = None


_WS_CACHE = {}


def _workspace(nbytes: int, device) -> torch.Tensor:
    key = (device.index,)
    buf = _WS_CACHE.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=device)
        _WS_CACHE[key] = buf
    return buf


def build_problem(field: Field, scheme: Scheme, loss: LossSpec, batch: int, ts: np.ndarray,
                  policy: CheckpointPolicy, solver_cfg: SolverConfig, batch_global: int):
    prob = _lib.Problem()
    prob.field = field.desc()
    prob.scheme = to_desc(scheme)
    prob.solver = solver_cfg.to_desc()
    prob.batch = batch
    prob.batch_global = batch_global
    prob.n_steps = len(ts) - 1
    prob.policy = _lib.OB_POLICY[policy.kind]
    prob.nc = policy.nc
    prob.loss = _lib.OB_LOSS[loss.kind]
    times = np.ascontiguousarray(ts, dtype=np.float64)
    prob.times = times.ctypes.data_as(C.POINTER(C.c_double))
    return prob, times


def workspace_size(prob) -> int:
    n = C.c_size_t()
    raise_status(_lib.load().ob_grad_workspace_size(C.byref(prob), C.byref(n)), _lib.last_error())
    return int(n.value)


def phase_cycles(reset=True):
    """Per-phase SM-cycle totals of the last profiled calls (grad(..., profile=True))."""
    buf = (C.c_uint64 * 16)()
    raise_status(_lib.load().ob_debug_phase_cycles(buf, 16, int(reset)), _lib.last_error())
    names = ["elementwise", "recompute", "vjp", "lam_update", "replay", "fwd_step", "gmres_apply",
             "gmres_scalar", "step_combine", "step_eval", "fwd_hidden|tc_mma", "fwd_out|tc_epilogue",
             "fwd_out_split", "fwd_out_reduce", "gmres_input|tc_prep", "p15"]
    return {n: int(buf[i]) for i, n in enumerate(names)}


def grad(field: Field, scheme: Scheme, loss: LossSpec, u0, t0, tF, ctrl,
         policy=CheckpointPolicy("store_all"), solver_cfg=None, counters=None, *,
         batch_global=None, profile=False, tensor_cores=True) -> GradResult:
    """Loss, dL/dtheta and dL/du0 by forward solve + discrete adjoint sweep.

    ``tensor_cores=False`` forces the SIMT (FMA) MLP tile where the tcgen05
    tile would apply (fp32 two-layer MLP fields on explicit fixed-step schemes).
    """
    solver_cfg = solver_cfg or SolverConfig()
    counters = counters if counters is not None else NfeCounters()
    if loss.times[-1] > tF + 1e-9 * max(1.0, abs(tF)):
        raise ValueError("observations extend past the final time")
    obs = loss.kind in OBSERVATION_KINDS
    if not obs and abs(loss.times[-1] - tF) > 1e-9 * max(1.0, abs(tF)):
        raise ValueError(f"{loss.kind} is a terminal loss at tF")
    adaptive = isinstance(ctrl, AdaptiveController)
    if adaptive:
        if tF <= t0:
            raise ValueError("tF must exceed t0")
        ts = np.array([t0, tF], dtype=np.float64)
        obs_steps = None
    else:
        ts = boundary_times(ctrl, t0, tF)
        obs_steps = match_boundaries(loss.times, ts) if obs else None
    host_io = not (isinstance(u0, torch.Tensor) and u0.is_cuda)
    dt = field.torch_dtype
    if isinstance(u0, torch.Tensor) and not u0.is_cuda:
        u0d = u0.to(device=torch.device("cuda", torch.cuda.current_device()), dtype=dt,
                    non_blocking=True).contiguous()
    else:
        u0d = to_device(u0, dt)
    if u0d.dim() == 1:
        u0d = u0d.unsqueeze(0)
    B, N = u0d.shape
    if N != field.n:
        raise ValueError(f"expected length {field.n}, got {N}")
    bg = int(batch_global) if batch_global is not None else B
    prob, _times = build_problem(field, scheme, loss, B, ts, policy, solver_cfg, bg)
    prob.flags = (1 if profile else 0) | (0 if tensor_cores else 2)
    if adaptive:
        prob.adaptive = 1
        prob.n_steps = 0
        prob.max_accepted = int(ctrl.max_accepted)
        prob.abstol, prob.reltol = float(ctrl.abstol), float(ctrl.reltol)
        prob.h_init, prob.h_min = float(ctrl.h_init), float(ctrl.h_min)
        prob.h_max, prob.safety = float(ctrl.h_max), float(ctrl.safety)
        prob.max_steps = int(ctrl.max_steps)
        prob.t0, prob.tF = float(t0), float(tF)
        if obs:
            otimes = (C.c_double * len(loss.times))(*loss.times)
            prob.n_obs = len(loss.times)
            prob.obs_times = C.cast(otimes, C.POINTER(C.c_double))
    elif obs:
        steps_c = (C.c_int32 * len(obs_steps))(*obs_steps)
        prob.n_obs = len(obs_steps)
        prob.obs_steps = C.cast(steps_c, C.POINTER(C.c_int32))
    nbytes = workspace_size(prob)
    dev = u0d.device
    ws = _workspace(nbytes, dev)
    u_final = torch.empty_like(u0d)
    du0 = torch.empty_like(u0d)
    dtheta = torch.empty(field.n_params, dtype=dt, device=dev)
    loss_t = torch.empty(1, dtype=torch.float64, device=dev)   # written by the reduction
    preds = obs_vals = lo = hi = None
    if obs:
        vals = []
        for v in loss.values:
            v = to_device(v, dt)
            if v.dim() == 1:
                v = v.unsqueeze(0).expand(B, -1)
            if tuple(v.shape) != (B, N):
                raise ValueError("observations must be [B, N] or [N]")
            vals.append(v)
        obs_vals = torch.stack(vals).contiguous()
        preds = torch.empty_like(obs_vals)
        if loss.scaling is not None:
            if loss.scaling.lo.shape != (N,):
                raise ValueError("scaling bounds must have the state dimension")
            lo = to_device(loss.scaling.lo, dt)
            hi = to_device(loss.scaling.hi, dt)
    aux = field.aux()
    bufs = _lib.Buffers()
    bufs.theta = field.theta_tensor().data_ptr()
    bufs.aux = aux.data_ptr() if aux is not None else None
    bufs.u0 = u0d.data_ptr()
    bufs.targets = None
    if obs:
        bufs.obs_values = obs_vals.data_ptr()
        bufs.predictions = preds.data_ptr()
        bufs.scale_lo = lo.data_ptr() if lo is not None else None
        bufs.scale_hi = hi.data_ptr() if hi is not None else None
    bufs.u_final = u_final.data_ptr()
    bufs.du0 = du0.data_ptr()
    bufs.dtheta = dtheta.data_ptr()
    bufs.loss = loss_t.data_ptr()
    bufs.workspace = ws.data_ptr()
    bufs.workspace_bytes = ws.numel()
    stats = torch.empty((B, _lib.OB_NSTATS), dtype=torch.int32, device=dev)   # copied from the zeroed device stats
    bufs.sample_stats = stats.data_ptr()
    dhead = None
    if loss.kind == "ce_head":
        head = to_device(loss.values[0], dt).reshape(-1)
        labels = to_device(loss.values[1], torch.int32).reshape(-1)
        if head.numel() != 10 * 64 + 10 or labels.numel() != B:
            raise ValueError("ce_head needs 650 head parameters and one label per sample")
        dhead = torch.empty_like(head)
        bufs.head, bufs.labels, bufs.dhead = head.data_ptr(), labels.data_ptr(), dhead.data_ptr()
        bufs.n_classes = 10
    grid_t = nacc_t = None
    if adaptive:
        grid_t = torch.empty((B, ctrl.max_accepted + 1), dtype=torch.float64, device=dev)
        nacc_t = torch.empty(B, dtype=torch.int32, device=dev)
        bufs.grid, bufs.n_accepted = grid_t.data_ptr(), nacc_t.data_ptr()
    cnt = _lib.Counters()
    rc = _lib.load().ob_grad(C.byref(prob), C.byref(bufs), C.byref(cnt), stream_ptr())
    raise_status(rc, _lib.last_error())
    c = cnt.as_dict()
    counters.nfe_forward += c["nfe_forward"]
    counters.nfe_backward += c["nfe_backward"]
    counters.steps_accepted += c["steps_accepted"]
    counters.steps_recomputed += c["steps_recomputed"]
    sc = StoreCounters(c["stored_states"], c["stored_stage_vectors"], c["max_live_slots"],
                       c["recomputed_steps"])
    if scheme.kind == "theta":
        st = stats.cpu().numpy().astype(np.int64)
        samp = {"nfe_forward": st[:, 0], "nfe_backward": st[:, 1], "newton_iters": st[:, 2],
                "gmres_iters_forward": st[:, 3], "gmres_iters_adjoint": st[:, 4]}
    elif adaptive:
        st = stats.cpu().numpy().astype(np.int64)
        samp = {"nfe_forward": st[:, 0], "nfe_backward": st[:, 1], "steps_accepted": st[:, 5],
                "steps_rejected": st[:, 6], "steps_recomputed": st[:, 7]}
        counters.steps_rejected += c["steps_rejected"]
    else:
        samp = {"nfe_forward": np.full(B, c["nfe_forward"]),
                "nfe_backward": np.full(B, c["nfe_backward"])}
    if host_io:
        # pinned staging (torch's caching host allocator) + async copies: one stream
        # synchronisation (the loss read below) instead of three pageable round trips
        staged = []
        for x in (dtheta, du0, u_final):
            h = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
            h.copy_(x, non_blocking=True)
            staged.append(h)
    loss_v = float(loss_t.item())
    if host_io:
        dtheta_o, du0_o, uf_o = (h.numpy() for h in staged)
    else:
        dtheta_o, du0_o, uf_o = dtheta, du0, u_final
    if dhead is not None and host_io:
        dhead = dhead.cpu().numpy()
    if obs:
        pr = preds.cpu().numpy() if host_io else preds
        predictions = [pr[k] for k in range(pr.shape[0])]
    else:
        predictions = [uf_o]
    grids = None
    if adaptive:
        g = grid_t.cpu().numpy()
        na = nacc_t.cpu().numpy()
        grids = [g[b, :na[b] + 1].copy() for b in range(B)]
    return GradResult(dtheta=dtheta_o, du0=du0_o, loss=loss_v, counters=counters,
                      predictions=predictions, u_final=uf_o, store_counters=sc, device=c,
                      sample_counters=samp, dtheta_head=dhead, grids=grids)


def continuous_adjoint_solve(field: Field, scheme: Scheme, dphi_du, u_final, t0, tF, n_steps,
                             counters=None):
    """Vanilla continuous-adjoint baseline (adjoint.py:314-331): integrate
    du/dtau = -f, dlam/dtau = J^T lam, dmu/dtau = P^T lam backward from
    (u_final, dphi_du) with the same explicit scheme on n_steps fixed steps.
    Batched: returns (lam0 [B, N], mu0 = sum over samples, counters)."""
    if scheme.kind != "rk":
        raise ValueError("the continuous-adjoint baseline supports explicit schemes")
    counters = counters if counters is not None else NfeCounters()
    dt = field.torch_dtype
    host_io = not (isinstance(u_final, torch.Tensor) and u_final.is_cuda)
    uf = to_device(u_final, dt)
    lamT = to_device(dphi_du, dt)
    if uf.dim() == 1:
        uf, lamT = uf.unsqueeze(0), lamT.unsqueeze(0)
    B, N = uf.shape
    if N != field.n or tuple(lamT.shape) != (B, N):
        raise ValueError(f"expected [B, {field.n}] terminal state and seed")
    ts = np.linspace(0.0, tF - t0, int(n_steps) + 1)
    prob, _times = build_problem(field, scheme, LossSpec("half_sqnorm", (tF,)), B, ts,
                                 CheckpointPolicy("store_solutions"), SolverConfig(), B)
    prob.tF = float(tF)
    ws = _workspace(workspace_size(prob), uf.device)
    lam0 = torch.empty_like(uf)
    mu0 = torch.empty(field.n_params, dtype=dt, device=uf.device)
    aux = field.aux()
    cnt = _lib.Counters()
    rc = _lib.load().ob_continuous_adjoint(
        C.byref(prob), field.theta_tensor().data_ptr(), aux.data_ptr() if aux is not None else None,
        uf.data_ptr(), lamT.data_ptr(), lam0.data_ptr(), mu0.data_ptr(), ws.data_ptr(), ws.numel(),
        C.byref(cnt), stream_ptr())
    raise_status(rc, _lib.last_error())
    c = cnt.as_dict()
    counters.nfe_forward += c["nfe_forward"]
    counters.nfe_backward += c["nfe_backward"]
    counters.steps_accepted += c["steps_accepted"]
    if host_io:
        return lam0.cpu().numpy(), mu0.cpu().numpy(), counters
    return lam0, mu0, counters
