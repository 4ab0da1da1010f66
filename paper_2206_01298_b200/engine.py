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
from .controls import (AdaptiveController, GradientExplosionError, NfeCounters, SolverConfig,
                       StoreCounters, boundary_times, raise_status)
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
    """Scratch of one grad() call, cached per (device, stream): calls on one stream
    are ordered, so they may share it; a call on another stream gets its own."""
    stream = torch.cuda.current_stream(device)
    key = (device.index, stream.cuda_stream)
    buf = _WS_CACHE.get(key)
    if buf is None or buf.numel() < nbytes:
        if buf is not None:
            # kernels of an earlier call may still read the old buffer on this stream
            buf.record_stream(stream)
        buf = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=device)
        _WS_CACHE[key] = buf
    return buf


def build_problem(field: Field, scheme: Scheme, loss: LossSpec, batch: int, ts: np.ndarray,
                  policy: CheckpointPolicy, solver_cfg: SolverConfig, batch_global: int,
                  loss_kind: str = None):
    prob = _lib.Problem()
    prob.field = field.desc()
    prob.scheme = to_desc(scheme)
    prob.solver = solver_cfg.to_desc()
    prob.batch = batch
    prob.batch_global = batch_global
    prob.n_steps = len(ts) - 1
    prob.policy = _lib.OB_POLICY[policy.kind]
    prob.nc = policy.nc
    prob.loss = _lib.OB_LOSS[loss_kind or loss.kind]
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


class _Call:
    """Device state of one gradient problem: the ob_problem / ob_buffers structs, the
    tensors they point to (kept alive here) and the host arrays the problem references."""

    def __init__(self, field: Field, scheme: Scheme, loss: LossSpec, u0, t0, tF, ctrl, policy,
                 solver_cfg, *, batch_global=None, profile=False, tensor_cores=True, tile_rows=None,
                 seeded=False, obs_times=(), own_workspace=False):
        self.field, self.scheme, self.policy, self.ctrl = field, scheme, policy, ctrl
        self.solver_cfg = solver_cfg
        self.t0, self.tF = float(t0), float(tF)
        self.seeded = seeded
        times_obs = tuple(float(t) for t in (obs_times if seeded else loss.times))
        if times_obs and times_obs[-1] > tF + 1e-9 * max(1.0, abs(tF)):
            raise ValueError("observations extend past the final time")
        obs = (not seeded and loss.kind in OBSERVATION_KINDS) or (seeded and len(times_obs) > 0)
        if not seeded and not obs and abs(loss.times[-1] - tF) > 1e-9 * max(1.0, abs(tF)):
            raise ValueError(f"{loss.kind} is a terminal loss at tF")
        self.obs, self.times_obs = obs, times_obs
        self.adaptive = adaptive = isinstance(ctrl, AdaptiveController)
        if adaptive:
            if tF <= t0:
                raise ValueError("tF must exceed t0")
            ts = np.array([t0, tF], dtype=np.float64)
            obs_steps = None
        else:
            ts = boundary_times(ctrl, t0, tF)
            obs_steps = match_boundaries(times_obs, ts) if obs else None
        self.ts, self.obs_steps = ts, obs_steps
        self.host_io = not (isinstance(u0, torch.Tensor) and u0.is_cuda)
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
        self.B, self.N = B, N
        bg = int(batch_global) if batch_global is not None else B
        prob, self._times = build_problem(field, scheme, loss, B, ts, policy, solver_cfg, bg,
                                          "seed" if seeded else None)
        prob.flags = (1 if profile else 0) | (0 if tensor_cores else 2)
        prob.tile_rows = int(tile_rows or 0)
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
                self._otimes = (C.c_double * len(times_obs))(*times_obs)
                prob.n_obs = len(times_obs)
                prob.obs_times = C.cast(self._otimes, C.POINTER(C.c_double))
        elif obs:
            self._steps_c = (C.c_int32 * len(obs_steps))(*obs_steps)
            prob.n_obs = len(obs_steps)
            prob.obs_steps = C.cast(self._steps_c, C.POINTER(C.c_int32))
        self.prob = prob
        nbytes = workspace_size(prob)
        dev = u0d.device
        # a forward_pass keeps its checkpoints until its backward_sweep: private scratch
        self.ws = (torch.empty(max(nbytes, 1), dtype=torch.uint8, device=dev) if own_workspace
                   else _workspace(nbytes, dev))
        self.u0d = u0d
        self.u_final = torch.empty_like(u0d)
        self.du0 = torch.empty_like(u0d)
        self.dtheta = torch.empty(field.n_params, dtype=dt, device=dev)
        self.loss_t = torch.empty(1, dtype=torch.float64, device=dev)   # written by the reduction
        self.preds = obs_vals = lo = hi = None
        if obs and not seeded:
            vals = []
            for v in loss.values:
                v = to_device(v, dt)
                if v.dim() == 1:
                    v = v.unsqueeze(0).expand(B, -1)
                if tuple(v.shape) != (B, N):
                    raise ValueError("observations must be [B, N] or [N]")
                vals.append(v)
            obs_vals = torch.stack(vals).contiguous()
            if loss.scaling is not None:
                if loss.scaling.lo.shape != (N,):
                    raise ValueError("scaling bounds must have the state dimension")
                lo = to_device(loss.scaling.lo, dt)
                hi = to_device(loss.scaling.hi, dt)
        if obs:
            self.preds = torch.empty((len(times_obs), B, N), dtype=dt, device=dev)
        self._keep = [obs_vals, lo, hi]
        aux = field.aux()
        bufs = _lib.Buffers()
        bufs.theta = field.theta_tensor().data_ptr()
        bufs.aux = aux.data_ptr() if aux is not None else None
        bufs.u0 = u0d.data_ptr()
        bufs.targets = None
        if obs:
            bufs.predictions = self.preds.data_ptr()
            if obs_vals is not None:
                bufs.obs_values = obs_vals.data_ptr()
            bufs.scale_lo = lo.data_ptr() if lo is not None else None
            bufs.scale_hi = hi.data_ptr() if hi is not None else None
        bufs.u_final = self.u_final.data_ptr()
        bufs.du0 = self.du0.data_ptr()
        bufs.dtheta = self.dtheta.data_ptr()
        bufs.loss = self.loss_t.data_ptr()
        bufs.workspace = self.ws.data_ptr()
        bufs.workspace_bytes = self.ws.numel()
        self.stats = torch.empty((B, _lib.OB_NSTATS), dtype=torch.int32, device=dev)
        bufs.sample_stats = self.stats.data_ptr()
        self.dhead = None
        if not seeded and loss.kind == "ce_head":
            head = to_device(loss.values[0], dt).reshape(-1)
            labels = to_device(loss.values[1], torch.int32).reshape(-1)
            if head.numel() != 10 * 64 + 10 or labels.numel() != B:
                raise ValueError("ce_head needs 650 head parameters and one label per sample")
            self.dhead = torch.empty_like(head)
            self._keep += [head, labels]
            bufs.head, bufs.labels, bufs.dhead = head.data_ptr(), labels.data_ptr(), self.dhead.data_ptr()
            bufs.n_classes = 10
        self.grid_t = self.nacc_t = None
        if adaptive:
            self.grid_t = torch.empty((B, ctrl.max_accepted + 1), dtype=torch.float64, device=dev)
            self.nacc_t = torch.empty(B, dtype=torch.int32, device=dev)
            bufs.grid, bufs.n_accepted = self.grid_t.data_ptr(), self.nacc_t.data_ptr()
        self.bufs = bufs
        self.kind = "theta" if scheme.kind == "theta" else ("adaptive" if adaptive else "fixed")

    def launch(self, fn_name: str):
        cnt = _lib.Counters()
        with _nvtx(fn_name):
            rc = getattr(_lib.load(), fn_name)(C.byref(self.prob), C.byref(self.bufs), C.byref(cnt),
                                               stream_ptr())
        raise_status(rc, _lib.last_error())
        return cnt.as_dict()

    def sample_counters(self, c):
        B = self.B
        if self.kind == "theta":
            st = self.stats.cpu().numpy().astype(np.int64)
            return {"nfe_forward": st[:, 0], "nfe_backward": st[:, 1], "newton_iters": st[:, 2],
                    "gmres_iters_forward": st[:, 3], "gmres_iters_adjoint": st[:, 4]}
        if self.kind == "adaptive":
            st = self.stats.cpu().numpy().astype(np.int64)
            return {"nfe_forward": st[:, 0], "nfe_backward": st[:, 1], "steps_accepted": st[:, 5],
                    "steps_rejected": st[:, 6], "steps_recomputed": st[:, 7]}
        return {"nfe_forward": np.full(B, c["nfe_forward"]), "nfe_backward": np.full(B, c["nfe_backward"])}

    def grids(self):
        if not self.adaptive:
            return None
        g = self.grid_t.cpu().numpy()
        na = self.nacc_t.cpu().numpy()
        return [g[b, :na[b] + 1].copy() for b in range(self.B)]


class _nvtx:
    """NVTX range around a native call (visible in nsys / ncu --nvtx timelines)."""

    def __init__(self, name):
        self.name = name

    def __enter__(self):
        torch.cuda.nvtx.range_push(self.name)

    def __exit__(self, *exc):
        torch.cuda.nvtx.range_pop()
        return False


def _add_counters(counters: NfeCounters, c: dict, adaptive: bool):
    counters.nfe_forward += c["nfe_forward"]
    counters.nfe_backward += c["nfe_backward"]
    counters.steps_accepted += c["steps_accepted"]
    counters.steps_recomputed += c["steps_recomputed"]
    if adaptive:
        counters.steps_rejected += c["steps_rejected"]


def grad(field: Field, scheme: Scheme, loss: LossSpec, u0, t0, tF, ctrl,
         policy=CheckpointPolicy("store_all"), solver_cfg=None, counters=None, *,
         batch_global=None, profile=False, tensor_cores=True, tile_rows=None) -> GradResult:
    """Loss, dL/dtheta and dL/du0 by forward solve + discrete adjoint sweep.

    ``tensor_cores=False`` forces the SIMT (FMA) MLP tile where the tcgen05
    tile would apply (fp32 two-layer MLP fields on explicit fixed-step schemes).
    ``tile_rows`` forces the samples per CTA tile (default: the planner's choice).
    """
    solver_cfg = solver_cfg or SolverConfig()
    counters = counters if counters is not None else NfeCounters()
    call = _Call(field, scheme, loss, u0, t0, tF, ctrl, policy, solver_cfg, batch_global=batch_global,
                 profile=profile, tensor_cores=tensor_cores, tile_rows=tile_rows)
    c = call.launch("ob_grad")
    _add_counters(counters, c, call.adaptive)
    sc = StoreCounters(c["stored_states"], c["stored_stage_vectors"], c["max_live_slots"],
                       c["recomputed_steps"])
    samp = call.sample_counters(c)
    dtheta, du0, u_final, dhead = call.dtheta, call.du0, call.u_final, call.dhead
    if call.host_io:
        # pinned staging (torch's caching host allocator) + async copies: one stream
        # synchronisation (the loss read below) instead of three pageable round trips
        staged = []
        for x in (dtheta, du0, u_final):
            h = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
            h.copy_(x, non_blocking=True)
            staged.append(h)
    loss_v = float(call.loss_t.item())
    if call.host_io:
        dtheta, du0, u_final = (h.numpy() for h in staged)
        if dhead is not None:
            dhead = dhead.cpu().numpy()
    if call.obs:
        pr = call.preds.cpu().numpy() if call.host_io else call.preds
        predictions = [pr[k] for k in range(pr.shape[0])]
    else:
        predictions = [u_final]
    return GradResult(dtheta=dtheta, du0=du0, loss=loss_v, counters=counters,
                      predictions=predictions, u_final=u_final, store_counters=sc, device=c,
                      sample_counters=samp, dtheta_head=dhead, grids=call.grids())


# ------------------------------------------------------------------ split sweep
@dataclass
class AdjointState:
    """Adjoint state (adjoint.py:37-44), batched: lam [B, N] = dL/du_n per sample,
    mu [Np] = accumulated dL/dtheta (summed over the batch)."""

    lam: object
    mu: object

    def check_finite(self):
        ok = all(x is None or bool(torch.isfinite(torch.as_tensor(x)).all()) for x in (self.lam, self.mu))
        if not ok:
            raise GradientExplosionError("non-finite adjoint state in reverse sweep")


def adjoint_terminal(dphi_du, dphi_dtheta=None) -> AdjointState:
    """Terminal condition lambda_N = dL/du_N, mu_N = dL/dtheta (adjoint.py:47-52).
    Batched: dphi_du [B, N]; dphi_dtheta [Np] or None (zero)."""
    return AdjointState(dphi_du, dphi_dtheta)


@dataclass
class ForwardSolution:
    """forward_pass result (adjoint.py:128-133): the checkpoints stay in the device
    workspace of this object until backward_sweep consumes them."""

    store_counters: StoreCounters
    boundary_times: object        # fixed grid [n_steps + 1]; adaptive: per-sample grids
    obs_states: list              # [B, N] state at each requested observation time
    u_final: object
    counters: dict = None
    _call: object = None


def forward_pass(field: Field, scheme: Scheme, u0, t0, tF, ctrl,
                 policy=CheckpointPolicy("store_all"), solver_cfg=None, counters=None,
                 obs_times=(), *, tensor_cores=True, tile_rows=None) -> ForwardSolution:
    """Forward solve filling the checkpoint store and capturing the states at
    ``obs_times`` (adjoint.py:151-210); the reverse half is ``backward_sweep``."""
    solver_cfg = solver_cfg or SolverConfig()
    counters = counters if counters is not None else NfeCounters()
    call = _Call(field, scheme, None, u0, t0, tF, ctrl, policy, solver_cfg, tensor_cores=tensor_cores,
                 tile_rows=tile_rows, seeded=True, obs_times=obs_times, own_workspace=True)
    c = call.launch("ob_forward_pass")
    counters.nfe_forward += c["nfe_forward"]
    counters.steps_accepted += c["steps_accepted"]
    if call.adaptive:
        counters.steps_rejected += c["steps_rejected"]
    sc = StoreCounters(c["stored_states"], c["stored_stage_vectors"], c["max_live_slots"],
                       c["recomputed_steps"])
    obs_states = [call.preds[k] for k in range(call.preds.shape[0])] if call.obs else []
    bt = call.grids() if call.adaptive else list(call.ts)
    u_final = call.u_final
    if call.host_io:
        u_final = u_final.cpu().numpy()
        obs_states = [o.cpu().numpy() for o in obs_states]
    return ForwardSolution(sc, bt, obs_states, u_final, c, call)


def backward_sweep(field: Field, scheme: Scheme, fwd: ForwardSolution, terminal: AdjointState,
                   injections=None, solver_cfg=None, counters=None) -> AdjointState:
    """Reverse every step from the forward's checkpoints (adjoint.py:235-253):
    lambda starts at ``terminal.lam`` [B, N], mu at ``terminal.mu``; ``injections``
    maps an observation's boundary index (fixed grids; adaptive grids: the index k of
    ``obs_times``) to a [B, N] seed added to lambda there (inject_observation,
    :135-140).  Only the boundaries named in forward_pass's ``obs_times`` can take
    injections.  Returns (lambda_0 [B, N], mu_0 [Np])."""
    call = fwd._call
    if call is None or call.field is not field:
        raise ValueError("forward solution was produced for another field")
    if solver_cfg is not None and solver_cfg != call.solver_cfg:
        raise ValueError("solver configuration differs from the forward pass")
    counters = counters if counters is not None else NfeCounters()
    dt = field.torch_dtype
    B, N = call.B, call.N
    lam = to_device(terminal.lam, dt)
    if lam.dim() == 1:
        lam = lam.unsqueeze(0)
    if tuple(lam.shape) != (B, N):
        raise ValueError(f"terminal lambda must be [{B}, {N}]")
    mu0 = None
    if terminal.mu is not None:
        mu0 = to_device(terminal.mu, dt).reshape(-1)
        if mu0.numel() != field.n_params:
            raise ValueError(f"terminal mu must have {field.n_params} entries")
    if not (bool(torch.isfinite(lam).all()) and (mu0 is None or bool(torch.isfinite(mu0).all()))):
        raise GradientExplosionError("non-finite adjoint state in reverse sweep")   # check_finite
    inj = None
    if injections:
        if not call.obs:
            raise ValueError("injections need forward_pass(..., obs_times=...) at those boundaries")
        slots = list(range(len(call.times_obs))) if call.adaptive else list(call.obs_steps)
        inj = torch.zeros((len(slots), B, N), dtype=dt, device=lam.device)
        for j, seed in injections.items():
            if j not in slots:
                raise ValueError(f"boundary {j} is not an observation boundary of the forward pass")
            v = to_device(seed, dt)
            inj[slots.index(j)] += v.unsqueeze(0).expand(B, -1) if v.dim() == 1 else v
    elif call.obs:
        inj = torch.zeros((len(call.times_obs), B, N), dtype=dt, device=lam.device)
    bufs = call.bufs
    bufs.seed = lam.data_ptr()
    bufs.dtheta_seed = mu0.data_ptr() if mu0 is not None else None
    bufs.obs_values = inj.data_ptr() if inj is not None else None
    call._keep += [lam, mu0, inj]
    c = call.launch("ob_backward_sweep")
    counters.nfe_backward += c["nfe_backward"]
    counters.steps_recomputed += c["steps_recomputed"]
    fwd.counters = {**(fwd.counters or {}), "backward": c}
    if call.host_io:
        return AdjointState(call.du0.cpu().numpy(), call.dtheta.cpu().numpy())
    return AdjointState(call.du0, call.dtheta)


def loss_value(field: Field, scheme: Scheme, loss: LossSpec, u0, t0, tF, ctrl, solver_cfg=None,
               counters=None, *, batch_global=None) -> float:
    """Forward-only loss (adjoint.py:282-291; the FD oracle's workhorse): one forward
    sweep with solution-only checkpoints, the loss reduced on the device."""
    solver_cfg = solver_cfg or SolverConfig()
    counters = counters if counters is not None else NfeCounters()
    call = _Call(field, scheme, loss, u0, t0, tF, ctrl, CheckpointPolicy("store_solutions"),
                 solver_cfg, batch_global=batch_global)
    c = call.launch("ob_forward_pass")
    counters.nfe_forward += c["nfe_forward"]
    return float(call.loss_t.item())


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
    prob.flags = 2   # OB_FLAG_NO_TENSOR_CORES: the augmented sweep runs on the SIMT tile
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
