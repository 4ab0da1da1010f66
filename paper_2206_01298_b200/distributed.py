"""Data-parallel batch sharding across GPUs (one process per GPU).

Samples are independent given theta (nn.py:26-35), so a batch shards into
contiguous slices with no data-path exchange; the one real exchange is the
parameter cotangent dL/dtheta = sum_b mu_b (plus the loss), once per grad,
after the reverse sweep (adjoint.py:245-252 makes mu final only at the end).

The reduction is deterministic: every rank all-gathers the per-rank partials
and sums them in rank order, so the result is bit-identical run to run (and
independent of NCCL's ring/tree choice).  dtheta is 0.13-3.3 MB, so the
gather costs tens of microseconds over NVLink 5.  The partials stay on the
device for NCCL (host-memory inputs are copied in before the sweep and the
results copied out after the reduction); a gloo group reduces host tensors.

Per-sample field data (the CNF Hutchinson probes) must be the shard's rows:
build the field of each rank from its slice (``workloads.field_from_config``
with ``rows``).
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def shard_bounds(batch_global: int, world: int, rank: int):
    """Contiguous [lo, hi) slice of rank ``rank`` (first ranks take the remainder)."""
    base, rem = divmod(batch_global, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def _comm_device(group=None) -> torch.device:
    if dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def ordered_sum(partial: torch.Tensor, group=None) -> torch.Tensor:
    """Deterministic all-reduce(sum): all_gather then sum in rank order (fp64)."""
    world = dist.get_world_size(group)
    if world == 1:
        return partial.to(torch.float64).clone()
    parts = [torch.empty_like(partial) for _ in range(world)]
    dist.all_gather(parts, partial.contiguous(), group=group)
    acc = parts[0].to(torch.float64).clone()
    for p in parts[1:]:
        acc += p.to(torch.float64)
    return acc


def reduce_grad(dtheta: torch.Tensor, loss: float, group=None):
    """Global (dtheta, loss) from this rank's partials (each already scaled by
    1/batch_global inside the engine).  ``dtheta`` may live on any device; the
    packed partial moves to the group's communication device (CUDA for NCCL)
    and the result comes back on ``dtheta``'s device."""
    dev = _comm_device(group)
    packed = torch.cat([dtheta.reshape(-1).to(device=dev, dtype=torch.float64),
                        torch.tensor([loss], dtype=torch.float64, device=dev)])
    total = ordered_sum(packed, group)
    return total[:-1].to(device=dtheta.device, dtype=dtheta.dtype), float(total[-1].item())


def grad_sharded(field, scheme, loss, u0_local, t0, tF, ctrl, policy, solver_cfg=None, *,
                 batch_global: int, group=None, **kw):
    """Run this rank's shard and reduce dtheta / loss across the group.

    Host inputs (numpy / CPU tensors) are staged to the device here so the
    reduction runs on device partials; the results are copied back to the host
    once, after the reduction (matching grad()'s host-in / host-out contract)."""
    from .engine import grad

    host_io = not (isinstance(u0_local, torch.Tensor) and u0_local.is_cuda)
    u0 = u0_local
    if host_io:
        t = u0_local if isinstance(u0_local, torch.Tensor) else torch.as_tensor(np.asarray(u0_local))
        u0 = t.to(device=torch.device("cuda", torch.cuda.current_device()), dtype=field.torch_dtype,
                  non_blocking=True)
    res = grad(field, scheme, loss, u0, t0, tF, ctrl, policy, solver_cfg, batch_global=batch_global, **kw)
    res.dtheta, res.loss = reduce_grad(res.dtheta, res.loss, group)
    if host_io:
        res.dtheta = res.dtheta.cpu().numpy()
        res.du0 = res.du0.cpu().numpy()
        res.u_final = res.u_final.cpu().numpy()
        res.predictions = [p.cpu().numpy() if isinstance(p, torch.Tensor) else p for p in res.predictions]
    return res
