"""The ODE block as a differentiable torch module (how PNODE is used inside a
network: an ODE block between other layers, trained by the surrounding
autograd graph).

``ODEBlock(field, scheme, t0, tF, ctrl, policy)`` maps u0 [B, N] -> u(tF) [B, N].
Its forward is ``forward_pass`` (checkpoints stay in the call's device workspace);
its backward is ``backward_sweep`` seeded with the incoming gradient dL/du(tF) as
the terminal adjoint state (adjoint_terminal, adjoint.py:47-52) -- the discrete
adjoint of the integrator, not autograd through the solver steps.  The field's
flat parameter vector is exposed as ``ODEBlock.theta`` (an ``nn.Parameter``
sharing the field's device storage), so optimizers update the field in place.
"""

from __future__ import annotations

import torch

from .engine import adjoint_terminal, backward_sweep, forward_pass
from .policies import CheckpointPolicy


class _OdeBlockFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, u0, theta, block):
        fwd = forward_pass(block.field, block.scheme, u0.detach(), block.t0, block.tF, block.ctrl,
                           block.policy, block.solver_cfg, tensor_cores=block.tensor_cores)
        ctx.fwd = fwd
        ctx.block = block
        return fwd.u_final

    @staticmethod
    def backward(ctx, grad_uF):
        block, fwd = ctx.block, ctx.fwd
        adj = backward_sweep(block.field, block.scheme, fwd,
                             adjoint_terminal(grad_uF.contiguous()), solver_cfg=block.solver_cfg)
        ctx.fwd = None   # the checkpoints are consumed
        return adj.lam, adj.mu, None


class ODEBlock(torch.nn.Module):
    def __init__(self, field, scheme, t0, tF, ctrl, policy=CheckpointPolicy("store_all"),
                 solver_cfg=None, tensor_cores=True):
        super().__init__()
        self.field, self.scheme = field, scheme
        self.t0, self.tF, self.ctrl = float(t0), float(tF), ctrl
        self.policy, self.solver_cfg, self.tensor_cores = policy, solver_cfg, tensor_cores
        self.theta = torch.nn.Parameter(field.theta_tensor(), requires_grad=True)

    def forward(self, u0: torch.Tensor) -> torch.Tensor:
        if u0.dtype != self.field.torch_dtype:
            raise ValueError(f"u0 must be {self.field.torch_dtype}")
        return _OdeBlockFunction.apply(u0, self.theta, self)
