"""Where the end-to-end (host buffers) time of one config goes: H2D, the call, D2H."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2206_01298_b200.configs import make_config
from paper_2206_01298_b200.controls import FixedController
from paper_2206_01298_b200.policies import CheckpointPolicy
from paper_2206_01298_b200.engine import grad
from paper_2206_01298_b200.schemes import tableau_catalog
from paper_2206_01298_b200.workloads import field_from_config, initial_state, loss_for, solver_from_config

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
ci = make_config(name)
field = field_from_config(ci)
scheme = tableau_catalog(ci.scheme)
loss = loss_for(ci, slice(0, ci.batch))
ctrl = FixedController(ci.n_steps)
scfg = solver_from_config(ci)
policy = CheckpointPolicy.parse(ci.policy)
tdt = field.torch_dtype
y0 = initial_state(ci)
u0_dev = torch.as_tensor(y0, dtype=tdt, device="cuda").contiguous()
u0_host = torch.as_tensor(y0, dtype=tdt).pin_memory()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timed(fn, n=8):
    out = []
    for _ in range(n):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        out.append((time.perf_counter() - t0) * 1e3)
    return float(np.median(out))


for _ in range(4):
    grad(field, scheme, loss, u0_host, ci.t0, ci.tF, ctrl, policy, scfg)
print(name, "host call  ", timed(lambda: grad(field, scheme, loss, u0_host, ci.t0, ci.tF, ctrl, policy, scfg)), "ms")
print(name, "device call", timed(lambda: grad(field, scheme, loss, u0_dev, ci.t0, ci.tF, ctrl, policy, scfg)), "ms")
print(name, "h2d u0     ", timed(lambda: u0_host.to("cuda", non_blocking=True)), "ms", u0_host.numel() * u0_host.element_size() / 1e6, "MB")
h = torch.empty(u0_dev.shape, dtype=tdt, pin_memory=True)
print(name, "d2h one    ", timed(lambda: h.copy_(u0_dev, non_blocking=True)), "ms")
print(name, "pinned alloc", timed(lambda: torch.empty(u0_dev.shape, dtype=tdt, pin_memory=True)), "ms")
r = grad(field, scheme, loss, u0_dev, ci.t0, ci.tF, ctrl, policy, scfg)
print(name, "kernels", {k: r.device[k] for k in ("ms_pack", "ms_forward", "ms_reverse", "ms_reduce")})
import cProfile, pstats
pr = cProfile.Profile()
torch.cuda.synchronize()
pr.enable()
for _ in range(5):
    grad(field, scheme, loss, u0_host, ci.t0, ci.tF, ctrl, policy, scfg)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
