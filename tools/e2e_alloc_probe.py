"""Does a host-buffer grad() call hit cudaMalloc / cudaHostAlloc every time?"""
import os, sys, time, gc
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2206_01298_b200.configs import make_config
from paper_2206_01298_b200.controls import FixedController
from paper_2206_01298_b200.policies import CheckpointPolicy
from paper_2206_01298_b200.engine import grad
from paper_2206_01298_b200.schemes import tableau_catalog
from paper_2206_01298_b200.workloads import field_from_config, initial_state, loss_for, solver_from_config

ci = make_config("C3")
field = field_from_config(ci)
scheme = tableau_catalog(ci.scheme)
loss = loss_for(ci, slice(0, ci.batch))
ctrl = FixedController(ci.n_steps)
scfg = solver_from_config(ci)
policy = CheckpointPolicy.parse(ci.policy)
tdt = field.torch_dtype
y0 = initial_state(ci)
u0_host = torch.as_tensor(y0, dtype=tdt).pin_memory()
keep = None
for hold in (False, True):
    for i in range(8):
        torch.cuda.synchronize()
        s0 = torch.cuda.memory_stats()
        h0 = torch.cuda.host_memory_stats() if hasattr(torch.cuda, "host_memory_stats") else {}
        t0 = time.perf_counter()
        r = grad(field, scheme, loss, u0_host, ci.t0, ci.tF, ctrl, policy, scfg)
        dt = (time.perf_counter() - t0) * 1e3
        s1 = torch.cuda.memory_stats()
        h1 = torch.cuda.host_memory_stats() if hasattr(torch.cuda, "host_memory_stats") else {}
        print("hold" if hold else "drop", i, f"{dt:.2f} ms", "cudaMalloc", s1["num_device_alloc"] - s0["num_device_alloc"],
              "cudaFree", s1["num_device_free"] - s0["num_device_free"],
              "host allocs", {k: h1[k] - h0[k] for k in h1 if "num_host_alloc" in k or "host_alloc_time.count" in k},
              "gc", gc.get_count(), flush=True)
        if hold:
            keep = r
        else:
            del r
