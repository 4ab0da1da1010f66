"""Python-side time of engine.grad() before and after the ob_grad C call (C2, device inputs)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2206_01298_b200.configs import make_config
from paper_2206_01298_b200.workloads import field_from_config, run_config, initial_state
import paper_2206_01298_b200.engine as E
ci = make_config("C2"); fld = field_from_config(ci)
u0 = torch.as_tensor(initial_state(ci), dtype=torch.float32, device="cuda")
for _ in range(3): run_config(ci, None, field=fld, u0=u0)
lib = E._lib.load(); orig = lib.ob_grad; marks = {}
class W:
    def __call__(self, *a):
        marks['c0'] = time.perf_counter(); r = orig(*a); marks['c1'] = time.perf_counter(); return r
E._lib._lib.ob_grad = W()
pre, post = [], []
for _ in range(20):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    r = run_config(ci, None, field=fld, u0=u0)
    t1 = time.perf_counter()
    pre.append(marks['c0'] - t0); post.append(t1 - marks['c1'])
print(f"python before ob_grad {np.median(pre)*1e6:.0f} us, after {np.median(post)*1e6:.0f} us")
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for _ in range(20): run_config(ci, None, field=fld, u0=u0)
pr.disable(); pstats.Stats(pr).sort_stats("tottime").print_stats(12)
