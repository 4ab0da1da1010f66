"""Python-side cost of grad() around the native call: cProfile over many C1 calls (short
device time), functions by own time."""
import cProfile, pstats, sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2206_01298_b200.configs import make_config
from paper_2206_01298_b200.controls import FixedController
from paper_2206_01298_b200.policies import CheckpointPolicy
from paper_2206_01298_b200.engine import grad
from paper_2206_01298_b200.schemes import tableau_catalog
from paper_2206_01298_b200.workloads import field_from_config, initial_state, loss_for, solver_from_config

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
ci = make_config(name)
field = field_from_config(ci)
scheme = tableau_catalog(ci.scheme)
loss = loss_for(ci, slice(0, ci.batch))
ctrl = FixedController(ci.n_steps)
scfg = solver_from_config(ci)
policy = CheckpointPolicy.parse(ci.policy)
u0 = torch.as_tensor(initial_state(ci), dtype=field.torch_dtype, device="cuda")
step = lambda: grad(field, scheme, loss, u0, ci.t0, ci.tF, ctrl, policy, scfg)
for _ in range(5):
    step()
n = 300
torch.cuda.synchronize()
t0 = time.perf_counter()
dev = 0.0
for _ in range(n):
    r = step()
    dev += sum(r.device[k] for k in ("ms_pack", "ms_forward", "ms_reverse", "ms_reduce"))
wall = (time.perf_counter() - t0) / n * 1e3
print(f"{name}: wall {wall:.3f} ms per grad, device phases {dev / n:.3f} ms, outside {wall - dev / n:.3f} ms")
pr = cProfile.Profile()
pr.enable()
for _ in range(n):
    step()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(28)
