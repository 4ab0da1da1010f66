"""Host-side overhead of one grad() call (C2): wall time vs device phase time, and a
cProfile of the Python + ctypes path."""
import cProfile, pstats, sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2206_01298_b200.configs import make_config
from paper_2206_01298_b200.workloads import field_from_config, run_config, initial_state

ci = make_config("C2")
fld = field_from_config(ci)
u0 = torch.as_tensor(initial_state(ci), dtype=torch.float32, device="cuda")
for _ in range(3):
    run_config(ci, None, field=fld, u0=u0)
torch.cuda.synchronize()
n = 10
t0 = time.perf_counter()
dev = 0.0
for _ in range(n):
    r = run_config(ci, None, field=fld, u0=u0)
    dev += sum(r.device[k] for k in ("ms_pack", "ms_forward", "ms_reverse", "ms_reduce"))
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / n * 1e3
print(f"wall per grad {wall:.3f} ms, device phases {dev / n:.3f} ms, host overhead {wall - dev / n:.3f} ms")
pr = cProfile.Profile()
pr.enable()
for _ in range(n):
    run_config(ci, None, field=fld, u0=u0)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(15)
pstats.Stats(pr).sort_stats("cumulative").print_stats(45)
