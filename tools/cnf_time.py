import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2206_01298_b200.configs import make_config
from paper_2206_01298_b200.workloads import field_from_config, initial_state, run_config
ci = make_config("C4"); fl = field_from_config(ci)
u0 = torch.as_tensor(initial_state(ci), dtype=torch.float32, device="cuda")
for _ in range(2): r = run_config(ci, "store_all", field=fl, u0=u0)
torch.cuda.synchronize(); t0 = time.perf_counter(); r = run_config(ci, "store_all", field=fl, u0=u0); torch.cuda.synchronize()
print(os.environ.get("OB_LIB_VARIANT", "base"), "%.2f ms" % ((time.perf_counter() - t0) * 1e3), "fwd %.2f rev %.2f pack %.3f reduce %.3f" % (r.device["ms_forward"], r.device["ms_reverse"], r.device["ms_pack"], r.device["ms_reduce"]))
