"""Device time of one grad() per tile geometry (tile_rows sweep) for a config."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2206_01298_b200.configs import make_config
from paper_2206_01298_b200.workloads import field_from_config, initial_state, run_config

name = sys.argv[1]
rows = [int(x) for x in sys.argv[2].split(",")]
ci = make_config(name)
fld = field_from_config(ci)
u0 = torch.as_tensor(initial_state(ci), dtype=fld.torch_dtype, device="cuda")
for r in rows:
    res = None
    for _ in range(2):
        res = run_config(ci, field=fld, u0=u0, tile_rows=r)
    ms = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = run_config(ci, field=fld, u0=u0, tile_rows=r)
        torch.cuda.synchronize()
        ms.append(1e3 * (time.perf_counter() - t0))
    d = res.device
    print(f"{name} tile_rows {d['tile_rows']:3d} tiles {d['tiles']:4d}  {min(ms):8.2f} ms/step  "
          f"fwd {d['ms_forward']:.2f}  rev {d['ms_reverse']:.2f}  -> {ci.batch / min(ms) * 1e3:.4g} samples/s")
