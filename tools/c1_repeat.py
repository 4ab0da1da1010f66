"""Repeat the C1 gradient (clusters of two CTAs, one exchange per VJP) and check that every
run returns identical bits: a race on the exchange buffers would show up as differing bits."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2206_01298_b200.configs import make_config
from paper_2206_01298_b200.workloads import field_from_config, initial_state, run_config

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
for batch in (512, 800, 77):
    ci = make_config("C1", batch=batch)
    fld = field_from_config(ci)
    u0 = torch.as_tensor(initial_state(ci), dtype=torch.float64, device="cuda")
    first = run_config(ci, "store_all", field=fld, u0=u0)
    bad = 0
    for _ in range(n):
        r = run_config(ci, "store_all", field=fld, u0=u0)
        if r.loss != first.loss or not torch.equal(r.dtheta, first.dtheta) or not torch.equal(r.du0, first.du0):
            bad += 1
    print(f"C1 B={batch}: {n} repeats, {bad} differing, tiles {first.device['tiles']} x {first.device['tile_rows']} rows", flush=True)
