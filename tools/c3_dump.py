"""Dump the full-batch C3 GPU result (u_final, du0, dtheta) for offline comparison."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_01298_b200.configs import make_config
from paper_2206_01298_b200.workloads import run_config
out = sys.argv[1]
os.makedirs(out, exist_ok=True)
res = run_config(make_config("C3"), "store_all")
for k in ("u_final", "du0", "dtheta"):
    np.save(os.path.join(out, k + ".npy"), np.asarray(res.__dict__[k]).astype(np.float32))
print("loss", res.loss)
