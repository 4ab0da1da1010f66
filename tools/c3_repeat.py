"""Stress aid: N full C3 gradients in a row (python tools/c3_repeat.py 256 [p]); with a library built
with -DOB_DEBUG_WATCHDOG a starved mbarrier wait reports itself instead of hanging."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2206_01298_b200.configs import make_config
from paper_2206_01298_b200.workloads import field_from_config, run_config
n = int(sys.argv[1]); prof = len(sys.argv) > 2
ci = make_config("C3").subset(n)
fld = field_from_config(ci)
for i in range(3):
    r = run_config(ci, "store_all", field=fld, profile=prof); print("grad ok", n, prof, i, r.loss, flush=True)
