"""Quick GPU check of the tcgen05 CNF tile against the SIMT tile and the oracle."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from oracle import core as oc
from oracle import fields_ext as ox
from paper_2206_01298_b200.configs import make_config
from paper_2206_01298_b200.workloads import field_from_config, initial_state, run_config

ci = make_config("C4").subset(12)
fld = field_from_config(ci)
ofl = ox.CnfField(oc.Mlp(ci.widths, ci.activation, ci.theta, True), ci.extras["eps"])
rng = np.random.default_rng(3)
Y = initial_state(ci).astype(np.float32).astype(np.float64)
Y[:, -1] = rng.standard_normal(ci.batch)
V = rng.standard_normal(Y.shape).astype(np.float32).astype(np.float64)
f_ref = ofl.eval(Y, 0.4, oc.Counters())
j_ref, p_ref = ofl.vjp(Y, 0.4, V, oc.Counters())
f = fld.eval(Y, 0.4).cpu().numpy()
print("eval err", oc.rel_error(f, f_ref), flush=True)
j, pp = fld.vjp(Y, 0.4, V)
print("vjp jtv err", oc.rel_error(j.cpu().numpy(), j_ref), "ptv err", oc.rel_error(pp.cpu().numpy(), p_ref), flush=True)
for n, rows in ((24, None), (64, 7)):
    ci = make_config("C4").subset(n)
    fl = field_from_config(ci)
    tc = run_config(ci, "store_all", field=fl, tile_rows=rows)
    si = run_config(ci, "store_all", field=fl, tile_rows=rows, tensor_cores=False)
    from oracle.problems import run_oracle
    ref = run_oracle(ci, "store_all")
    e = {k: oc.rel_error(np.asarray(getattr(tc, k)), ref[k]) for k in ("u_final", "du0", "dtheta")}
    e2 = {k: oc.rel_error(np.asarray(getattr(si, k)), ref[k]) for k in ("u_final", "du0", "dtheta")}
    print(n, "tc", tc.device["tensor_cores"], tc.device["tile_rows"], e, "loss", abs(tc.loss - ref["loss"]) / abs(ref["loss"]), flush=True)
    print(n, "simt", e2, flush=True)
ci = make_config("C4")
fl = field_from_config(ci)
u0 = torch.as_tensor(initial_state(ci), dtype=torch.float32, device="cuda")
for tcf in ((True,) if os.environ.get("OB_CNF_CLUSTER") else (True, False)):
    for _ in range(2):
        r = run_config(ci, "store_all", field=fl, u0=u0, tensor_cores=tcf)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    r = run_config(ci, "store_all", field=fl, u0=u0, tensor_cores=tcf)
    torch.cuda.synchronize()
    print("C4 full tc" if tcf else "C4 full simt", (time.perf_counter() - t0) * 1e3, "ms", r.device["ms_forward"], r.device["ms_reverse"], flush=True)
