"""Quick GPU check of the tcgen05 conv tile (C3) against the SIMT tile and the oracle."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from oracle import core as oc
from oracle import fields_ext as ox
from oracle.problems import run_oracle
from paper_2206_01298_b200.configs import make_config
from paper_2206_01298_b200.workloads import field_from_config, initial_state, run_config

ci = make_config("C3").subset(3)
fld = field_from_config(ci)
ofl = ox.ConvField(ci.theta)
rng = np.random.default_rng(9)
U = ci.u0.reshape(3, -1)
V = rng.standard_normal(U.shape).astype(np.float32).astype(np.float64)
f_ref = ofl.eval(U, 0.35, oc.Counters())
j_ref, p_ref = ofl.vjp(U, 0.35, V, oc.Counters())
f = fld.eval(U, 0.35).cpu().numpy()
print("eval err", oc.rel_error(f, f_ref), flush=True)
j, pp = fld.vjp(U, 0.35, V)
pp = pp.cpu().numpy()
print("vjp jtv err", oc.rel_error(j.cpu().numpy(), j_ref), "ptv err", oc.rel_error(pp, p_ref), flush=True)
# per parameter block (W1 incl. time channel, b1, W2, b2)
o = 0
for name, n in (("W1", 64 * 9 * 65), ("b1", 64), ("W2", 64 * 9 * 64), ("b2", 64)):
    print("  ", name, oc.rel_error(pp[o:o + n], p_ref[o:o + n]), flush=True)
    o += n
w1 = pp[:64 * 9 * 65].reshape(64, 9, 65)
r1 = p_ref[:64 * 9 * 65].reshape(64, 9, 65)
print("   W1 time channel", oc.rel_error(w1[:, :, 64], r1[:, :, 64]), flush=True)

ci = make_config("C3").subset(6)
fl = field_from_config(ci)
ref = run_oracle(ci, "store_all")
for tcf in (True, False):
    r = run_config(ci, "store_all", field=fl, tensor_cores=tcf)
    e = {k: oc.rel_error(np.asarray(getattr(r, k)), ref[k]) for k in ("u_final", "du0", "dtheta")}
    print("subset6", "tc" if tcf else "simt", r.device["tensor_cores"], e, "loss", abs(r.loss - ref["loss"]) / abs(ref["loss"]), flush=True)
r2 = run_config(ci, "revolve:3", field=fl)
r1 = run_config(ci, "store_all", field=fl)
print("policies bit-identical:", np.array_equal(np.asarray(r1.dtheta), np.asarray(r2.dtheta)), r1.loss == r2.loss, flush=True)

ci = make_config("C3")
fl = field_from_config(ci)
u0 = torch.as_tensor(initial_state(ci), dtype=torch.float32, device="cuda")
for tcf in (True, False):
    for _ in range(2):
        r = run_config(ci, "store_all", field=fl, u0=u0, tensor_cores=tcf)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    r = run_config(ci, "store_all", field=fl, u0=u0, tensor_cores=tcf)
    torch.cuda.synchronize()
    print("C3 full tc" if tcf else "C3 full simt", (time.perf_counter() - t0) * 1e3, "ms", r.device["ms_forward"], r.device["ms_reverse"], flush=True)

# per-image du0 error against the oracle (ReLU kinks: images whose adjoint jumps)
n = int(os.environ.get("C3_IMAGES", "64"))
ci = make_config("C3").subset(n)
fl = field_from_config(ci)
t0 = time.perf_counter()
ref = run_oracle(ci, "store_all")
print("oracle", n, "images", time.perf_counter() - t0, "s", flush=True)
scale = np.max(np.abs(ref["du0"]))
for tcf in (True, False):
    r = run_config(ci, "store_all", field=fl, tensor_cores=tcf)
    per = np.max(np.abs(np.asarray(r.du0, dtype=np.float64) - ref["du0"]), axis=1) / scale
    over = np.nonzero(per > 1e-4)[0]
    print("tc" if tcf else "simt", "median", np.median(per), "over the bar:", len(over), [(int(b), float(per[b])) for b in over],
          "dtheta", oc.rel_error(np.asarray(r.dtheta), ref["dtheta"]), "u_final", oc.rel_error(np.asarray(r.u_final), ref["u_final"]), flush=True)
