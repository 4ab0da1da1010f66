"""How many C3 images have a discrete adjoint that is discontinuous at the precision of a
3-pass bf16 split (relative error ~2^-16 per product)?  Perturb the conv weights by
independent relative noise of that size, rerun the fp64 oracle, and count the images whose
du0 moves by more than the fp32 parity bar (1e-4 of max|du0|).  A ReLU kink that a
pre-activation crosses under the perturbation flips ReLU' and moves lambda locally."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_01298_b200.configs import make_config
from oracle.problems import run_oracle

ci = make_config("C3")
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
base = run_oracle(ci.subset(n), "store_all")
scale = np.max(np.abs(base["du0"]))
rng = np.random.default_rng(0)
for rel in (2.0 ** -24, 2.0 ** -20, 2.0 ** -16):
    c2 = make_config("C3").subset(n)
    c2.theta = c2.theta * (1 + rng.uniform(-1, 1, c2.theta.shape) * rel)
    r = run_oracle(c2, "store_all")
    per = np.max(np.abs(r["du0"] - base["du0"]), axis=1) / scale
    print(f"relative weight noise {rel:.2e}: images with du0 moved > 1e-4: {np.sum(per > 1e-4)}/{n}, "
          f"> 1e-5: {np.sum(per > 1e-5)}/{n}, median {np.median(per):.2e}", flush=True)
