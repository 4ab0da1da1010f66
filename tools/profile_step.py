"""Minimal driver for ncu: run ``--iters`` grad() calls of one config with
device-resident inputs (no CPU baseline, no e2e), e.g.

    python tools/profile_step.py --config C2 --policy revolve:8 --iters 3
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--policy", default=None)
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--phases", action="store_true")
    a = ap.parse_args()
    import torch

    from paper_2206_01298_b200.configs import make_config
    from paper_2206_01298_b200.workloads import field_from_config, run_config

    ci = make_config(a.config) if a.batch is None else make_config(a.config).subset(a.batch)
    fld = field_from_config(ci)
    from paper_2206_01298_b200.workloads import initial_state
    u0 = torch.as_tensor(initial_state(ci), dtype=fld.torch_dtype, device="cuda")
    for _ in range(a.iters):
        res = run_config(ci, a.policy, field=fld, u0=u0)
    torch.cuda.synchronize()
    if a.phases:
        from paper_2206_01298_b200.engine import phase_cycles
        phase_cycles(reset=True)
        res = run_config(ci, a.policy, field=fld, u0=u0, profile=True)
        cyc = phase_cycles(reset=True)
        tot = sum(cyc.values())
        tiles = res.device["tiles"]
        print("phase cycles per CTA (and share):")
        for k, v in cyc.items():
            if v:
                print(f"  {k:12s} {v / tiles / 1e6:8.3f} Mcyc  {100 * v / max(tot, 1):5.1f}%")
    print({k: v for k, v in res.device.items() if k.startswith("ms_") or k in ("tiles", "tile_rows")})


if __name__ == "__main__":
    main()
