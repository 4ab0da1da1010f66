#!/usr/bin/env python
"""Benchmark: ODE-block forward + discrete-adjoint gradient, samples/s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--policy revolve:8]
    python bench.py --impl reference ...      # the CPU reference path (oracle port)

Workload (BASELINE.json configs[1], "C2"): MLP (64+t)-256-64 tanh, fp32,
Dopri5 x 40 on [0,1], binomial checkpointing with 8 slots, loss
0.5*mean||u(1)||^2, batch 4096 per GPU (weak scaling: each rank owns a
4096-sample shard of an N*4096 global batch; dtheta and the loss are reduced
once per step with a deterministic ordered all-gather-sum over NCCL).

One step = one full grad() over this rank's shard with inputs resident in HBM
(``value``); ``e2e`` re-times the same call through the public API from pinned
host memory with results read back.  L2 is flushed (256 MiB write) between
timed steps.  Rank 0 prints one JSON line.

``--gpus N`` outside torchrun starts N ranks itself (torch.distributed.run on
127.0.0.1).  ``--scaling strong`` keeps the global batch fixed and shards it
(the default for C3 / C4, whose BASELINE batch is a global batch).  At N = 1 the
line also carries ``per_config``: value, e2e, roofline and CPU baseline of the
other BASELINE configs (C1, C3, C4, C5), measured the same way with fewer steps.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ODE-block fwd+discrete-adjoint grad samples/s at 1–8 B200; % of roofline"
WORKLOADS = {
    "C1": "C1: MLP 64-256-64 tanh fp64, RK4 x10 on [0,1], store_all, B=512/GPU",
    "C2": "C2: MLP (64+t)-256-64 tanh fp32, Dopri5 x40 on [0,1], revolve:8, B=4096/GPU",
    "C3": "C3: conv ODE block 16x16x64 fp32, conv3x3(65->64)+relu+conv3x3(64->64), RK4 x10, "
          "store_all, GAP+linear+CE head, B=256/GPU",
    "C4": "C4: CNF (43+t)-860-860-43 softplus fp32 + Hutchinson (1 Rademacher probe), Dopri5 x20, "
          "store_all, NLL loss, B=1000/GPU",
    "C5": "C5: stiff a*u + 0.1*MLP 128-512-128 tanh fp64, Crank-Nicolson x20, Newton 1e-10 + "
          "GMRES(30) (maxit 1000), store_all, B=256/GPU",
}


PER_GPU = {"C1": 512, "C2": 4096, "C3": 256, "C4": 1000, "C5": 256}
# BASELINE: C3 / C4 are a fixed global batch sharded over the GPUs (strong scaling);
# C1 / C2 / C5 keep their batch per GPU (weak scaling)
DEFAULT_SCALING = {"C1": "weak", "C2": "weak", "C3": "strong", "C4": "strong", "C5": "weak"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--policy", default=None)
    ap.add_argument("--scaling", default=None, choices=["weak", "strong"],
                    help="weak: batch per GPU fixed; strong: global batch fixed (default per config)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--per-config", default="C1,C3,C4,C5",
                    help="configs also measured (N=1 only) into the line's per_config block; '' for none")
    ap.add_argument("--per-config-steps", type=int, default=3)
    return ap.parse_args()


def relaunch_distributed(args) -> int:
    """--gpus N > 1 outside torchrun: start N ranks (one per GPU) on this node."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__),
           *sys.argv[1:]]
    return subprocess.call(cmd)


# ----------------------------------------------------------------- CPU side
def _cpu_worker_init(cfg_name, policy):
    global _W
    from paper_2206_01298_b200.configs import make_config
    ci = make_config(cfg_name).subset(64)
    _W = (ci, policy)


def _cpu_task(idx):
    """One sample through the oracle's per-sample path (the reference's
    forward_pass + backward_sweep restated, GEMV per sample like odegrad)."""
    from oracle.problems import run_oracle
    ci, policy = _W
    i = idx % ci.batch
    run_oracle(ci, policy, rows=slice(i, i + 1))
    return 1


class CpuPool:
    def __init__(self, cfg_name, policy):
        import multiprocessing as mp
        self.cores = len(os.sched_getaffinity(0))
        ctx = mp.get_context("spawn")
        env_threads = {k: os.environ.get(k) for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS")}
        os.environ["OMP_NUM_THREADS"] = "1"
        os.environ["OPENBLAS_NUM_THREADS"] = "1"
        self.pool = ctx.Pool(self.cores, initializer=_cpu_worker_init, initargs=(cfg_name, policy))
        for k, v in env_threads.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
        self.pool.map(_cpu_task, range(self.cores))          # warm every worker

    def run(self, n_samples):
        t0 = time.perf_counter()
        done = sum(self.pool.map(_cpu_task, range(n_samples), chunksize=1))
        return done, time.perf_counter() - t0

    def rate_for(self, seconds):
        """samples/s from a bounded sample of about ``seconds`` of CPU work."""
        done, el = self.run(self.cores)
        per = el / max(1, done // self.cores)
        n = max(self.cores, int(seconds / max(per, 1e-6)) * self.cores)
        done, el = self.run(n)
        return done / el, done, el

    def close(self):
        self.pool.terminate()


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from paper_2206_01298_b200.configs import make_config
    ci = make_config(args.config, batch=1)
    policy = args.policy or ci.policy
    scaling = args.scaling or DEFAULT_SCALING[args.config]
    gb = PER_GPU[args.config] * (args.gpus if scaling == "weak" else 1)
    pool = CpuPool(args.config, policy)
    per_step = pool.cores * 2
    for _ in range(args.warmup):
        pool.run(pool.cores)
    times = []
    total = 0
    for _ in range(args.steps):
        done, el = pool.run(per_step)
        times.append(el)
        total += done
    pool.close()
    value = total / sum(times)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "samples/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * statistics.mean(times), "higher_is_better": True, "scaling": scaling,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE shapes)",
        "config": {"workload": WORKLOADS.get(args.config, args.config), "policy": policy,
                   "global_batch": gb, "scheme": ci.scheme, "n_steps": ci.n_steps,
                   "samples_per_step": per_step,
                   "note": "each step is a bounded sample of the workload: samples_per_step "
                           "samples of the global batch on the host cores"},
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": pool.cores, "kind": "port",
                         "sample": f"{per_step} samples/step of {args.config} through the oracle's "
                                   "per-sample restatement of odegrad forward_pass+backward_sweep, "
                                   "one process per core"},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock + throttle reasons sampled DURING the timed region: NVML polled
    in-process every ~2 ms (short timed regions still get samples); nvidia-smi
    polling is the fallback when NVML is unavailable."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    # NVML clocks-event reason bits
    REASONS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
               "hw_thermal_slowdown": 0x40}

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None
        self.nv = None
        self.stop_evt = threading.Event()

    def start(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.mx = float(nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM))
            self.nv = nv
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
            return
        except Exception:
            self.nv = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _poll(self):
        nv = self.nv
        get_r = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        while not self.stop_evt.is_set():
            try:
                self.rows.append((float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)),
                                  int(get_r(self.h))))
            except Exception:
                pass
            self.stop_evt.wait(0.002)

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.nv is not None:
            self.stop_evt.set()
            self.thread.join(timeout=5)
            sm = [r[0] for r in self.rows]
            reasons = {nm for nm, bit in self.REASONS.items() if any(r[1] & bit for r in self.rows)}
            return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.mx,
                    "reasons": sorted(reasons), "samples": len(sm), "source": "nvml"}
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx = float(r[1])
                for nm, v in zip(names, r[4:8]):
                    if v.lower() == "active":
                        reasons.add(nm)
            except (ValueError, IndexError):
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvidia-smi"}


# ----------------------------------------------------------------- GPU side
def fp_peak(dtype):
    """FP32/FP64 FMA-pipe peak: builder-measured on this pool (tools/peaks_probe.cu,
    profiles/fp_peaks.json), or the nominal B200 figure, with the source named."""
    path = os.path.join(ROOT, "profiles", "fp_peaks.json")
    key = "fp32_tflops" if dtype == "f32" else "fp64_tflops"
    try:
        with open(path) as fh:
            d = json.load(fh)
        return float(d[key]), "builder-measured FMA peak (tools/peaks_probe.cu -> profiles/fp_peaks.json)"
    except (OSError, KeyError, ValueError):
        nominal = 148 * (128 if dtype == "f32" else 64) * 2 * 1.965e9 / 1e12
        return nominal, "nominal 148 SM x FMA lanes x 2 x 1.965 GHz"


def bf16_peak():
    """Driver-measured dense bf16 tensor throughput (MEASURED_PEAKS.json), burst figure:
    the dominant kernel is timed alone by its own CUDA events."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["bf16_tflops"]), "MEASURED_PEAKS.json bf16_tflops (burst)"
    except (OSError, KeyError, ValueError):
        return 2250.0, "nominal B200 dense bf16 (2.25 PFLOP/s)"


def roofline(ci, scheme, dev, nloc, phases, K, policy_key):
    """Roofline of the dominant kernel: EXECUTED algorithmic FLOPs per launch (SURVEY
    8d per-unit work x the samples of one launch; stage evaluations / VJPs the device
    skips are not counted) / its CUDA-event time measured in-library on the launch
    stream.  Per-sample work: MLP f-eval 2 Pw, VJP pair 4 Pw; CNF
    f_aug (f and J eps) 4 Pw, VJP 8 Pw; conv f-eval 2 * 256 * 9 * (65*64 + 64*64),
    VJP twice that; theta methods (NFE-F + NFE-B) * 2 Pw."""
    Pw = sum(ci.widths[l] * ci.widths[l + 1] for l in range(len(ci.widths) - 1))
    if ci.kind == "conv":
        Pw = 256 * 9 * (65 * 64 + 64 * 64)
    s = scheme.stages
    replays = dev["steps_recomputed"]
    fe, ve = (4, 8) if ci.kind == "cnf" else (2, 4)
    if scheme.kind == "theta":
        fwd_flops = nloc * dev["nfe_forward"] * 2 * Pw
        rev_flops = nloc * dev["nfe_backward"] * 2 * Pw
    else:
        tab = scheme.tableau
        unused = sum(1 for i in range(s) if tab.b[i] == 0.0 and not np.any(tab.a[i + 1:, i]))
        rs = replays * (s - unused)                       # replayed stage evaluations executed
        fwd_evals = dev["device_rhs_evals"] - rs
        fwd_flops = nloc * fwd_evals * fe * Pw
        rev_flops = nloc * (rs * fe * Pw + dev["device_vjp_evals"] * ve * Pw)
    kern = {"forward": (phases["ms_forward"] / K, fwd_flops),
            "reverse": (phases["ms_reverse"] / K, rev_flops)}
    dom = max(kern, key=lambda k: kern[k][0])
    dms, dfl = kern[dom]
    peak, peak_src = fp_peak(ci.dtype)
    achieved = dfl / (dms / 1e3) / 1e12
    pipe, bound, tc_extra = f"{ci.dtype} FMA (SIMT)", "compute", {}
    if dev.get("tensor_cores") == 2:   # fp64 cluster MLP: same 64 FMA/clk/SM on the DMMA pipe as on the vector pipe
        pipe = "f64 mma.sync m8n8k4 (weights resident across a cluster of 8 CTAs) + f64 FMA"
    if dev.get("tensor_cores") == 1:
        # tcgen05 kind::f16 tile: each fp32 product is 3 bf16 MMAs (hi*hi + hi*lo + lo*hi),
        # so the fp32-equivalent ceiling is the measured dense bf16 peak / 3; the executed
        # tensor-pipe FLOPs (split passes and the sample-column padding included) are
        # reported beside it
        bf16, bf16_src = bf16_peak()
        peak, peak_src = bf16 / 3.0, f"{bf16_src} / 3 (3-pass bf16 split)"
        pipe, bound = "tcgen05 kind::f16 (bf16 3-pass split, fp32 accumulate in TMEM)", "tensor"
        if ci.kind == "conv":   # fp16 two-term split (same 3 passes at the same rate), one tap per TMEM partial
            peak_src = f"{bf16_src} / 3 (3-pass fp16 split)"
            pipe = "tcgen05 kind::f16 (fp16 3-pass split, per-tap TMEM partials summed in fp32 registers)"
    if dev.get("tensor_cores") == 1 and ci.kind == "mlp":
        D0, H = ci.widths[-1], ci.widths[1]
        nmb, t = H // 128, dev["tiles"]
        ncol = 32   # MMA N per tile (samples, padded)
        ev = 2 * 3 * (128 * ncol * D0 * nmb + 64 * ncol * H)                    # one f-eval
        vj = 2 * 3 * (4 * 128 * ncol * D0 * nmb + 64 * ncol * H)   # z, dW2^T, dH, dW1 + dX
        tab = scheme.tableau
        unused = sum(1 for i in range(s) if tab.b[i] == 0.0 and not np.any(tab.a[i + 1:, i]))
        rs = replays * (s - unused)
        dev_fwd = t * (dev["device_rhs_evals"] - rs) * ev
        dev_rev = t * (rs * ev + dev["device_vjp_evals"] * vj)
        ex = dev_rev if dom == "reverse" else dev_fwd
        tc_extra = {"tensor_pipe_flops_per_launch": ex,
                    "tensor_pipe_tflops": ex / (dms / 1e3) / 1e12,
                    "tensor_pipe_frac": ex / (dms / 1e3) / 1e12 / bf16}
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            traffic = json.load(fh).get(f"{ci.name}:{policy_key}:{dom}")
    except (OSError, ValueError):
        pass
    return {"bound": bound, "pipe": pipe, "kernel": dom, "achieved": achieved, "peak": peak,
            "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
            "algorithmic_flops_per_launch": dfl, "ms_per_launch": dms,
            "phase_ms_per_step": {k: v / K for k, v in phases.items()}, **tc_extra}


def measure(name, args, steps, warmup, world, rank, local, flush, policy_arg=None, cpu=True):
    """One config: device-resident timing (value), end-to-end timing from pinned host
    memory (e2e), the dominant kernel's roofline, and (rank 0, N=1) the CPU baseline."""
    import torch
    import torch.distributed as dist

    from paper_2206_01298_b200 import CheckpointPolicy, FixedController, tableau_catalog
    from paper_2206_01298_b200.configs import make_config
    from paper_2206_01298_b200.distributed import grad_sharded, shard_bounds
    from paper_2206_01298_b200.engine import grad
    from paper_2206_01298_b200.workloads import (field_from_config, initial_state, loss_for,
                                                 solver_from_config)

    base = make_config(name, batch=1)
    scaling = (args.scaling if name == args.config else None) or DEFAULT_SCALING[name]
    per_gpu = PER_GPU[name]
    gb = per_gpu * world if scaling == "weak" else per_gpu
    ci = make_config(name, batch=gb)
    lo, hi = shard_bounds(ci.batch, world, rank)
    policy = CheckpointPolicy.parse(policy_arg or base.policy)
    field = field_from_config(ci, rows=slice(lo, hi))
    scheme = tableau_catalog(ci.scheme)
    loss = loss_for(ci, slice(lo, hi))
    ctrl = FixedController(ci.n_steps)
    scfg = solver_from_config(ci)
    tdt = field.torch_dtype
    y0 = initial_state(ci)[lo:hi]
    u0_dev = torch.as_tensor(y0, dtype=tdt, device="cuda").contiguous()
    u0_host = torch.as_tensor(y0, dtype=tdt).pin_memory()

    def step(u0):
        if world > 1:
            return grad_sharded(field, scheme, loss, u0, ci.t0, ci.tF, ctrl, policy, scfg,
                                batch_global=ci.batch)
        return grad(field, scheme, loss, u0, ci.t0, ci.tF, ctrl, policy, scfg)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(max(3, warmup)):
        res = step(u0_dev)
    # ---- device-resident timing (value): inputs in HBM, L2 flushed between steps
    sampler = ClockSampler(local)
    sampler.start()
    ms, phases = [], {"ms_pack": 0.0, "ms_forward": 0.0, "ms_reverse": 0.0, "ms_reduce": 0.0}
    launches = 0
    stream = torch.cuda.current_stream()
    for _ in range(steps):
        flush.zero_()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        res = step(u0_dev)
        e1.record(stream)
        barrier()
        ms.append(e0.elapsed_time(e1))
        for k in phases:
            phases[k] += res.device[k]
        launches += res.device["kernel_launches"]
    clocks = sampler.stop()
    ms_step = statistics.mean(ms)
    # ---- end-to-end through the public API from pinned host memory (H2D in, results D2H)
    # warm-up: the results come back in pinned staging buffers from torch's caching host
    # allocator, and two generations of them are alive at once (the previous result is
    # released after the next call returns); four calls that hold their result populate the cache, otherwise
    # cudaHostAlloc (milliseconds per 16 MB) lands in the timed steps
    r = None
    for _ in range(4):
        r = step(u0_host)   # held like in the timed loop, so both generations get allocated
    e2e_s = []
    for _ in range(steps):
        flush.zero_()
        barrier()
        t0 = time.perf_counter()
        r = step(u0_host)
        _ = (np.asarray(r.dtheta) if not isinstance(r.dtheta, torch.Tensor) else r.dtheta.cpu(), r.loss)
        e2e_s.append(time.perf_counter() - t0)
    e2e_mean = statistics.mean(e2e_s)
    if world > 1:
        t = torch.tensor([ms_step, e2e_mean], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step, e2e_mean = float(t[0]), float(t[1])
    value = ci.batch / (ms_step / 1e3)
    esz = 4 if ci.dtype == "f32" else 8
    nloc = hi - lo
    h2d = y0.size * esz
    d2h = 2 * y0.size * esz + field.n_params * esz + 8
    dev = res.device
    rf = roofline(ci, scheme, dev, nloc, phases, steps, str(policy))
    cpu_b = None
    if cpu and rank == 0 and world == 1 and not args.no_cpu_baseline:
        pool = CpuPool(name, str(policy))
        rate, done, el = pool.rate_for(args.cpu_seconds)
        pool.close()
        cpu_b = {"value": rate, "unit": "samples/s", "cores": pool.cores, "kind": "port",
                 "sample": f"{done} samples of {name} in {el:.1f}s through the oracle's "
                           "per-sample restatement of odegrad forward_pass+backward_sweep, "
                           "one process per core"}
    return {
        "value": value, "ms_per_step": ms_step, "scaling": scaling, "dtype": ci.dtype,
        "config": {"workload": WORKLOADS.get(name, name), "global_batch": ci.batch,
                   "batch_per_gpu": nloc, "scheme": ci.scheme, "n_steps": ci.n_steps,
                   "policy": str(policy), "parallelism": f"dp{world}",
                   "l2": "flushed (256 MiB write) between timed steps",
                   "tile_rows": dev["tile_rows"], "tiles": dev["tiles"]},
        "e2e": {"value": ci.batch / e2e_mean, "unit": "samples/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h},
        "gpu_launches": launches, "roofline": rf, "cpu_baseline": cpu_b, "clocks": clocks,
        "counters": {k: dev[k] for k in ("nfe_forward", "nfe_backward", "steps_recomputed",
                                         "max_live_slots", "device_vjp_evals")},
        "loss": res.loss,
    }


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_distributed(args)
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    flush = torch.empty(256 * 2**20 // 4, dtype=torch.float32, device="cuda")
    head = measure(args.config, args, args.steps, args.warmup, world, rank, local, flush, args.policy)
    per_config = {}
    if world == 1 and args.per_config:
        for name in [c for c in args.per_config.split(",") if c and c != args.config]:
            r = measure(name, args, args.per_config_steps, 3, world, rank, local, flush)
            per_config[name] = {k: r[k] for k in ("value", "ms_per_step", "dtype", "config", "e2e",
                                                  "roofline", "cpu_baseline", "clocks", "loss")}
    if rank == 0:
        line = {
            "metric": METRIC, "value": head["value"], "unit": "samples/s", "n_gpus": world,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": head["ms_per_step"],
            "higher_is_better": True, "scaling": head["scaling"], "vs_baseline": None,
            "dtype": head["dtype"], "data": "synthetic (seeded, BASELINE shapes)",
            **{k: head[k] for k in ("config", "e2e", "gpu_launches", "roofline", "cpu_baseline",
                                    "clocks", "counters", "loss")},
        }
        if per_config:
            line["per_config"] = per_config
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
