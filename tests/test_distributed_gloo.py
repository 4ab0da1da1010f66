"""Multi-process (world_size 2, gloo, CPU) checks of the data-parallel host logic:
batch sharding bounds and the deterministic ordered all-reduce of dtheta/loss.
The per-rank partials come from the CPU oracle (the GPU engine is exercised
by the -m gpu tests); the reduction must reproduce the single-process batch
gradient."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2206_01298_b200.distributed import reduce_grad, shard_bounds


def test_shard_bounds_cover_batch():
    for B in (1, 7, 512, 4096, 1000):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_bounds(B, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == B
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import core as oc
        from paper_2206_01298_b200.configs import make_config

        ci = make_config("C1", batch=12)
        lo, hi = shard_bounds(ci.batch, world, rank)
        fld = oc.MlpField(oc.Mlp(ci.widths, ci.activation, ci.theta))
        B = ci.batch

        def seed(uf):  # batch-global seed, like the engine's batch_global
            return float(np.sum(0.5 * np.sum(uf * uf, axis=1)) / B), uf / B

        r = oc.grad_terminal(fld, ci.scheme, ci.u0[lo:hi], ci.t0, ci.tF, ci.n_steps, seed_fn=seed)
        dth, loss = reduce_grad(torch.as_tensor(r["dtheta"]), r["loss"])
        dth2, loss2 = reduce_grad(torch.as_tensor(r["dtheta"]), r["loss"])
        out_q.put((rank, dth.numpy(), loss, bool(torch.equal(dth, dth2)), loss == loss2))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_reduction_matches_full_batch():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from oracle import core as oc
    from paper_2206_01298_b200.configs import make_config

    ci = make_config("C1", batch=12)
    full = oc.grad_terminal(oc.MlpField(oc.Mlp(ci.widths, ci.activation, ci.theta)), ci.scheme,
                            ci.u0, ci.t0, ci.tF, ci.n_steps)
    outs.sort(key=lambda o: o[0])
    for rank, dth, loss, det_d, det_l in outs:
        assert det_d and det_l                       # bit-reproducible
        assert oc.rel_error(dth, full["dtheta"]) <= 1e-13
        assert abs(loss - full["loss"]) <= 1e-13 * full["loss"]
    assert np.array_equal(outs[0][1], outs[1][1])    # every rank holds the same result
