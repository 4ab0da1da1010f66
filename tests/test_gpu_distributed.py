"""World-size-2 data-parallel gradient through the engine (VERDICT r01 "next" #4).

Two processes share the one GPU of the test box, each running its batch shard
through ``grad_sharded`` (the native kernels) and reducing dtheta / loss over a
gloo group -- the same host logic bench.py runs over NCCL with one GPU per rank.
The ranks' kernels never wait on each other (the only exchange is the host-side
collective after each rank's sweep), so sharing one GPU is sound.

Checks: both ranks hold the same result; it is bit-identical to the ordered
fp64 sum of the two shards computed in one process (the determinism
contract); it equals the full-batch single call to rounding (the reduction
order differs: per-tile sums inside a shard, then shards); host-memory inputs
(numpy) give the same bits as device inputs.
"""

import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


# batches of the configs that would take long at full size (C3: tcgen05 conv tile, one image
# per CTA; C5: cluster theta kernels, two clusters per shard)
_BATCH = {"C3": 12, "C4": 96, "C5": 64}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, name, out_q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2206_01298_b200 import CheckpointPolicy, FixedController, tableau_catalog
        from paper_2206_01298_b200.configs import make_config
        from paper_2206_01298_b200.distributed import grad_sharded, shard_bounds
        from paper_2206_01298_b200.workloads import (field_from_config, initial_state, loss_for,
                                                     solver_from_config)

        ci = make_config(name, batch=_BATCH.get(name))
        lo, hi = shard_bounds(ci.batch, world, rank)
        fld = field_from_config(ci, rows=slice(lo, hi))
        args = (tableau_catalog(ci.scheme), loss_for(ci, slice(lo, hi)))
        y0 = initial_state(ci)[lo:hi]
        kw = dict(batch_global=ci.batch)
        pol = CheckpointPolicy.parse(ci.policy)
        dev = grad_sharded(fld, *args, torch.as_tensor(y0, dtype=fld.torch_dtype, device="cuda"),
                           ci.t0, ci.tF, FixedController(ci.n_steps), pol, solver_from_config(ci), **kw)
        host = grad_sharded(fld, *args, y0, ci.t0, ci.tF, FixedController(ci.n_steps), pol,
                            solver_from_config(ci), **kw)
        out_q.put((rank, dev.dtheta.cpu().numpy(), dev.loss, host.dtheta, host.loss,
                   dev.du0.cpu().numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_two_rank_grad_sharded_through_engine(name):
    import torch.multiprocessing as mp
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = sorted([q.get(timeout=600) for _ in range(world)], key=lambda o: o[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0

    from oracle import core as oc
    from paper_2206_01298_b200 import CheckpointPolicy, FixedController, grad, tableau_catalog
    from paper_2206_01298_b200.configs import make_config
    from paper_2206_01298_b200.distributed import shard_bounds
    from paper_2206_01298_b200.workloads import (field_from_config, initial_state, loss_for, run_config,
                                                 solver_from_config)

    ci = make_config(name, batch=_BATCH.get(name))
    # the same shards in one process, summed in rank order in fp64
    parts, losses, du0 = [], [], []
    for r in range(world):
        lo, hi = shard_bounds(ci.batch, world, r)
        fld = field_from_config(ci, rows=slice(lo, hi))
        res = grad(fld, tableau_catalog(ci.scheme), loss_for(ci, slice(lo, hi)),
                   torch.as_tensor(initial_state(ci)[lo:hi], dtype=fld.torch_dtype, device="cuda"),
                   ci.t0, ci.tF, FixedController(ci.n_steps), CheckpointPolicy.parse(ci.policy),
                   solver_from_config(ci), batch_global=ci.batch)
        parts.append(res.dtheta.double())
        losses.append(res.loss)
        du0.append(res.du0.cpu().numpy())
    expect = (parts[0] + parts[1]).to(res.dtheta.dtype).cpu().numpy()
    expect_loss = losses[0] + losses[1]
    for rank, dth, loss, hdth, hloss, rdu0 in outs:
        assert np.array_equal(dth, expect), rank            # bit-identical ordered reduction
        assert loss == expect_loss
        assert np.array_equal(hdth, dth) and hloss == loss   # host-memory inputs: same bits
        assert np.array_equal(rdu0, du0[rank])
    full = run_config(ci)
    tol = 1e-13 if ci.dtype == "f64" else 1e-4   # fp32: a different tile geometry per shard
    assert oc.rel_error(outs[0][1], full.dtheta.cpu().numpy() if isinstance(full.dtheta, torch.Tensor)
                        else full.dtheta) <= tol
    assert abs(outs[0][2] - full.loss) <= tol * abs(full.loss)
