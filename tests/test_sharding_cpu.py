"""Host-side logic of the row-sharded path on the CPU: the row
partition (cparls_plan_rows, a host-only library call) and the SPMD agreement
of two ranks over torch.distributed (gloo, world_size 2)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _plan(deg, P):
    from paper_2006_16438_b200 import build, plan_rows
    build.build()
    return plan_rows(deg, P)


@pytest.mark.parametrize("P", [1, 2, 3, 8])
def test_plan_rows_covers_and_balances(P):
    rng = np.random.default_rng(P)
    n = 5000
    deg = (rng.zipf(1.6, size=n) % 400).astype(np.uint64)
    b = _plan(deg, P)
    assert b[0] == 0 and b[-1] == n and (np.diff(b) >= 0).all()
    total = int(deg.sum())
    loads = [int(deg[b[p]:b[p + 1]].sum()) for p in range(P)]
    assert sum(loads) == total
    # every block is within one row of the ideal split
    assert max(loads) <= total / P + int(deg.max())


def test_plan_rows_degenerate():
    b = _plan(np.zeros(10, dtype=np.uint64), 4)
    assert b[0] == 0 and b[-1] == 10
    b = _plan(np.array([100, 0, 0, 0], dtype=np.uint64), 3)   # one heavy row
    assert b[-1] == 4 and (np.diff(b) >= 0).all()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import synth
    T = synth.make(synth.scaled("C2", 20_000))
    mine = T.coords[rank::world].to(torch.int64)
    res = []
    for k in range(len(T.dims)):
        deg = torch.bincount(mine[:, k], minlength=T.dims[k]).to(torch.int64)
        dist.all_reduce(deg)   # global per-row counts, as cparls_create does with NCCL
        b = _plan(deg.numpy().astype(np.uint64), world)
        res.append(b.tolist())
    # every rank must hold the same plan; gather them on rank 0
    out = [None] * world
    dist.all_gather_object(out, res)
    if rank == 0:
        q.put(out)
    dist.destroy_process_group()


def test_two_rank_plan_agreement_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert out[0] == out[1]
    import synth
    T = synth.make(synth.scaled("C2", 20_000))
    for k, b in enumerate(out[0]):
        deg = np.bincount(T.coords[:, k].numpy(), minlength=T.dims[k]).astype(np.uint64)
        assert b == _plan(deg, 2).tolist()   # equals the plan from the full tensor
