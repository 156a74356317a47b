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
    from paper_2006_16438_b200 import build, plan_rows
    build.build()
    b, heavy = plan_rows(deg, P, with_heavy=True)
    assert b[0] == 0 and b[-1] == n and (np.diff(b) >= 0).all()
    total = int(deg.sum())
    # heavy rows: more nonzeros than a rank's share, spread over all ranks
    assert (heavy == ((deg > total // P) & (P > 1))).all()
    w = np.where(heavy, (deg + P - 1) // P, deg).astype(np.int64)
    loads = [int(w[b[p]:b[p + 1]].sum()) for p in range(P)]
    assert sum(loads) == int(w.sum())
    # every block is within one row's weight of the ideal split
    assert max(loads) <= w.sum() / P + int(w.max())


def test_plan_rows_degenerate():
    b = _plan(np.zeros(10, dtype=np.uint64), 4)
    assert b[0] == 0 and b[-1] == 10
    from paper_2006_16438_b200 import plan_rows
    b, heavy = plan_rows(np.array([100, 0, 0, 0], dtype=np.uint64), 3, with_heavy=True)   # one heavy row
    assert b[-1] == 4 and (np.diff(b) >= 0).all()
    assert heavy.tolist() == [True, False, False, False]


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


def _step_worker(rank, world, port, q):
    """One sharded CP-ARLS-LEV mode step on the CPU: the
    library's host-side rules (cparls_plan_rows with heavy rows,
    cparls_route_nonzeros) place the nonzeros, gloo carries the exchanges the
    GPU path makes with NCCL (build-time all-to-all, heavy-row RHS partials,
    the owned-row Gram, the p~ allgather), and the oracle stands in for the
    kernels on each rank's slice."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import synth
    from paper_2006_16438_b200 import build, plan_rows, route_nonzeros
    build.build()
    dims, coords_all, vals_all = _skewed_tensor()
    chunk = np.arange(rank, len(vals_all), world)            # this rank's input chunk
    r, s, seed, k = 5, 512, 7, 1                              # mode 1, row 0 holds > 1/2 of the nonzeros: heavy
    g = np.random.default_rng(3)
    As = [g.uniform(size=(n, r)) + 0.05 for n in dims]
    # build-time routing of mode k (global degrees, plan, all-to-all)
    deg = torch.from_numpy(np.bincount(coords_all[chunk, k], minlength=dims[k]).astype(np.int64))
    dist.all_reduce(deg)
    bound, heavy = plan_rows(deg.numpy().astype(np.uint64), world, with_heavy=True)
    dest = route_nonzeros(coords_all[chunk], k, world, bound, heavy)
    sent = [chunk[dest == p] for p in range(world)]
    got = [None] * world
    dist.all_gather_object(got, sent)
    mine = np.sort(np.concatenate([got[p][rank] for p in range(world)]))
    lo, hi = int(bound[rank]), int(bound[rank + 1])
    # the rank's slice: one sampled mode step (identical sample on every rank)
    o = oracle.Oracle(dims, coords_all[mine], vals_all[mine], r)
    for m, A in enumerate(As):
        o.set_factor(m, A)
    o.sample(k, s, -1.0, seed, 0)
    keys = o.get_sample()["keys"]
    o.solve_mode(k)
    G, M, _ = o.last_solve(k)
    # rows of M this rank must not touch: non-heavy rows outside its block
    outside = np.ones(dims[k], dtype=bool)
    outside[lo:hi] = False
    assert not M[outside & ~heavy].any()
    # heavy rows: partial RHS rows summed over the ranks (the library: int64 sums)
    Mh = torch.from_numpy(M[heavy].copy())
    dist.all_reduce(Mh)
    M[heavy] = Mh.numpy()
    w, V = np.linalg.eigh(G)
    keep = w > r * np.finfo(float).eps * w.max()
    Gp = (V[:, keep] / w[keep]) @ V[:, keep].T
    B_own = M[lo:hi] @ Gp                                     # the owner solves its block (heavy rows included)
    BtB = torch.from_numpy(B_own.T @ B_own)
    dist.all_reduce(BtB)                                      # Gram of B over the owned rows
    lam = np.sqrt(np.diag(BtB.numpy()))
    GA = BtB.numpy() / np.outer(lam, lam)
    wa, Va = np.linalg.eigh(GA)
    ka = wa > r * np.finfo(float).eps * wa.max()
    A_own = B_own / lam
    ell_own = np.einsum("ij,jk,ik->i", A_own, (Va[:, ka] / wa[ka]) @ Va[:, ka].T, A_own)
    parts = [None] * world
    dist.all_gather_object(parts, (lo, hi, ell_own, B_own, keys))
    if rank == 0:
        q.put((parts, heavy.tolist()))
    dist.destroy_process_group()


def _skewed_tensor():
    """20 x 12 x 15 x 10 with every cell of mode-1 row 0 present (3000) and 8%
    of the others: row 0 holds more than half the nonzeros (a heavy row at
    world size 2) and every sampled fiber is populated."""
    g = np.random.default_rng(5)
    dims = (20, 12, 15, 10)
    cells = np.stack(np.unravel_index(np.arange(np.prod(dims)), dims, order="F"), 1).astype(np.int64)
    keep = (cells[:, 1] == 0) | (g.uniform(size=len(cells)) < 0.08)
    coords = cells[keep]
    coords = coords[g.permutation(len(coords))]
    return dims, coords, g.uniform(0.5, 2.0, len(coords))


def test_two_rank_sharded_mode_step_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_step_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    parts, heavy = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert any(heavy)                                          # the split path was exercised
    import oracle
    dims, coords_all, vals_all = _skewed_tensor()
    r, s, seed, k = 5, 512, 7, 1
    g = np.random.default_rng(3)
    As = [g.uniform(size=(n, r)) + 0.05 for n in dims]
    o = oracle.Oracle(dims, coords_all, vals_all, r)
    for m, A in enumerate(As):
        o.set_factor(m, A)
    o.sample(k, s, -1.0, seed, 0)
    keys = o.get_sample()["keys"]
    o.solve_mode(k)
    _, _, B_ref = o.last_solve(k)
    ell_ref, _ = oracle.leverage(B_ref)
    assert (parts[0][4] == keys).all() and (parts[1][4] == keys).all()   # replicated sampling
    B = np.zeros_like(B_ref)
    ell = np.zeros(dims[k])
    for lo, hi, e, b, _ in parts:
        B[lo:hi] = b
        ell[lo:hi] = e
    assert parts[0][0] == 0 and parts[0][1] == parts[1][0] and parts[1][1] == dims[k]
    np.testing.assert_allclose(B, B_ref, rtol=1e-10, atol=1e-12 * np.abs(B_ref).max())
    np.testing.assert_allclose(ell, ell_ref, rtol=1e-9, atol=1e-12)


def test_generator_rank_chunks_are_slices_of_the_tensor():
    """bench.py --gpus N builds each rank's chunk only (synth.make part/parts):
    rank p's chunk is cells p, p + N, ... of the single-GPU tensor."""
    import synth
    cfg = synth.scaled("C2", 40_000)
    T = synth.make(cfg)
    for P in (2, 3):
        for p in range(P):
            ch = synth.make(cfg, part=p, parts=P)
            assert torch.equal(ch.coords, T.coords[p::P]) and torch.equal(ch.vals, T.vals[p::P])
