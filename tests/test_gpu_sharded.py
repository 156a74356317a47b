"""Row-sharded CP-ARLS-LEV on one B200 through the in-process
shard simulator (cparls_comm_create_local: P shards, one host thread and one
CUDA stream each, host-rendezvous collectives).  Every mode step is run in
lockstep against the single-shard context from the same state: sampled rows
must be bit-identical (replicated sampling, no communication), the sharded
solve must equal the unsharded one to reduction-order rounding, and the fit to
1e-10."""
import threading

import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


def need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def on_shards(P, fn):
    """Run fn(p) for p in range(P) concurrently (collectives rendezvous)."""
    out, err = [None] * P, []

    def work(p):
        try:
            torch.cuda.set_device(0)
            out[p] = fn(p)
        except BaseException as e:   # noqa: BLE001
            err.append(e)

    ts = [threading.Thread(target=work, args=(p,)) for p in range(P)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    if err:
        raise err[0]
    return out


def make_shards(T, P, rank):
    from paper_2006_16438_b200 import Comm, Cparls
    comm = Comm.local(P)
    c = T.coords.cuda()
    v = T.vals.cuda()
    streams = [torch.cuda.Stream() for _ in range(P)]

    def create(p):
        return Cparls(T.dims, c[p::P].contiguous(), v[p::P].contiguous(), rank, comm=comm, world_size=P,
                      world_rank=p, stream=streams[p].cuda_stream)

    return comm, on_shards(P, create)


def lockstep_sharded(T, rank, P, iters, s, seed):
    need_gpu()
    from paper_2006_16438_b200 import Cparls
    g = Cparls(T.dims, T.coords.cuda(), T.vals.cuda(), rank)
    comm, shards = make_shards(T, P, rank)
    D = len(T.dims)
    for k in range(D):   # row blocks cover each mode exactly once
        spans = sorted(sh.owned_rows(k) for sh in shards)
        assert spans[0][0] == 0 and spans[-1][1] == T.dims[k]
        assert all(spans[i][1] == spans[i + 1][0] for i in range(P - 1))
    for t in range(iters):
        for k in range(D):
            for m in range(D):
                A, _ = g.get_factor(m)
                pt = g.get_ptilde(m)
                for sh in shards:
                    sh.set_factor(m, A)
                    sh.set_ptilde(m, pt)
            step = t * D + k
            gi = g.sample(k, s, seed, step)
            ref = g.get_sample()
            for sh in shards:
                si = sh.sample(k, s, seed, step)
                assert (si.s_det, si.s_bar, si.attempts) == (gi.s_det, gi.s_bar, gi.attempts)
                smp = sh.get_sample()
                assert (smp["keys"] == ref["keys"]).all() and (smp["counts"] == ref["counts"]).all()
            gs = g.solve_mode(k)
            infos = on_shards(P, lambda p: shards[p].solve_mode(k))
            for inf in infos:
                assert inf.matched_nnz == gs.matched_nnz and inf.touched_rows == gs.touched_rows
            _, Bg = g.last_solve(k)
            Ag, lg = g.get_factor(k)
            # factor getters of a sharded run are collective (only owned rows are current)
            lasts = on_shards(P, lambda p: shards[p].last_solve(k))
            facs = on_shards(P, lambda p: shards[p].get_factor(k))
            for p, sh in enumerate(shards):
                Bs = lasts[p][1]
                As, ls = facs[p]
                nb = np.linalg.norm(Bg)
                assert np.linalg.norm(Bs - Bg) <= 1e-11 * max(nb, 1e-300)
                np.testing.assert_allclose(ls, lg, rtol=1e-11)   # B^T B summation grouping differs by shard
                # p~ of all rows from the owners' rows (allgather of p~ only)
                np.testing.assert_allclose(sh.get_ptilde(k), g.get_ptilde(k), rtol=1e-10, atol=1e-16)
        fg = g.fit()
        fs = on_shards(P, lambda p: shards[p].fit())
        for f in fs:
            assert abs(f - fg) <= 1e-10, (f, fg)
    for sh in shards:
        sh.close()
    comm.close()


@pytest.mark.parametrize("P", [2, 3])
def test_sharded_c1_lockstep(P):
    T = synth.make("C1")
    lockstep_sharded(T, 3, P, 3, 256, 3)


@pytest.mark.parametrize("P", [4, 8])
def test_sharded_c2_lockstep(P):
    """C2 (Uber-shaped) at P = 4 and 8: mode 1 has 24 rows, so at P = 8 its Zipf
    head rows hold more than a rank's share and are split over the ranks."""
    T = synth.make("C2", device="cuda")
    T = synth.Tensor(T.cfg, T.dims, T.coords.cpu(), T.vals.cpu())
    if P == 8:
        from paper_2006_16438_b200 import plan_rows
        deg = np.bincount(T.coords[:, 1].numpy(), minlength=T.dims[1]).astype(np.uint64)
        _, heavy = plan_rows(deg, P, with_heavy=True)
        assert heavy.any()
    lockstep_sharded(T, 25, P, 1, 1 << 17, 3)


@pytest.mark.parametrize("s", [256, 1 << 14])
def test_sharded_communication_volume(s):
    """Per mode step a rank exchanges the cheaper of the sampled other-mode
    rows (s x (D-1) rows of ld doubles, from their owners) and those modes'
    dense factors, plus p~_k (n_k doubles) and r x r Grams -- never more
    (SURVEY 8(e)); both branches give the single-context samples."""
    need_gpu()
    T = synth.make("C2", device="cuda")
    T = synth.Tensor(T.cfg, T.dims, T.coords.cpu(), T.vals.cpu())
    P, r = 4, 25
    comm, shards = make_shards(T, P, r)
    for sh in shards:
        sh.reset_stats()
    on_shards(P, lambda p: shards[p].run(1, s, 3, fit_every=0))
    D = len(T.dims)
    ld = 32
    bound = 0.0
    for k in range(D):
        others = sum(n for m, n in enumerate(T.dims) if m != k)
        bound += 8.0 * (min(s * (D - 1), others) * ld + T.dims[k] + 64 * ld * P + 2 * r * r)
    for sh in shards:
        b = sh.stats()["bytes_comm"]
        assert 0 < b <= bound, (b, bound)
    for sh in shards:
        sh.close()
    comm.close()
