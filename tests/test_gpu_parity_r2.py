"""GPU parity, round 2: the method branches and workload shapes the round-1
lockstep did not reach, each against the CPU oracle through the C ABI.

* AMB-6 truncation: |DetSet| > s, with ties at the cut, on DIDX's
  brute-force-sized and pruned paths;
* AMB-7 skip: a point mass (every drawable row deterministic) and
  1 - p_det <= 1e-12;
* multi-window SIDX (AMB-8): opts.sidx_window forces the continuation over
  many windows; attempts, keys and counts stay bit-exact and equal the
  single-window run;
* C3 (Enron-shaped, 4-way, 36-43-bit keys, fp64 values): one lockstep
  iteration at full size;
* C5 dims (Reddit-shaped: 46-bit keys, fp32 log(1+c) values) at reduced nnz:
  one lockstep iteration.
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from test_gpu_parity import compare_sample, kept_kappa, lockstep, log_solve, need_gpu, solve_tol

pytestmark = pytest.mark.gpu


def _ctx(dims, coords, vals, r, **kw):
    from paper_2006_16438_b200 import Cparls
    return Cparls(dims, torch.from_numpy(coords).cuda(), torch.from_numpy(vals).cuda(), r, **kw)


def _tiny_tensor(dims, nnz, seed):
    g = np.random.default_rng(seed)
    coords = np.stack([g.integers(0, n, nnz) for n in dims], 1).astype(np.int64)
    coords = np.unique(coords, axis=0)
    vals = g.uniform(0.5, 2.0, len(coords))
    return coords, vals


def _step_lockstep(g, o, k, s, tau, seed, step):
    gi = g.sample(k, s, seed, step)
    oi = o.sample(k, s, tau, seed, step)
    assert (gi.s_det, gi.s_rnd, gi.s_bar, gi.attempts, gi.skipped_random) == \
           (oi.s_det, oi.s_rnd, oi.s_bar, oi.attempts, oi.skipped_random)
    assert abs(gi.p_det - oi.p_det) <= 1e-14 * max(1.0, oi.p_det)
    compare_sample(g, o)
    gs, os_ = g.solve_mode(k), o.solve_mode(k)
    assert gs.matched_nnz == os_.matched_nnz and gs.touched_rows == os_.touched_rows
    Gg, Bg = g.last_solve(k)
    Go, _, Bo = o.last_solve(k)
    np.testing.assert_allclose(Gg, Go, rtol=1e-11, atol=1e-13 * max(1.0, np.abs(Go).max()))
    nb = np.linalg.norm(Bo)
    if nb > 0:
        tol = solve_tol(Go, f"r2 step k={k} s={s} tau={tau}")
        rel = np.linalg.norm(Bg - Bo) / nb
        log_solve(rel)
        assert rel <= tol, (rel, tol)
    return gi


@pytest.mark.parametrize("case", ["brute_path", "pruned_path"])
def test_gpu_didx_truncation_matches_oracle(case):
    """AMB-6: s_det > s keeps the top s by (p desc, key asc), s_rnd = 0."""
    need_gpu()
    if case == "brute_path":
        pts = [np.array([0.3, 0.3, 0.2, 0.1, 0.1]), np.array([0.25, 0.25, 0.2, 0.1, 0.1, 0.1])]
        tau, s = 1e-3, 7
    else:
        nA, nB = 4000, 3000
        pA = np.full(nA, 0.2 / (nA - 4)); pA[[7, 100, 2500, 3999]] = 0.2
        pB = np.full(nB, 0.25 / (nB - 3)); pB[[0, 1500, 2999]] = 0.25
        pts, tau, s = [pA, pB], 1e-6, 5
    dims = (6, len(pts[0]), len(pts[1]))
    coords, vals = _tiny_tensor(dims, 3000, 41)
    # put nonzeros on the kept fibers so the solve has work
    big0, big1 = np.argsort(-pts[0])[:4], np.argsort(-pts[1])[:3]
    extra = np.array([[i, a, b] for i in range(6) for a in big0 for b in big1], dtype=np.int64)
    coords = np.unique(np.concatenate([coords, extra]), axis=0)
    vals = np.random.default_rng(42).uniform(0.5, 2.0, len(coords))
    g = _ctx(dims, coords, vals, 2, tau=tau)
    o = oracle.Oracle(dims, coords, vals, 2)
    for m in range(3):
        A, _ = g.get_factor(m)
        o.set_factor(m, A)
    for j, pt in enumerate(pts):
        g.set_ptilde(j + 1, pt)
        o.set_ptilde(j + 1, pt)
    gi = _step_lockstep(g, o, 0, s, tau, 77, 3)
    assert gi.s_det == s and gi.s_rnd == 0 and gi.s_bar == s


@pytest.mark.parametrize("variant", ["point_mass", "p_det_near_one"])
def test_gpu_amb7_skip_matches_oracle(variant):
    """AMB-7: the random phase is skipped when every drawable row is
    deterministic, or when 1 - p_det <= 1e-12 (flag, s_bar = s_det)."""
    need_gpu()
    dims = (5, 3, 4)
    coords, vals = _tiny_tensor(dims, 40, 43)
    coords = np.unique(np.concatenate([coords, np.array([[i, 1, 2] for i in range(5)])]), axis=0)
    vals = np.random.default_rng(44).uniform(0.5, 2.0, len(coords))
    if variant == "point_mass":
        pts = [np.array([0.0, 1.0, 0.0]), np.array([0.0, 0.0, 1.0, 0.0])]
    else:
        e = 1e-14
        pts = [np.array([e, 1.0 - 2 * e, e]), np.array([0.0, 0.0, 1.0, 0.0])]
    g = _ctx(dims, coords, vals, 2)
    o = oracle.Oracle(dims, coords, vals, 2)
    for m in range(3):
        o.set_factor(m, g.get_factor(m)[0])
    for j, pt in enumerate(pts):
        g.set_ptilde(j + 1, pt)
        o.set_ptilde(j + 1, pt)
    gi = _step_lockstep(g, o, 0, 16, -1.0, 5, 0)
    assert gi.skipped_random == 1 and gi.s_det == 1 and gi.s_bar == 1


@pytest.mark.parametrize("window", [1, 17, 128])
def test_gpu_sidx_multi_window_bit_exact(window):
    """AMB-8: the SIDX result is the first s_rnd accepted attempts in attempt
    order whatever the window size: windows of 1, 17 and 128 attempts give
    the oracle's sample (attempts included) and the default-window sample."""
    need_gpu()
    from paper_2006_16438_b200 import Cparls
    T = synth.make("C1")
    cfg = T.cfg
    lockstep_ctx = Cparls(T.dims, T.coords.cuda(), T.vals.cuda(), cfg.rank, sidx_window=window)
    ref = Cparls(T.dims, T.coords.cuda(), T.vals.cuda(), cfg.rank)
    o = oracle.Oracle(T.dims, T.coords.to(torch.int64).numpy(), T.vals.numpy(), cfg.rank)
    for k in range(3):
        for m in range(3):
            A, _ = lockstep_ctx.get_factor(m)
            o.set_factor(m, A)
            ref.set_factor(m, A)
            pt = lockstep_ctx.get_ptilde(m)
            o.set_ptilde(m, pt)
            ref.set_ptilde(m, pt)
        gi = _step_lockstep(lockstep_ctx, o, k, cfg.s, -1.0, cfg.sample_seed, k)
        ri = ref.sample(k, cfg.s, cfg.sample_seed, k)
        assert (gi.s_det, gi.s_bar, gi.attempts) == (ri.s_det, ri.s_bar, ri.attempts)
        assert gi.attempts > window          # the continuation really ran
        a, b = lockstep_ctx.get_sample(), ref.get_sample()
        assert (a["keys"] == b["keys"]).all() and (a["counts"] == b["counts"]).all()


def test_c3_lockstep_one_iteration():
    """C3 (BASELINE configs[2], Enron-shaped 6066 x 5699 x 244268 x 1176,
    54.2M nonzeros, fp64 counts, 36-43-bit keys): one lockstep iteration of
    all four modes plus the fit, at full size."""
    T = synth.make("C3", device="cuda")
    T = synth.Tensor(T.cfg, T.dims, T.coords.cpu(), T.vals.cpu())
    lockstep(T, T.cfg.rank, 1, T.cfg.s, T.cfg.sample_seed)


def test_c5_dims_reduced_nnz_lockstep():
    """C5 dims (BASELINE configs[4], Reddit-shaped 8,211,298 x 176,962 x
    8,116,559: 41/46/41-bit keys) with fp32 log(1+c) values (the C5 value
    recipe) at 2M nonzeros: one lockstep iteration plus the fit."""
    need_gpu()
    cfg = synth.scaled("C5", 2_000_000)
    T = synth.make(cfg, device="cuda")
    assert T.vals.dtype == torch.float32
    Tc = synth.Tensor(T.cfg, T.dims, T.coords.cpu(), T.vals.cpu())
    lockstep(Tc, cfg.rank, 1, cfg.s, cfg.sample_seed)


# ---------------------------------------------------------------- sync-free mode step
def _factors(g):
    return [g.get_factor(m) for m in range(g.D)]


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_run_is_sync_free_and_equals_stepwise(name):
    """cparls_run enqueues every mode step without host synchronisation (one
    synchronisation per call, counted by cparls_stats.host_syncs) and gives
    the bit-identical factors and fit trace of the same steps taken one
    cparls_sample + cparls_solve_mode at a time (the fixed-point RHS makes a
    step's result independent of how it was scheduled)."""
    need_gpu()
    from paper_2006_16438_b200 import Cparls
    T = synth.make(name) if name == "C1" else synth.make(name, device="cuda")
    cfg = T.cfg
    a = Cparls(T.dims, T.coords.cuda(), T.vals.cuda(), cfg.rank)
    b = Cparls(T.dims, T.coords.cuda(), T.vals.cuda(), cfg.rank)
    iters = 3
    a.reset_stats()
    ta = a.run(iters, cfg.s, cfg.sample_seed, iter0=0, fit_every=1)
    st = a.stats()
    assert st["host_syncs"] <= 1, st["host_syncs"]
    tb = []
    D = len(T.dims)
    for t in range(iters):
        for k in range(D):
            b.sample(k, cfg.s, cfg.sample_seed, t * D + k)
            b.solve_mode(k)
        tb.append(b.fit())
    assert np.array_equal(np.asarray(ta), np.asarray(tb)), (ta, tb)
    for (Aa, la), (Ab, lb) in zip(_factors(a), _factors(b)):
        assert np.array_equal(Aa.view(np.uint64), Ab.view(np.uint64)) and np.array_equal(la, lb)
    for m in range(D):
        assert np.array_equal(a.get_ptilde(m), b.get_ptilde(m))


def test_run_recovers_aborted_steps_with_the_host_sampler():
    """tau = 1e-6 < 1/s makes |DetSet| > s in every step (AMB-6 truncation, a
    host-path branch): every asynchronous step aborts and is redone by the
    host sampler; the run still equals the oracle's steps (lockstep on the
    first iteration) and the step-by-step GPU sequence."""
    need_gpu()
    from paper_2006_16438_b200 import Cparls
    T = synth.make("C1")
    cfg = T.cfg
    a = Cparls(T.dims, T.coords.cuda(), T.vals.cuda(), cfg.rank, tau=1e-6)
    b = Cparls(T.dims, T.coords.cuda(), T.vals.cuda(), cfg.rank, tau=1e-6)
    ta = a.run(2, cfg.s, 9, iter0=0, fit_every=1)
    tb = []
    for t in range(2):
        for k in range(3):
            info = b.sample(k, cfg.s, 9, t * 3 + k)
            assert info.s_det == cfg.s and info.s_rnd == 0
            b.solve_mode(k)
        tb.append(b.fit())
    assert np.array_equal(np.asarray(ta), np.asarray(tb)), (ta, tb)
    for (Aa, _), (Ab, _) in zip(_factors(a), _factors(b)):
        assert np.array_equal(Aa.view(np.uint64), Ab.view(np.uint64))
    # the truncated steps against the oracle
    o = oracle.Oracle(T.dims, T.coords.to(torch.int64).numpy(), T.vals.numpy(), cfg.rank)
    g = Cparls(T.dims, T.coords.cuda(), T.vals.cuda(), cfg.rank, tau=1e-6)
    for k in range(3):
        for m in range(3):
            o.set_factor(m, g.get_factor(m)[0])
            o.set_ptilde(m, g.get_ptilde(m))
        _step_lockstep(g, o, k, cfg.s, 1e-6, 9, k)


# ---------------------------------------------------------------- hot-row RHS
@pytest.mark.parametrize("name,hot", [("C1", -1), ("C1", 7), ("C2", -1), ("C2", 100), ("C3", -1)])
def test_hot_row_rhs_is_bit_identical(name, hot):
    """The fixed-point RHS with the hot rows summed per CTA in shared memory
    (rhs.cuh k_rhs_hot; two 32-bit words with exact carries) gives the same
    int64 sums as the plain L2 reductions, so the run's factors, p~ and fit
    trace are bit-identical with and without it.  hot = -1: automatic (every
    row hot on C1 and C2's small modes: slot = row); 7 / 100: a capped hot set
    (hot_slot table, hot and cold entries mixed in every warp)."""
    need_gpu()
    from paper_2006_16438_b200 import Cparls
    T = synth.make(name) if name == "C1" else synth.make(name, device="cuda")
    cfg = T.cfg
    a = Cparls(T.dims, T.coords.cuda(), T.vals.cuda(), cfg.rank, rhs_hot_rows=hot)
    b = Cparls(T.dims, T.coords.cuda(), T.vals.cuda(), cfg.rank, rhs_hot_rows=0)
    sa, sb = a.stats(), b.stats()
    D = len(T.dims)
    assert all(n == 0 for n in sb["rhs_hot_rows"])
    used = [n for n in sa["rhs_hot_rows"][:D]]
    assert any(n > 0 for n in used), sa["rhs_hot_rows"]
    if hot > 0:
        assert all(n == min(hot, T.dims[m]) for m, n in enumerate(used)), used
    for m, n in enumerate(used):
        if n == T.dims[m]:
            assert sa["rhs_hot_share"][m] == 1.0
        elif n > 0:
            assert 0.0 < sa["rhs_hot_share"][m] < 1.0
    del T
    torch.cuda.empty_cache()
    ta = a.run(2, cfg.s, cfg.sample_seed, iter0=0, fit_every=1)
    tb = b.run(2, cfg.s, cfg.sample_seed, iter0=0, fit_every=1)
    assert np.array_equal(np.asarray(ta), np.asarray(tb)), (ta, tb)
    for (Aa, la), (Ab, lb) in zip(_factors(a), _factors(b)):
        assert np.array_equal(Aa.view(np.uint64), Ab.view(np.uint64)) and np.array_equal(la, lb)
    for m in range(D):
        assert np.array_equal(a.get_ptilde(m), b.get_ptilde(m))


# ---------------------------------------------------------------- short modes (n_k < r)
@pytest.mark.parametrize("dup", [False, True])
def test_leverage_short_mode(dup):
    """A mode with fewer rows than r (C2's 24-row mode at r = 25).  Linearly
    independent rows: the hat matrix is the identity, l_i = 1 and the kept
    rank is n_k (kernels.cuh short_full_row_rank, AMB-11: the eigen cutoff of
    A^T A keeps exactly the n_k eigenvalues it shares with A A^T).  Two equal
    rows: the eigen path.  Both against the oracle's eigen pseudo-inverse."""
    need_gpu()
    from paper_2006_16438_b200 import Cparls
    dims = (7, 30, 40)
    r = 9
    coords, vals = _tiny_tensor(dims, 3000, 5)
    g = _ctx(dims, coords, vals, r)
    rng = np.random.default_rng(11)
    A = rng.uniform(0.1, 1.0, (dims[0], r))
    if dup:
        A[3] = A[1]
    g.set_factor(0, A)
    ell, rank = g.leverage(0)
    ref, rref = oracle.leverage(A)
    assert rank == rref == (dims[0] - 1 if dup else dims[0])
    if not dup:
        assert np.all(ell == 1.0)
    kappa = kept_kappa(A.T @ A)
    tol = 1e-12 * max(1.0, kappa / 1e3)
    err = np.abs(ell - ref) / np.maximum(np.abs(ref), r / A.shape[0])
    assert err.max() <= tol, (err.max(), kappa)
    # p~ = l / rank feeds the sampler: one lockstep step of the short mode's
    # neighbour (it samples mode 0's rows) against the oracle
    pt = g.get_ptilde(0)
    assert np.abs(pt - ref / rref).max() <= tol * max(1.0, (ref / rref).max())
    o = oracle.Oracle(dims, coords, vals, r)
    for m in range(3):
        o.set_factor(m, g.get_factor(m)[0])
        o.set_ptilde(m, g.get_ptilde(m))
    _step_lockstep(g, o, 1, 256, -1.0, 3, 0)


@pytest.mark.parametrize("name", ["C2", "C3"])
def test_row_degrees_from_run_boundaries(name):
    """The single-sort build takes each mode's row degrees from the run
    boundaries of the copy whose slowest key mode it is (k_slow_bounds, no
    atomics); the RHS hot rows are the top-H rows by those degrees.  With
    H = 100 forced, the share of nonzeros the library reports for every mode
    equals the top-100 share of torch.bincount of that mode's coordinates."""
    need_gpu()
    from paper_2006_16438_b200 import Cparls
    T = synth.make(name, device="cuda")
    cfg = T.cfg
    g = Cparls(T.dims, T.coords, T.vals, cfg.rank, rhs_hot_rows=100)
    st = g.stats()
    nnz = T.coords.shape[0]
    for m, n in enumerate(T.dims):
        deg = torch.bincount(T.coords[:, m].long(), minlength=n)
        H = min(100, n)
        assert st["rhs_hot_rows"][m] == H
        if H == n:
            assert st["rhs_hot_share"][m] == 1.0
        else:
            top = int(torch.topk(deg, H).values.sum())
            assert st["rhs_hot_share"][m] == top / nnz, (m, st["rhs_hot_share"][m], top / nnz)
