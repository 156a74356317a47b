"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs.  Bars (BASELINE.json north_star): sampled indices, dedup
counts, s_det and fiber matches bit-exact given the same p~ bits, seed and
step; leverage <= 1e-12 relative; per-mode solution <= 1e-9 relative
Frobenius on the same sample set; fit <= 1e-8 absolute."""
import math

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu


def need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def make_ctx(T, rank, tau=-1.0, init_seed=2, device="cuda", rhs_path=0):
    from paper_2006_16438_b200 import Cparls
    coords = T.coords.to(device) if device else T.coords.numpy()
    vals = T.vals.to(device) if device else T.vals.numpy()
    return Cparls(T.dims, coords, vals, rank, tau=tau, init_seed=init_seed, rhs_path=rhs_path)


def make_oracle(T, rank):
    return oracle.Oracle(T.dims, T.coords.to(torch.int64).numpy(), T.vals.to(torch.float64).numpy(), rank)


def sync_oracle_from_gpu(g, o):
    for m in range(g.D):
        A, lam = g.get_factor(m)
        o.set_factor(m, A)
        o.set_ptilde(m, g.get_ptilde(m))


def assert_leverage_close(g, o, m):
    """GPU p~ (computed inside the solve from the normalized factor) vs the
    oracle's leverage of the exported factor: |dl| <= 1e-12 max(l, r/n) * kappa/1e3."""
    A, _ = g.get_factor(m)
    ell_ref, rank_ref = oracle.leverage(A)
    pt = g.get_ptilde(m)
    ell_gpu = pt * rank_ref
    n, r = A.shape
    kappa = kept_kappa(A.T @ A)
    tol = 1e-12 * max(1.0, kappa / 1e3)   # scale by kappa/1e3 above 1e3
    scale = np.maximum(np.abs(ell_ref), r / n)
    err = np.abs(ell_gpu - ell_ref) / scale
    assert err.max() <= tol, (m, err.max(), kappa)


def kept_kappa(G):
    """Condition number over the eigenvalues the pseudo-inverse keeps (AMB-11)."""
    ev = np.linalg.eigvalsh(G)
    r = len(ev)
    if ev[-1] <= 0:
        return 1.0
    keep = ev[ev > r * np.finfo(float).eps * ev[-1]]
    return keep[-1] / keep[0]


SOLVE_LOG = []


def solve_tol(G, tag=""):
    """North-star bar: 1e-9 relative Frobenius on the same sample set.  kappa
    of the sampled Gram (over the kept spectrum, AMB-11) is logged with every
    case in SOLVE_LOG / gpurun_out/solve_bars.jsonl (round 2: 226 cases, max
    kappa 4.9e4, max relative error 8.4e-13)."""
    SOLVE_LOG.append({"case": tag, "kappa": float(kept_kappa(G)), "bar": 1e-9})
    return 1e-9


def log_solve(rel):
    """Attach the measured relative error to the last logged case and append
    it to gpurun_out/solve_bars.jsonl (when that directory exists)."""
    import json
    import os
    if SOLVE_LOG:
        SOLVE_LOG[-1]["rel_err"] = float(rel)
        d = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")
        if os.path.isdir(d):
            with open(os.path.join(d, "solve_bars.jsonl"), "a") as f:
                f.write(json.dumps(SOLVE_LOG[-1]) + "\n")


def compare_sample(g, o):
    a, b = g.get_sample(), o.get_sample()
    assert len(a["keys"]) == len(b["keys"])
    assert (a["keys"] == b["keys"]).all()
    assert (a["counts"] == b["counts"]).all()
    assert (a["is_det"] == b["is_det"]).all()
    assert (a["p"] == b["p"]).all()               # same canonical product bits
    np.testing.assert_allclose(a["w2"], b["w2"], rtol=1e-14, atol=0)
    la, oa, va = canonical_fibers(*g.get_fibers())
    lb, ob, vb = canonical_fibers(*o.get_fibers())
    assert (la == lb).all() and (oa == ob).all() and (va == vb).all()
    return a


def canonical_fibers(lens, out, val):
    """Entries of each fiber ordered by (row, value): duplicate coordinates
    (equal key and row) may come in any order; everything else is unique."""
    fid = np.repeat(np.arange(len(lens)), lens)
    o = np.lexsort((val, out, fid))
    return lens, out[o], val[o]


def lockstep(T, rank, iters, s, seed, tau=-1.0, check_fit=True, rhs_path=0):
    need_gpu()
    g = make_ctx(T, rank, tau=tau, rhs_path=rhs_path)
    o = make_oracle(T, rank)
    D = len(T.dims)
    stats = []
    for t in range(iters):
        for k in range(D):
            sync_oracle_from_gpu(g, o)
            step = t * D + k
            gi = g.sample(k, s, seed, step)
            oi = o.sample(k, s, tau, seed, step)
            assert (gi.s_det, gi.s_rnd, gi.s_bar, gi.attempts, gi.skipped_random) == \
                   (oi.s_det, oi.s_rnd, oi.s_bar, oi.attempts, oi.skipped_random)
            assert abs(gi.p_det - oi.p_det) <= 1e-14 * max(1.0, oi.p_det)
            compare_sample(g, o)
            gs = g.solve_mode(k)
            os_ = o.solve_mode(k)
            assert gs.matched_nnz == os_.matched_nnz
            assert gs.touched_rows == os_.touched_rows
            assert gs.rank_used == os_.rank_used
            Gg, Bg = g.last_solve(k)
            Go, Mo, Bo = o.last_solve(k)
            np.testing.assert_allclose(Gg, Go, rtol=1e-11, atol=1e-13 * max(1.0, np.abs(Go).max()))
            nb = np.linalg.norm(Bo)
            if nb > 0:
                tol = solve_tol(Go, f"{getattr(T, 'cfg', None) and T.cfg.name} dims={tuple(T.dims)} r={rank} t={t} k={k}")
                rel = np.linalg.norm(Bg - Bo) / nb
                log_solve(rel)
                assert rel <= tol, (t, k, rel, tol)
            else:
                assert np.linalg.norm(Bg) == 0
            Ag, lg = g.get_factor(k)
            Ao, lo = o.get_factor(k)
            np.testing.assert_allclose(lg, lo, rtol=1e-9, atol=1e-300)
            assert_leverage_close(g, o, k)
            stats.append((gi.s_det, gi.s_bar, gs.matched_nnz))
        if check_fit:
            fg, fo = g.fit(), o.fit()
            assert abs(fg - fo) <= 1e-8, (t, fg, fo)
    return g, o, stats


def test_c1_lockstep_20_iterations():
    T = synth.make("C1")
    cfg = T.cfg
    lockstep(T, cfg.rank, cfg.iters, cfg.s, cfg.sample_seed)


@pytest.mark.parametrize("rhs_path", [1, 3])
def test_c1_lockstep_rhs_paths(rhs_path):
    """Both RHS implementations (fixed-point int64 reductions into M, fp64
    reductions into M) against the oracle."""
    T = synth.make("C1")
    cfg = T.cfg
    lockstep(T, cfg.rank, 6, cfg.s, cfg.sample_seed, rhs_path=rhs_path)


def test_c2_lockstep_fp64_rhs_path():
    T = synth.make("C2", device="cuda")
    T = synth.Tensor(T.cfg, T.dims, T.coords.cpu(), T.vals.cpu())
    lockstep(T, 25, 1, 1 << 17, 3, rhs_path=3)


def test_rhs_paths_agree_f32_values():
    """fp32-valued tensor (the C4/C5 storage): the fixed-point and the fp64
    reduction paths give the same B to the quantisation bound (<= 1e-11
    relative), over a few free-running steps; the removed rhs_path 2 is
    rejected."""
    need_gpu()
    cfg = synth.scaled("C2", 300_000)
    T = synth.make(cfg, device="cuda")
    from paper_2006_16438_b200 import Cparls, CparlsError
    from paper_2006_16438_b200 import cparls as cp
    with pytest.raises(CparlsError) as e:
        Cparls(T.dims, T.coords, T.vals.float(), 25, rhs_path=2)
    assert e.value.status == cp.EINVAL
    a = Cparls(T.dims, T.coords, T.vals.float(), 25, rhs_path=1)
    b = Cparls(T.dims, T.coords, T.vals.float(), 25, rhs_path=3)
    for t in range(2):
        for k in range(len(T.dims)):
            ia, ib = a.sample(k, 4096, 5, 4 * t + k), b.sample(k, 4096, 5, 4 * t + k)
            assert ia.s_bar == ib.s_bar
            sa, sb = a.solve_mode(k), b.solve_mode(k)
            assert (sa.matched_nnz, sa.touched_rows) == (sb.matched_nnz, sb.touched_rows)
            _, Ba = a.last_solve(k)
            _, Bb = b.last_solve(k)
            assert np.linalg.norm(Ba - Bb) <= 1e-11 * np.linalg.norm(Ba), (t, k)
            # continue both from identical factors so the comparison stays per-step
            A, _ = a.get_factor(k)
            b.set_factor(k, A)
            b.set_ptilde(k, a.get_ptilde(k))


def test_c1_random_only_tau1():
    T = synth.make("C1")
    lockstep(T, 3, 3, 256, 7, tau=1.0)


def test_init_matches_synth_uniform_init():
    need_gpu()
    T = synth.make("C1")
    g = make_ctx(T, 3, init_seed=2)
    ref = synth.uniform_init(T.dims, 3, 2)
    for m in range(3):
        A, lam = g.get_factor(m)
        assert (A == ref[m].numpy()).all()
        assert (lam == 1).all()


def test_leverage_parity_random_factors():
    need_gpu()
    T = synth.make("C1")
    g = make_ctx(T, 3)
    rng = np.random.default_rng(0)
    for m in range(3):
        A = rng.standard_normal((T.dims[m], 3)) * [1.0, 10.0, 0.1]
        g.set_factor(m, A)
        ell, rank = g.leverage(m)
        ref, rref = oracle.leverage(A)
        assert rank == rref == 3
        assert np.abs(ell - ref).max() <= 1e-12 * max(1.0, 1.0)


def test_leverage_rank_deficient_fallback():
    need_gpu()
    T = synth.make("C1")
    from paper_2006_16438_b200 import Cparls
    g = Cparls(T.dims, T.coords.cuda(), T.vals.cuda(), 5)
    rng = np.random.default_rng(1)
    A = rng.standard_normal((T.dims[0], 3)) @ rng.standard_normal((3, 5))
    g.set_factor(0, A)
    ell, rank = g.leverage(0)
    ref, rref = oracle.leverage(A)
    assert rank == rref == 3
    # the leverage bar of SURVEY 8(c): 1e-12 * max(l, r/n), scaled by kappa/1e3
    # above kappa = 1e3 (kappa over the kept spectrum of A^T A)
    kappa = kept_kappa(A.T @ A)
    tol = 1e-12 * max(1.0, kappa / 1e3)
    err = np.abs(ell - ref) / np.maximum(np.abs(ref), 5 / A.shape[0])
    assert err.max() <= tol, (err.max(), kappa)


def test_c2_lockstep_2_iterations():
    T = synth.make("C2", device="cuda")
    T = synth.Tensor(T.cfg, T.dims, T.coords.cpu(), T.vals.cpu())
    lockstep(T, 25, 2, 1 << 17, 3)


def test_generator_cpu_cuda_identical():
    need_gpu()
    cfg = synth.scaled("C2", 200_000)
    a = synth.make(cfg, device="cpu")
    b = synth.make(cfg, device="cuda")
    assert torch.equal(a.coords, b.coords.cpu())
    assert torch.equal(a.vals, b.vals.cpu())


def test_full_inclusion_equals_exact_als_gpu():
    """PIN-9 through the GPU: tau = 0, s = N_k -> every row deterministic with
    w = 1, so B is the exact ALS update (oracle's own CP-ALS routine)."""
    need_gpu()
    dims = (5, 6, 4)
    rng = np.random.default_rng(3)
    lin = rng.choice(120, 70, replace=False)
    coords = np.stack(np.unravel_index(lin, dims, order="F"), 1).astype(np.int32)
    vals = rng.standard_normal(70)
    T = synth.Tensor(synth.CONFIGS["C1"], dims, torch.from_numpy(coords), torch.from_numpy(vals))
    g = make_ctx(T, 3, tau=0.0)
    for k in range(3):
        o = make_oracle(T, 3)
        sync_oracle_from_gpu(g, o)
        for m in range(3):
            o.set_factor(m, g.get_factor(m)[0])
        Nk = int(np.prod([n for m, n in enumerate(dims) if m != k]))
        info = g.sample(k, Nk, 1, k)
        assert info.s_det == Nk and info.s_bar == Nk
        g.solve_mode(k)
        _, Bg = g.last_solve(k)
        o.als_update(k)
        _, _, Bo = o.last_solve(k)
        assert np.linalg.norm(Bg - Bo) <= 1e-9 * np.linalg.norm(Bo)


def test_two_way_and_rank_edges():
    need_gpu()
    rng = np.random.default_rng(4)
    for dims, r in (((37, 53), 1), ((37, 53), 4), ((9, 11, 13), 64)):
        N = int(np.prod(dims))
        nnz = min(N, 400)
        lin = rng.choice(N, nnz, replace=False)
        coords = np.stack(np.unravel_index(lin, dims, order="F"), 1).astype(np.int32)
        vals = rng.standard_normal(nnz)
        T = synth.Tensor(synth.CONFIGS["C1"], dims, torch.from_numpy(coords), torch.from_numpy(vals))
        lockstep(T, r, 2, 64, 11)


def test_empty_tensor_and_errors():
    need_gpu()
    from paper_2006_16438_b200 import Cparls, CparlsError
    from paper_2006_16438_b200 import cparls as cp
    g = Cparls((4, 5, 6), np.zeros((0, 3), dtype=np.int32), np.zeros(0), 2)
    g.sample(0, 16, 1, 0)
    info = g.solve_mode(0)
    assert info.matched_nnz == 0
    with pytest.raises(CparlsError) as e:
        g.fit()
    assert e.value.status == cp.ENUMERIC
    with pytest.raises(CparlsError) as e:
        g.solve_mode(1)
    assert e.value.status == cp.ESTATE
    with pytest.raises(CparlsError) as e:
        g.sample(7, 16, 1, 0)
    assert e.value.status == cp.EINVAL
    with pytest.raises(CparlsError) as e:
        Cparls((4, 5, 6), np.array([[0, 5, 0]], dtype=np.int32), np.ones(1), 2)
    assert e.value.status == cp.ERANGE
    with pytest.raises(CparlsError) as e:
        Cparls((4, 5, 6), np.zeros((1, 3), dtype=np.int32), np.ones(1), 65)
    assert e.value.status == cp.EINVAL


def test_host_and_device_inputs_agree():
    need_gpu()
    T = synth.make("C1")
    a = make_ctx(T, 3, device="cuda")
    b = make_ctx(T, 3, device=None)
    ta = a.run(3, 256, 3, fit_every=1)
    tb = b.run(3, 256, 3, fit_every=1)
    np.testing.assert_allclose(ta, tb, rtol=0, atol=1e-12)


def test_planted_recovery_gpu():
    """Fully populated planted rank-3 C1 variant: CP-ARLS-LEV reaches fit >= 0.999."""
    need_gpu()
    T = synth.make("C1", dense_planted=True)
    g = make_ctx(T, 3)
    trace = g.run(60, 256, 3, fit_every=1)
    assert np.nanmax(trace) >= 0.999


def test_free_running_matches_oracle():
    need_gpu()
    T = synth.make("C1", dense_planted=True)
    g = make_ctx(T, 3)
    o = make_oracle(T, 3)
    for m in range(3):
        o.set_factor(m, g.get_factor(m)[0])
    tg = g.run(5, 256, 3, fit_every=1)
    to = o.run(5, 256, -1, 3, 1)
    np.testing.assert_allclose(tg, to, atol=1e-8)


# ---------------------------------------------------------------- estimated fit (N1)
@pytest.mark.parametrize("name,alpha", [("C1", 0.5), ("C2", 0.3)])
def test_fit_sample_and_estimate_parity(name, alpha):
    """The frozen stratified sample is bit-identical to the oracle's (same COO
    order, seed, alpha; AMB-32) and the estimate agrees (F^ <= 1e-12 rel, fit
    <= 1e-8) after a few lockstep-synced mode steps."""
    need_gpu()
    from paper_2006_16438_b200 import Cparls
    T = synth.make(name, device="cpu" if name == "C1" else "cuda")
    T = synth.Tensor(T.cfg, T.dims, T.coords.cpu(), T.vals.cpu())
    r = T.cfg.rank
    s_fit, seed = 20000, 1234567
    g = Cparls(T.dims, T.coords.cuda(), T.vals.cuda(), r, fit_samples=s_fit, fit_alpha=alpha, fit_seed=seed)
    o = make_oracle(T, r)
    nn, nz = o.fit_sample(s_fit, alpha, seed)
    gc, gx, gnz = g.get_fit_sample()
    oc, ox, onz = o.get_fit_sample()
    assert gc.shape == oc.shape and (gc == oc).all() and (gx == ox).all() and (gnz == onz).all()
    assert gnz.sum() == nn and (~gnz).sum() == nz
    D = len(T.dims)
    for t in range(2):
        for k in range(D):
            g.sample(k, T.cfg.s, 3, t * D + k)
            g.solve_mode(k)
        for m in range(D):
            o.set_factor(m, g.get_factor(m)[0])
        # the model's lambda lives with the last solved mode; the oracle takes
        # unit-column factors and lambda through set_factor of that mode
        A, lam = g.get_factor(D - 1)
        o.set_factor(D - 1, A * lam)
        fg, Fg = g.fit_estimate()
        fo, Fo = o.fit_estimate()
        # the model at the sample positions, from the oracle's factors
        m_o = np.array([np.prod([o.get_factor(q)[0][c[q]] for q in range(D)], axis=0).sum() for c in oc[:500]])
        np.testing.assert_allclose(g.fit_sample_model()[:500], m_o, rtol=1e-12, atol=1e-14 * np.abs(m_o).max())
        assert abs(Fg - Fo) <= 1e-12 * abs(Fo), (Fg, Fo)
        assert abs(fg - fo) <= 1e-8


def test_run_until_matches_oracle():
    """Alg. 3 with the stopping rule, free running on the planted C1 variant:
    same number of epochs and fit trace within 1e-8 (exact and estimated)."""
    need_gpu()
    from paper_2006_16438_b200 import Cparls
    T = synth.make("C1", dense_planted=True)
    init = synth.uniform_init(T.dims, 3, 2)
    for estimated in (False, True):
        g = Cparls(T.dims, T.coords.cuda(), T.vals.cuda(), 3, fit_samples=4096, fit_seed=5)
        o = make_oracle(T, 3)
        for m in range(3):
            o.set_factor(m, init[m].numpy())
        if estimated:
            o.fit_sample(4096, 0.5, 5)
        tg = g.run_until(256, 3, eta=5, pi=3, tol=1e-4, max_epochs=12, estimated=estimated)
        to = o.run_until(256, -1.0, 3, eta=5, pi=3, tol=1e-4, max_epochs=12, estimated=estimated)
        assert len(tg) == len(to) and len(tg) >= 3
        np.testing.assert_allclose(tg, to, atol=1e-8)


# ---------------------------------------------------------------- exact CP-ALS baseline (N2)
@pytest.mark.parametrize("name", ["C1", "C2"])
def test_als_update_parity(name):
    """One exact CP-ALS mode update per mode against the oracle's
    or_als_update from the same factors: V, B (<= 1e-9), lambda, leverage."""
    need_gpu()
    T = synth.make(name, device="cpu" if name == "C1" else "cuda")
    T = synth.Tensor(T.cfg, T.dims, T.coords.cpu(), T.vals.cpu())
    r = T.cfg.rank
    g = make_ctx(T, r)
    o = make_oracle(T, r)
    for t in range(2):
        for k in range(len(T.dims)):
            sync_oracle_from_gpu(g, o)
            g.als_update(k)
            o.als_update(k)
            Gg, Bg = g.last_solve(k)
            Go, _, Bo = o.last_solve(k)
            np.testing.assert_allclose(Gg, Go, rtol=1e-12, atol=1e-14 * np.abs(Go).max())
            tol = solve_tol(Go, f"als {name} t={t} k={k}")
            rel = np.linalg.norm(Bg - Bo) / np.linalg.norm(Bo)
            log_solve(rel)
            assert rel <= tol, (t, k, rel, tol)
            np.testing.assert_allclose(g.get_factor(k)[1], o.get_factor(k)[1], rtol=1e-9)
            assert_leverage_close(g, o, k)


def test_run_als_trace_and_monotone():
    """CP-ALS free running on the planted C1 variant: the exact fit trace
    matches the oracle's ALS to 1e-8 and never decreases (ALS property)."""
    need_gpu()
    T = synth.make("C1", dense_planted=True)
    g = make_ctx(T, 3)
    o = make_oracle(T, 3)
    init = synth.uniform_init(T.dims, 3, 2)
    for m in range(3):
        o.set_factor(m, init[m].numpy())
    tg = g.run_als(12, fit_every=1)
    to = []
    for t in range(12):
        for k in range(3):
            o.als_update(k)
        to.append(o.fit())
    np.testing.assert_allclose(tg, to, atol=1e-8)
    assert (np.diff(tg) >= -1e-10).all()


# ---------------------------------------------------------------- RRF initialization (N4)
@pytest.mark.parametrize("name", ["C1", "C2"])
def test_rrf_init_parity(name):
    """cparls_init_rrf vs the oracle's RRF (AMB-34): every factor to 1e-12
    (Box-Muller's libm differs by ulps between host and device), lambda = 1,
    and the leverage refresh of the new factors; then one lockstep iteration."""
    need_gpu()
    T = synth.make(name, device="cpu" if name == "C1" else "cuda")
    T = synth.Tensor(T.cfg, T.dims, T.coords.cpu(), T.vals.cpu())
    r = T.cfg.rank
    g = make_ctx(T, r)
    o = make_oracle(T, r)
    g.init_rrf(1000, 42)
    o.init_rrf(1000, 42)
    for k in range(len(T.dims)):
        Ag, lg = g.get_factor(k)
        Ao, lo = o.get_factor(k)
        np.testing.assert_allclose(Ag, Ao, rtol=1e-12, atol=1e-12 * np.abs(Ao).max())
        assert (lg == 1).all()
        assert_leverage_close(g, o, k)


def test_c2_hybrid_concentrated_leverage_lockstep():
    """Regression: an exact-ALS (rank 10) solution concentrates the leverage, so
    the DIDX candidate list of a small mode's neighbour exceeds that small
    mode's length (candidate slot j holds the j-th OTHER mode: it must take
    max n_m).  Bit-exact sample vs the oracle at s = 2^17, hybrid."""
    need_gpu()
    T = synth.make("C2", device="cuda")
    from paper_2006_16438_b200 import Cparls
    r = 10
    g = Cparls(T.dims, T.coords, T.vals, r)
    g.run_als(5, fit_every=0)
    A = [g.get_factor(m)[0] for m in range(4)]
    A[3] = A[3] * g.get_factor(0)[1]
    o = oracle.Oracle(T.dims, T.coords.cpu().numpy().astype(np.int64), T.vals.cpu().numpy(), r)
    for k in range(4):
        for m in range(4):
            g.set_factor(m, A[m])
            o.set_factor(m, A[m])
            o.set_ptilde(m, g.get_ptilde(m))
        gi = g.sample(k, 1 << 17, 1000, k)
        oi = o.sample(k, 1 << 17, -1.0, 1000, k)
        assert (gi.s_det, gi.s_bar, gi.attempts) == (oi.s_det, oi.s_bar, oi.attempts)
        assert oi.s_det > 0
        a, b = g.get_sample(), o.get_sample()
        assert (a["keys"] == b["keys"]).all() and (a["counts"] == b["counts"]).all()


@pytest.mark.parametrize("rank", [10, 25, 40])
def test_rhs_fixed_point_deterministic_and_close(rank):
    """AMB-35: the fixed-point RHS (rhs_path 1) is bit-reproducible run to run,
    and agrees with the fp64-reduction path (rhs_path 3) to the quantisation
    bound (<= 1e-11 relative Frobenius on B; HI lanes covered by rank 40)."""
    need_gpu()
    T = synth.make("C2", device="cuda")
    from paper_2006_16438_b200 import Cparls
    gs = {p: Cparls(T.dims, T.coords, T.vals, rank, rhs_path=p, init_seed=5) for p in (1, 3)}
    A = [gs[1].get_factor(m)[0] for m in range(4)]
    for k in range(4):
        out = {}
        for p, g in gs.items():
            Bs = []
            for rep in range(2):
                for m in range(4):
                    g.set_factor(m, A[m])
                g.sample(k, 1 << 16, 77, k)
                g.solve_mode(k)
                Bs.append(g.last_solve(k)[1].copy())
            out[p] = Bs
        assert np.array_equal(out[1][0].view(np.uint64), out[1][1].view(np.uint64)), k
        nb = np.linalg.norm(out[3][0])
        rel = np.linalg.norm(out[1][0] - out[3][0]) / nb
        assert rel <= 1e-11, (k, rel)
    for g in gs.values():
        g.close()


@pytest.mark.parametrize("scale", [1.0, 1e150, 1e-290])
def test_rhs_fixed_point_duplicates_and_range(scale):
    """AMB-35 bound with duplicate coordinates (dupmax = 4) and value ranges
    that keep the fixed-point path (1, 1e150) or push 2^e_c out of range so
    the step falls back to fp64 reductions (1e-290): lockstep vs the oracle."""
    import types
    rng = np.random.default_rng(11)
    dims = (30, 20, 25)
    base = np.stack([rng.integers(0, n, 300) for n in dims], 1)
    reps = rng.integers(1, 5, len(base))
    reps[0] = 4
    coords = np.repeat(base, reps, axis=0)
    vals = rng.uniform(0.5, 2.0, len(coords)) * scale
    perm = rng.permutation(len(coords))
    T = types.SimpleNamespace(dims=dims, coords=torch.from_numpy(coords[perm].astype(np.int64)),
                              vals=torch.from_numpy(vals[perm]))
    lockstep(T, 4, 2, 64, 5, check_fit=(scale == 1.0), rhs_path=1)


@pytest.mark.parametrize("dims,r", [((5, 6, 7, 4, 3), 3), ((3, 4, 3, 5, 2, 4), 2), ((20, 30, 25), 32),
                                    ((20, 30, 25), 33)])
def test_higher_order_and_rank_boundaries(dims, r):
    """D = 5, 6 (DIDX over 4-5 levels, the thread-per-nonzero fit k_fit_thread)
    and ranks at the 32-lane boundary of k_rhs (r = 32 one lane pass, r = 33
    the second pass, RMAX 32 -> 64 row kernels): lockstep vs the oracle."""
    need_gpu()
    rng = np.random.default_rng(sum(dims) + r)
    N = int(np.prod(dims))
    nnz = min(N, 500)
    lin = rng.choice(N, nnz, replace=False)
    coords = np.stack(np.unravel_index(lin, dims, order="F"), 1).astype(np.int32)
    vals = rng.uniform(0.5, 2.0, nnz)
    T = synth.Tensor(synth.CONFIGS["C1"], dims, torch.from_numpy(coords), torch.from_numpy(vals))
    lockstep(T, r, 2, 96, 13)


@pytest.mark.parametrize("dims", [(4194301, 2097151, 2097143), (4194319, 2097169, 2097157)])
def test_index_build_at_the_64_bit_composite_boundary(dims):
    """The single-sort build (composite key key*n_k + out, prod n_m < 2^64) at
    prod n_m just below 2^64 (cbits = 64) and the two-sort fallback just above
    it: fibers, samples, solves and fit in lockstep with the oracle.  Rows of
    the slow key modes come from small hot sets so fibers hold several
    entries (row degrees from run boundaries, duplicates merged)."""
    need_gpu()
    assert (int(np.prod(dims, dtype=object)) < 2 ** 64) == (dims[0] < 2 ** 22)
    rng = np.random.default_rng(dims[0])
    nnz = 3000
    hot = [rng.choice(n, 40, replace=False) for n in dims]
    coords = np.stack([rng.integers(0, dims[0], nnz)] +
                      [hot[m][rng.integers(0, 40, nnz)] for m in (1, 2)], 1)
    coords = np.unique(coords, axis=0).astype(np.int32)
    vals = rng.uniform(0.5, 2.0, len(coords))
    T = synth.Tensor(synth.CONFIGS["C1"], dims, torch.from_numpy(coords), torch.from_numpy(vals))
    lockstep(T, 3, 1, 128, 17)
