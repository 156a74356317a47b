"""Parity at the benchmark's full size (BASELINE.json configs[3] = C4: 4.8M x 1.8M
x 1.8M, 1.74B nonzeros, r = 25, s = 2^17), in the launch configuration bench.py
times (default options, after bench.py's 3 warm-up iterations).

The CPU oracle cannot hold the whole C4 tensor, so every check here either
gives the oracle exactly the data the checked step depends on, or checks a
property that holds at any size:

* sampling (DIDX/SIDX/CIDX) depends on the p~ vectors only: an oracle with C4's
  dims and no nonzeros, given the GPU's p~ bits (the lockstep protocol of
  test_gpu_parity.py), must draw the identical sample -- bit-exact keys,
  counts, det flags and w^2 to 1e-14;
* a mode step reads only the nonzeros of the sampled fibers: torch selects
  them from the COO by brute force (isin over the canonical keys -- code that
  shares nothing with the CUDA path), the oracle is built on that subset and
  given the GPU's factors, and then its fibers, matched-nonzero count, touched
  rows, sampled Gram and B must match the GPU exactly as in the small cases;
* leverage of every row of the solved factor against oracle.leverage;
* the exact fit against its definition evaluated by torch in fp64 over all
  1.74B nonzeros (chunked), to 1e-8 absolute.
"""
import math

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

SEED = 3
FIT_SAMPLES = 1 << 27     # the paper's s_fit for Amazon
FIT_SEED = 17


def need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


@pytest.fixture(scope="module")
def c4():
    need_gpu()
    from paper_2006_16438_b200 import Cparls
    cfg = synth.CONFIGS["C4"]
    dev = torch.device("cuda", 0)
    T = synth.make(cfg, device=dev, index_dtype=torch.int32)
    torch.cuda.empty_cache()
    g = Cparls(cfg.dims, T.coords, T.vals, cfg.rank, tau=-1.0, init_seed=cfg.init_seed,
               fit_samples=FIT_SAMPLES, fit_alpha=0.5, fit_seed=FIT_SEED)
    g.run(3, cfg.s, SEED, iter0=0, fit_every=0)        # bench.py's warm-up
    yield cfg, T, g
    g.close()
    del T
    torch.cuda.empty_cache()


def canonical_keys(coords, dims, k, lo, hi):
    """eq:bijection (AMB-1): other modes ascending, first fastest, int64."""
    key = torch.zeros(hi - lo, dtype=torch.int64, device=coords.device)
    mult = 1
    for m in range(len(dims)):
        if m == k:
            continue
        key += coords[lo:hi, m].to(torch.int64) * mult
        mult *= dims[m]
    return key


def fiber_subset(T, k, skeys):
    """All nonzeros whose other-mode coordinates form a sampled key (brute force)."""
    dims = T.dims
    sk = torch.from_numpy(skeys.astype(np.int64)).to(T.coords.device)
    sk, _ = torch.sort(sk)
    parts_c, parts_v = [], []
    n = T.coords.shape[0]
    step = 1 << 27
    for lo in range(0, n, step):
        hi = min(n, lo + step)
        key = canonical_keys(T.coords, dims, k, lo, hi)
        pos = torch.searchsorted(sk, key).clamp_(max=sk.numel() - 1)
        hit = sk[pos] == key
        idx = torch.nonzero(hit).squeeze(1) + lo
        parts_c.append(T.coords[idx].to(torch.int64).cpu())
        parts_v.append(T.vals[idx].to(torch.float64).cpu())
    return torch.cat(parts_c).numpy(), torch.cat(parts_v).numpy()


def test_c4_sampling_bit_exact_all_modes(c4):
    cfg, T, g = c4
    o = oracle.Oracle(cfg.dims, np.zeros((0, 3), dtype=np.int64), np.zeros(0), cfg.rank)
    for m in range(3):
        o.set_ptilde(m, g.get_ptilde(m))
    for k in range(3):
        step = 3 * 3 + k
        gi = g.sample(k, cfg.s, SEED, step)
        oi = o.sample(k, cfg.s, -1.0, SEED, step)
        assert (gi.s_det, gi.s_rnd, gi.s_bar, gi.attempts, gi.skipped_random) == \
               (oi.s_det, oi.s_rnd, oi.s_bar, oi.attempts, oi.skipped_random)
        a, b = g.get_sample(), o.get_sample()
        assert (a["keys"] == b["keys"]).all()
        assert (a["counts"] == b["counts"]).all()
        assert (a["is_det"] == b["is_det"]).all()
        assert (a["p"] == b["p"]).all()
        np.testing.assert_allclose(a["w2"], b["w2"], rtol=1e-14, atol=0)
    o.close()


@pytest.mark.parametrize("k", [0, 1, 2])
def test_c4_mode_step_against_oracle_on_the_sampled_fibers(c4, k):
    cfg, T, g = c4
    step = 3 * 3 + 3 + k      # the next steps of the sequence (after the sampling test's steps)
    gi = g.sample(k, cfg.s, SEED, step)
    smp = g.get_sample()
    coords, vals = fiber_subset(T, k, smp["keys"])
    o = oracle.Oracle(cfg.dims, coords, vals, cfg.rank)
    for m in range(3):
        A, _ = g.get_factor(m)
        o.set_factor(m, A)
        o.set_ptilde(m, g.get_ptilde(m))
    oi = o.sample(k, cfg.s, -1.0, SEED, step)
    assert (gi.s_det, gi.s_bar, gi.attempts) == (oi.s_det, oi.s_bar, oi.attempts)
    b = o.get_sample()
    assert (smp["keys"] == b["keys"]).all() and (smp["counts"] == b["counts"]).all()
    la, oa, va = g.get_fibers()
    lb, ob, vb = o.get_fibers()
    assert (la == lb).all() and (oa == ob).all() and (va == vb).all()
    gs = g.solve_mode(k)
    os_ = o.solve_mode(k)
    assert gs.matched_nnz == os_.matched_nnz == int(la.sum())
    assert gs.touched_rows == os_.touched_rows
    assert gs.rank_used == os_.rank_used
    Gg, Bg = g.last_solve(k)
    Go, _, Bo = o.last_solve(k)
    np.testing.assert_allclose(Gg, Go, rtol=1e-11, atol=1e-13 * np.abs(Go).max())
    from test_gpu_parity import log_solve, solve_tol
    tol = solve_tol(Go, f"C4 full size k={k}")
    rel = np.linalg.norm(Bg - Bo) / np.linalg.norm(Bo)
    log_solve(rel)
    assert rel <= tol, (rel, tol)
    Ag, lg = g.get_factor(k)
    Ao, lo = o.get_factor(k)
    np.testing.assert_allclose(lg, lo, rtol=1e-9, atol=1e-300)
    # leverage of the solved factor, every row
    ell_ref, rank_ref = oracle.leverage(Ag)
    ell = g.get_ptilde(k) * rank_ref
    n, r = Ag.shape
    err = np.abs(ell - ell_ref) / np.maximum(np.abs(ell_ref), r / n)
    assert err.max() <= 1e-12 * 10, err.max()   # kappa-scaled bar; kappa << 1e4 here
    o.close()


def test_c4_exact_fit_against_its_definition(c4):
    """fit = 1 - ||X - M|| / ||X|| (eq:fit), <X, M> and ||X||^2 summed by torch
    in fp64 over all nonzeros, ||M||^2 = lambda^T (*_m A_m^T A_m) lambda."""
    cfg, T, g = c4
    fg = g.fit()
    dev = T.coords.device
    A = []
    for m in range(3):
        Am, lam = g.get_factor(m)        # lam = the model's lambda (AMB-31)
        A.append(torch.from_numpy(Am).to(dev))
    lam_model = torch.from_numpy(lam).to(dev)
    inner = torch.zeros((), dtype=torch.float64, device=dev)
    nx2 = torch.zeros((), dtype=torch.float64, device=dev)
    n = T.coords.shape[0]
    step = 1 << 24
    for lo in range(0, n, step):
        hi = min(n, lo + step)
        c = T.coords[lo:hi].to(torch.int64)
        x = T.vals[lo:hi].to(torch.float64)
        h = A[0][c[:, 0]] * A[1][c[:, 1]] * A[2][c[:, 2]]
        inner += (x * (h @ lam_model)).sum()
        nx2 += (x * x).sum()
    V = torch.ones((cfg.rank, cfg.rank), dtype=torch.float64, device=dev)
    for m in range(3):
        V = V * (A[m].T @ A[m])
    nm2 = lam_model @ V @ lam_model
    resid2 = torch.clamp(nx2 - 2 * inner + nm2, min=0.0)
    fref = float(1.0 - torch.sqrt(resid2) / torch.sqrt(nx2))
    assert abs(fg - fref) <= 1e-8, (fg, fref)


def test_c4_fit_sample_and_estimate(c4):
    """N1 at full size: the frozen stratified sample re-derived from its
    definition (AMB-32) with the generator's independent Philox on the GPU
    (nonzero stratum: COO entries mulhi(R, nnz); zero stratum: the proposed
    cells in attempt order, every skipped proposal a nonzero and a random
    subset of the accepted ones checked absent by brute force), and F^ against
    its definition evaluated by torch in fp64 over the sample."""
    from synth import philox4x32_10
    cfg, T, g = c4
    dev = T.coords.device
    gc, gx, gnz = g.get_fit_sample()
    nn = (FIT_SAMPLES + 1) // 2
    nz = FIT_SAMPLES // 2
    assert gnz.sum() == nn and (~gnz).sum() == nz
    nnz = T.coords.shape[0]

    def words(ctr, lane):
        c0 = (ctr & 0xFFFFFFFF).to(torch.int64)
        c1 = (ctr >> 32).to(torch.int64)
        return philox4x32_10(c0, c1, 0x46495400, lane, FIT_SEED & 0xFFFFFFFF, FIT_SEED >> 32)

    def mulhi(lo32, hi32, n):
        # floor(((hi << 32) | lo) * n / 2^64) with 64-bit limbs (n < 2^32)
        a = lo32 * n
        b = hi32 * n + (a >> 32)
        return b >> 32

    gcd = torch.from_numpy(gc).to(dev)
    step = 1 << 24
    for lo in range(0, nn, step):
        i = torch.arange(lo, min(nn, lo + step), device=dev, dtype=torch.int64)
        w = words(i, 0)
        e = mulhi(w[0], w[1], nnz)
        assert torch.equal(T.coords[e].to(torch.int64), gcd[lo:lo + len(i)])
        assert torch.equal(T.vals[e].to(torch.float64), torch.from_numpy(gx[lo:lo + len(i)]).to(dev))
    # zero stratum: proposals in attempt order
    a = torch.arange(0, nz, device=dev, dtype=torch.int64)
    w1, w2 = words(a, 1), words(a, 2)
    cells = torch.stack([mulhi(w1[0], w1[1], cfg.dims[0]), mulhi(w1[2], w1[3], cfg.dims[1]),
                         mulhi(w2[0], w2[1], cfg.dims[2])], 1)
    zs = gcd[nn:]
    # density ~1e-10: with this seed no proposal among the first n_z hits a
    # nonzero, so the zero stratum is exactly the first n_z proposals
    assert torch.equal(cells[:nz], zs)
    for cell in zs[torch.randint(0, nz, (64,), device=dev, generator=torch.Generator(device=dev).manual_seed(0))]:
        hit = ((T.coords[:, 0] == cell[0]) & (T.coords[:, 1] == cell[1]) & (T.coords[:, 2] == cell[2])).any()
        assert not bool(hit)
    # F^ from its definition over the (validated) sample
    fg, Fg = g.fit_estimate()
    A = [torch.from_numpy(g.get_factor(m)[0]).to(dev) for m in range(3)]
    lam = torch.from_numpy(g.get_factor(0)[1]).to(dev)
    x = torch.from_numpy(gx).to(dev)
    m = torch.zeros(len(gx), dtype=torch.float64, device=dev)
    am = torch.zeros(len(gx), dtype=torch.float64, device=dev)   # sum_c |lambda_c prod_m A_m(i_m, c)|
    for lo in range(0, len(gx), step):
        c = gcd[lo:lo + step]
        h = A[0][c[:, 0]] * A[1][c[:, 1]] * A[2][c[:, 2]]
        m[lo:lo + step] = h @ lam
        am[lo:lo + step] = h.abs() @ lam.abs()
    f64 = dict(dtype=torch.float64, device=dev)   # (torch.where on Python scalars would give fp32)
    phi = torch.where(torch.from_numpy(gnz).to(dev), torch.tensor(nnz / nn, **f64),
                      torch.tensor((float(cfg.dims[0]) * float(cfg.dims[1]) * float(cfg.dims[2]) - nnz) / nz, **f64))
    Fref = float((phi * (m - x) ** 2).sum())
    # m_i is a sum of r signed terms: its rounding is bounded by (r + d + 2) ulps
    # of sum |terms| (both sides), so F^ is only that well determined where the
    # terms cancel (zero cells); plus the long-sum rounding of F^ itself
    eps = 2.0 ** -53
    bound = float((phi * 2 * (m - x).abs() * (cfg.rank + 5) * eps * am).sum()) + 1e-13 * abs(Fref)
    assert abs(Fg - Fref) <= bound, (Fg, Fref, bound)
    fref = 1.0 - math.sqrt(max(Fref, 0.0)) / math.sqrt(float((T.vals.to(torch.float64) ** 2).sum()))
    assert abs(fg - fref) <= 1e-8, (fg, fref)


def test_c4_als_update_sampled_rows(c4):
    """N2 at full size: one exact CP-ALS update of mode 0; B rows of sampled
    output rows (random + the heaviest) against B_i = M_i V^+ from their
    definitions: M_i = sum over the nonzeros of row i of x * (A_1 * A_2) rows
    (brute-force row selection over the COO, fp64), V = (A_1^T A_1) * (A_2^T A_2),
    V^+ with the oracle's Jacobi eigen-solver and the AMB-11/12 cutoff."""
    cfg, T, g = c4
    dev = T.coords.device
    k = 0
    A = [g.get_factor(m)[0] for m in range(3)]
    g.als_update(k)
    _, Bg = g.last_solve(k)
    V = (A[1].T @ A[1]) * (A[2].T @ A[2])
    w, Q = oracle.jacobi_eig(V)
    keep = w > cfg.rank * np.finfo(float).eps * w.max()
    Vp = (Q[:, keep] / w[keep]) @ Q[:, keep].T
    deg = torch.bincount(T.coords[:, 0].to(torch.int64), minlength=cfg.dims[0])
    rows = torch.cat([torch.topk(deg, 4).indices,
                      torch.randint(0, cfg.dims[0], (12,), device=dev,
                                    generator=torch.Generator(device=dev).manual_seed(1))]).tolist()
    A1, A2 = torch.from_numpy(A[1]).to(dev), torch.from_numpy(A[2]).to(dev)
    for i in rows:
        sel = torch.nonzero(T.coords[:, 0] == i).squeeze(1)
        c = T.coords[sel].to(torch.int64)
        x = T.vals[sel].to(torch.float64)
        Mi = (x[:, None] * A1[c[:, 1]] * A2[c[:, 2]]).sum(0).cpu().numpy()
        Bi = Mi @ Vp
        nb = np.linalg.norm(Bi)
        assert np.linalg.norm(Bg[i] - Bi) <= 1e-9 * max(nb, 1e-300), (i, np.linalg.norm(Bg[i] - Bi), nb)
