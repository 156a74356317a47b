"""Round-2 pins of the CPU oracle (CPU only, -m "not gpu"):

* AMB-6 truncation (Alg. 1: "If not, we take the s highest
  probabilities"): when |DetSet| > s the oracle keeps the top s by
  (p desc, key asc) -- checked against a numpy brute force over every KRP row,
  on the brute-force and on the pruned DIDX path, with ties at the cut.
* AMB-11 (Alg. 3 lines 2/9): p~ = l/rank for a rank-deficient
  factor, after set_factor and after a solve with n_k < r -- checked against
  numpy's SVD (l_i = ||U(i, :rank)||^2, a library routine) divided by the
  numerical rank; sum p~ = 1.
* PIN-15 / sec:combine: combining repeats never changes the
  sketched solution (numpy lstsq on the uncombined rows) and never grows the
  right-hand side's nonzeros.
* PIN-15 / sec:hybrid-rand: on a problem with concentrated
  leverage, the relative residual difference shrinks as s grows and
  hybrid sampling (tau = 1/s) is at least as accurate as random (tau = 1)
  at every s (medians over 10 seeded runs).
"""
import math

import numpy as np
import pytest

import oracle


def _oracle_with_ptilde(dims_other, pts, r=2):
    """Mode 0 is solved; the other modes get the given p~ (set_ptilde)."""
    dims = [3] + list(dims_other)
    o = oracle.Oracle(dims, np.zeros((1, len(dims)), dtype=np.int64), np.ones(1), r)
    for j, pt in enumerate(pts):
        o.set_ptilde(j + 1, pt)
    return o


def _brute_top_s(pts, tau, s):
    """numpy brute force: every KRP row (key = i1 + n1 i2 + ..., AMB-1), the
    canonical left-to-right product (AMB-5), DetSet = {p > tau} (AMB-4), then
    the s largest by (p desc, key asc) (AMB-6)."""
    p = pts[0].copy()
    for q in pts[1:]:
        p = (p[:, None] * q[None, :]).reshape(-1, order="F")   # first mode fastest
    keys = np.arange(p.size, dtype=np.uint64)
    sel = p > tau
    p, keys = p[sel], keys[sel]
    o = np.lexsort((keys, -p))[:s]
    return np.sort(keys[o]), p[o], int(sel.sum())


@pytest.mark.parametrize("case", ["brute_path", "pruned_path"])
def test_didx_truncation_top_s(case):
    if case == "brute_path":
        # 5 x 6 KRP rows; products tie in pairs, the cut falls inside a tie
        pts = [np.array([0.3, 0.3, 0.2, 0.1, 0.1]), np.array([0.25, 0.25, 0.2, 0.1, 0.1, 0.1])]
        tau, s = 1e-3, 7
    else:
        # N = 1.2e7 > 1e7: the oracle's pruned enumeration (didx_collect);
        # 12 equal products 0.05 at the top, s = 5 cuts inside them
        nA, nB = 4000, 3000
        pA = np.full(nA, 0.2 / (nA - 4)); pA[[7, 100, 2500, 3999]] = 0.2
        pB = np.full(nB, 0.25 / (nB - 3)); pB[[0, 1500, 2999]] = 0.25
        pts, tau, s = [pA, pB], 1e-6, 5
    o = _oracle_with_ptilde([len(p) for p in pts], pts)
    info = o.sample(0, s, tau, 77, 3)
    ref_keys, ref_p, n_det = _brute_top_s(pts, tau, s)
    assert n_det > s                                   # the truncation branch runs
    assert info.s_det == s and info.s_rnd == 0 and info.s_bar == s
    smp = o.get_sample()
    assert smp["is_det"].all()
    assert list(smp["keys"]) == list(ref_keys)
    assert (smp["w2"] == 1.0).all() and (smp["counts"] == 1).all()
    # p_det = sum of the kept p (compensated sum vs math.fsum)
    assert abs(info.p_det - math.fsum(ref_p)) <= 1e-15 * math.fsum(ref_p)
    # the cut falls inside a tie, so a (p desc, key desc) tie-break or an
    # ascending order would keep other keys: the fixture can tell them apart
    p = pts[0].copy()
    for q in pts[1:]:
        p = (p[:, None] * q[None, :]).reshape(-1, order="F")
    keys = np.arange(p.size, dtype=np.uint64)
    sel = p > tau
    kdesc = np.sort(keys[sel][np.lexsort((-keys[sel].astype(np.int64), -p[sel]))[:s]])
    pasc = np.sort(keys[sel][np.lexsort((keys[sel], p[sel]))[:s]])
    assert list(kdesc) != list(ref_keys) and list(pasc) != list(ref_keys)


def _svd_ptilde(A, r):
    U, S, _ = np.linalg.svd(A, full_matrices=False)
    if S.size == 0 or S[0] == 0.0:
        return np.zeros(A.shape[0]), 0
    rank = int((S ** 2 > r * np.finfo(float).eps * S[0] ** 2).sum())
    ell = (U[:, :rank] ** 2).sum(1)
    return ell / rank, rank


def test_refresh_rank_deficient_ptilde_set_factor():
    g = np.random.default_rng(21)
    dims, r = (40, 7, 9), 5
    coords = np.stack([g.integers(0, n, 30) for n in dims], 1)
    o = oracle.Oracle(dims, coords, g.uniform(size=30), r)
    A = g.standard_normal((40, 3)) @ g.standard_normal((3, r))      # rank 3 < r
    o.set_factor(0, A)
    ref, rank = _svd_ptilde(A, r)
    assert rank == 3
    pt = o.get_ptilde(0)
    np.testing.assert_allclose(pt, ref, rtol=1e-10, atol=1e-14)
    assert abs(pt.sum() - 1.0) <= 1e-12                 # l/r would sum to 3/5
    o.set_factor(1, np.zeros((7, r)))                   # rank 0: no drawable row
    assert (o.get_ptilde(1) == 0).all()


def test_refresh_rank_deficient_ptilde_after_solve():
    """Alg. 3 line 9: the refresh after a solve whose factor has
    n_k = 3 < r = 5 rows (rank <= 3)."""
    g = np.random.default_rng(22)
    dims, r = (3, 8, 9), 5
    lin = g.choice(np.prod(dims), 120, replace=False)
    coords = np.stack(np.unravel_index(lin, dims, order="F"), 1).astype(np.int64)
    o = oracle.Oracle(dims, coords, g.uniform(0.5, 2.0, 120), r)
    for k, n in enumerate(dims):
        o.set_factor(k, g.uniform(size=(n, r)) + 0.1)
    o.sample(0, 64, -1.0, 5, 0)
    o.solve_mode(0)
    A0, _ = o.get_factor(0)
    ref, rank = _svd_ptilde(A0, r)
    assert 1 <= rank <= 3
    pt = o.get_ptilde(0)
    np.testing.assert_allclose(pt, ref, rtol=1e-9, atol=1e-14)
    assert abs(pt.sum() - 1.0) <= 1e-12


def _dense(dims, coords, vals):
    X = np.zeros(dims)
    X[tuple(coords.T)] = vals
    return X


def test_combining_never_changes_the_solution():
    """sec:combine: the combined rows (w^2 = c(1-p_det)/(s_rnd p))
    give the same B as the uncombined sketch (each draw its own row, weight
    (1-p_det)/(s_rnd p)) solved by numpy lstsq, and carry fewer RHS nonzeros
    whenever a row repeats."""
    g = np.random.default_rng(23)
    dims, r = (10, 12, 8), 3
    lin = g.choice(np.prod(dims), 600, replace=False)
    coords = np.stack(np.unravel_index(lin, dims, order="F"), 1).astype(np.int64)
    vals = g.uniform(0.5, 2.0, 600)
    o = oracle.Oracle(dims, coords, vals, r)
    As = [g.uniform(size=(n, r)) + 0.05 for n in dims]
    As[1][:2] *= 8.0                                         # concentrate the leverage: repeats
    for k, A in enumerate(As):
        o.set_factor(k, A)
    for tau in (1.0, -1.0):
        for k in range(3):
            cur = [o.get_factor(m)[0] for m in range(3)]
            info = o.sample(k, 200, tau, 31 + k, k)
            smp = o.get_sample()
            lens, outs, fv = o.get_fibers()
            others = [m for m in range(3) if m != k]
            rows_z, rows_x = [], []
            off = 0
            for j, key in enumerate(smp["keys"]):
                idx = oracle.decode(dims, k, int(key))
                z = cur[others[0]][idx[others[0]]] * cur[others[1]][idx[others[1]]]
                x = np.zeros(dims[k])
                x[outs[off:off + lens[j]]] = fv[off:off + lens[j]]
                off += lens[j]
                c = int(smp["counts"][j])
                w2_one = smp["w2"][j] / c            # each repeated draw's own weight
                for _ in range(c):
                    rows_z.append(math.sqrt(w2_one) * z)
                    rows_x.append(math.sqrt(w2_one) * x)
            Bref = np.linalg.lstsq(np.array(rows_z), np.array(rows_x), rcond=None)[0].T
            o.solve_mode(k)
            _, _, B = o.last_solve(k)
            assert np.linalg.norm(B - Bref) <= 1e-10 * np.linalg.norm(Bref), (tau, k)
            nnz_comb = int(lens.sum())
            nnz_uncomb = int((lens * smp["counts"]).sum())
            assert nnz_comb <= nnz_uncomb
            if (smp["counts"][lens > 0] > 1).any():
                assert nnz_comb < nnz_uncomb
            assert info.s_bar <= 200


def _residual_study(s_list, runs=10):
    """Concentrated-leverage least squares for mode 0 of a fully populated
    20 x 60 x 60 tensor (sec:hybrid-rand, P:1177-1209 at toy size): returns
    the median relative residual difference per s for tau = 1 and
    tau = 1/s."""
    g = np.random.default_rng(24)
    dims, r = (20, 60, 60), 4
    A1 = g.standard_normal((60, r)); A1[:3] *= 25.0
    A2 = g.standard_normal((60, r)); A2[:2] *= 25.0
    Bt = g.standard_normal((20, r))
    Z = (A1[:, None, :] * A2[None, :, :]).transpose(1, 0, 2).reshape(-1, r)   # key = i1 + 60 i2
    X0 = Z @ Bt.T + 0.5 * g.standard_normal((3600, 20))                        # X_(0)^T
    X = X0.T.reshape(20, 60, 60, order="F")
    coords = np.stack(np.unravel_index(np.arange(X.size), dims, order="F"), 1).astype(np.int64)
    vals = X.reshape(-1, order="F")
    Bstar = np.linalg.lstsq(Z, X0, rcond=None)[0]
    rstar = np.linalg.norm(Z @ Bstar - X0) ** 2
    o = oracle.Oracle(dims, coords, vals, r)
    o.set_factor(1, A1)
    o.set_factor(2, A2)
    out = {}
    for s in s_list:
        for name, tau in (("random", 1.0), ("hybrid", -1.0)):
            diffs = []
            for run in range(runs):
                o.sample(0, s, tau, 1000 + run, s)
                o.solve_mode(0)
                _, _, B = o.last_solve(0)
                rs = np.linalg.norm(Z @ B.T - X0) ** 2
                diffs.append(abs(rs - rstar) / max(1.0, rstar))
            out[(name, s)] = float(np.median(diffs))
    return out


def test_hybrid_vs_random_residual_trend():
    s_list = (32, 128, 512)
    med = _residual_study(s_list)
    for name in ("random", "hybrid"):
        seq = [med[(name, s)] for s in s_list]
        assert all(b < a for a, b in zip(seq, seq[1:])), (name, seq)   # decreases in s
    for s in s_list:
        assert med[("hybrid", s)] <= med[("random", s)], (s, med)      # hybrid no worse
