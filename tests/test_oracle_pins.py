"""Pins of the CPU oracle against things other than itself (PIN-1..PIN-13 of
DESIGN.md): the paper's worked examples and closed forms, brute force on tiny
inputs, numpy/LAPACK library routines, and invariants the paper states.
CPU only (-m "not gpu")."""
import itertools
import json
import math
import os

import numpy as np
import pytest

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


def rng(seed=0):
    return np.random.default_rng(seed)


# ----------------------------------------------------------------- Philox
def test_philox_known_answers():
    for case in GOLD["philox4x32_10_kat"]["cases"]:
        ctr = [int(x, 16) for x in case["ctr"]]
        key = [int(x, 16) for x in case["key"]]
        out = [int(x, 16) for x in case["out"]]
        assert list(oracle.philox4x32_10(ctr, key)) == out


# ----------------------------------------------------------------- PIN-1 key
def test_bijection_examples():
    for ex in GOLD["bijection"]:
        dims = ex["dims"]
        if "mode" in ex:
            assert oracle.key(dims, ex["mode"], ex["coord0"]) == ex["key"]
        else:
            # no excluded mode: pass k = D (out of range) so every mode counts
            assert oracle.key(dims, len(dims), ex["idx0"]) == ex["key"]


def test_bijection_uber_rows():
    u = GOLD["uber_rows"]
    dims = u["dims"]
    N = 1
    for m, n in enumerate(dims):
        if m != u["mode"]:
            N *= n
    assert N == u["N"]
    last = [n - 1 for n in dims]
    assert oracle.key(dims, u["mode"], last) == u["N"] - 1   # max key = N-1


def test_bijection_round_trip_exhaustive():
    dims = [4, 5, 6, 3]
    for k in range(len(dims)):
        others = [n for m, n in enumerate(dims) if m != k]
        seen = set()
        for multi in itertools.product(*[range(n) for n in others]):
            idx = list(multi)
            idx.insert(k, 0)
            key = oracle.key(dims, k, idx)
            seen.add(key)
            dec = oracle.decode(dims, k, key)
            assert [dec[m] for m in range(len(dims)) if m != k] == list(multi)
        assert seen == set(range(int(np.prod(others))))


def test_bijection_first_mode_fastest():
    # column-major / first index fastest (PAPER.md:221 with AMB-1 reading)
    dims = [7, 11, 13]
    assert oracle.key(dims, 2, [1, 0, 0]) == 1
    assert oracle.key(dims, 2, [0, 1, 0]) == 7
    assert oracle.key(dims, 0, [0, 0, 1]) == 11


# ----------------------------------------------------------------- PIN-2 leverage
def test_leverage_worked_example():
    ex = GOLD["leverage"]
    ell, rank = oracle.leverage(np.array(ex["A"], dtype=float))
    assert rank == 2
    np.testing.assert_allclose(ell, ex["ell"], rtol=0, atol=1e-15)


def test_leverage_identity_and_orthonormal():
    ell, rank = oracle.leverage(np.eye(5))
    assert rank == 5
    np.testing.assert_allclose(ell, 1.0, atol=1e-15)
    Q, _ = np.linalg.qr(rng(1).standard_normal((40, 6)))
    ell, rank = oracle.leverage(Q)
    np.testing.assert_allclose(ell, (Q ** 2).sum(1), rtol=1e-12, atol=1e-15)


def test_leverage_vs_numpy_qr_and_invariants():
    g = rng(2)
    for trial in range(20):
        n, r = int(g.integers(8, 80)), int(g.integers(1, 8))
        A = g.standard_normal((n, r)) * g.uniform(0.1, 10, size=r)
        ell, rank = oracle.leverage(A)
        Q, _ = np.linalg.qr(A)
        ref = (Q ** 2).sum(1)
        np.testing.assert_allclose(ell, ref, rtol=1e-10, atol=1e-13)
        assert rank == r
        assert abs(ell.sum() - r) < 1e-10
        assert ell.min() >= 0 and ell.max() <= 1 + 1e-12
        T = g.standard_normal((r, r)) + 3 * np.eye(r)
        ell2, _ = oracle.leverage(A @ T)                         # basis invariance
        np.testing.assert_allclose(ell2, ell, rtol=1e-9, atol=1e-12)


def test_leverage_rank_deficient():
    g = rng(3)
    A = g.standard_normal((30, 3)) @ g.standard_normal((3, 5))   # rank 3, r = 5
    ell, rank = oracle.leverage(A)
    assert rank == 3
    Q, _ = np.linalg.qr(A[:, :3])
    np.testing.assert_allclose(ell, (Q ** 2).sum(1), rtol=1e-8, atol=1e-10)
    A0 = np.zeros((4, 3))
    ell, rank = oracle.leverage(A0)
    assert rank == 0 and (ell == 0).all()


def test_jacobi_vs_eigh():
    g = rng(4)
    for r in (1, 2, 5, 25):
        X = g.standard_normal((50, r))
        G = X.T @ X
        w, V = oracle.jacobi_eig(G)
        np.testing.assert_allclose(np.sort(w), np.linalg.eigvalsh(G), rtol=1e-11, atol=1e-11)
        np.testing.assert_allclose(V @ np.diag(w) @ V.T, G, rtol=1e-11, atol=1e-10)


# ----------------------------------------------------------------- PIN-3 Lemma 5.1
def krp_explicit(As):
    """Rows in eq:bijection order (first factor fastest): Z[key] = A1[i1]*...*Ad[id]."""
    ns = [A.shape[0] for A in As]
    r = As[0].shape[1]
    N = int(np.prod(ns))
    Z = np.zeros((N, r))
    for key in range(N):
        t = key
        z = np.ones(r)
        for A, n in zip(As, ns):
            z = z * A[t % n]
            t //= n
        Z[key] = z
    return Z


def test_lemma_5_1_leverage_bound():
    g = rng(5)
    for trial in range(50):
        d = int(g.integers(2, 4))
        r = int(g.integers(1, 4))
        As = [g.standard_normal((int(g.integers(r + 1, 9)), r)) for _ in range(d)]
        Z = krp_explicit(As)
        Q, _ = np.linalg.qr(Z)
        lz = (Q ** 2).sum(1)
        ells = [oracle.leverage(A)[0] for A in As]
        bound = krp_explicit([e[:, None] for e in ells])[:, 0]
        assert (lz <= bound + 1e-10).all()


# ----------------------------------------------------------------- PIN-4 CDF/draw
def test_cdf_exact_dyadic_and_boundaries():
    pt = np.array([0.25, 0.0, 0.25, 0.5])
    Cc = oracle.cdf(pt)
    assert list(Cc) == [1 << 60, 1 << 60, 1 << 61, 1 << 62]
    # W = 2^62 so t = R >> 2 exactly
    assert oracle.draw(Cc, 4 * ((1 << 60) - 1)) == 0
    assert oracle.draw(Cc, 4 * (1 << 60)) == 2          # zero-weight entry 1 skipped
    assert oracle.draw(Cc, 4 * ((1 << 61) - 1)) == 2
    assert oracle.draw(Cc, 4 * (1 << 61)) == 3
    assert oracle.draw(Cc, (1 << 64) - 1) == 3
    assert oracle.draw(Cc, 0) == 0


def test_cdf_law_matches_ptilde():
    g = rng(6)
    for n in (1, 3, 100, 4097):
        pt = g.dirichlet(np.full(n, 0.3))
        Cc = oracle.cdf(pt)
        q = np.diff(np.concatenate([[0], Cc.astype(object)])).astype(float)
        W = float(int(Cc[-1]))
        np.testing.assert_allclose(q / W, pt, atol=n * 2.0 ** -60)


def _mk_oracle_with_ptilde(dims_other, pts, r=2):
    """A tensor whose mode 0 is the solved mode; other modes get given p~."""
    dims = [3] + list(dims_other)
    coords = np.zeros((1, len(dims)), dtype=np.int64)
    o = oracle.Oracle(dims, coords, np.ones(1), r)
    for j, pt in enumerate(pts):
        o.set_ptilde(j + 1, pt)
    return o


def test_sampler_tv_distance_product_law():
    # Lemma 5.4; SPEC acceptance 2: TV < 0.02
    g = rng(7)
    ns = [4, 5, 6]
    pts = [g.dirichlet(np.ones(n)) for n in ns]
    o = _mk_oracle_with_ptilde(ns, pts)
    s = 100_000
    o.sample(0, s, 1.0, 11, 0)
    smp = o.get_sample()
    assert not smp["is_det"].any() and smp["counts"].sum() == s
    N = int(np.prod(ns))
    emp = np.zeros(N)
    emp[smp["keys"].astype(np.int64)] = smp["counts"] / s
    prob = krp_explicit([p[:, None] for p in pts])[:, 0]
    assert 0.5 * np.abs(emp - prob).sum() < 0.02


# ----------------------------------------------------------------- PIN-5 DIDX
def test_didx_worked_example():
    ex = GOLD["didx"]
    keys, p, pdet = oracle.didx(ex["pt"], ex["tau"])
    assert list(keys) == ex["keys"]
    assert abs(pdet - ex["p_det"]) < 1e-15


def test_didx_tau_one_empty():
    keys, p, pdet = oracle.didx([[0.5, 0.5], [0.2, 0.8]], 1.0)
    assert len(keys) == 0 and pdet == 0.0


def test_didx_vs_brute_force():
    g = rng(8)
    for trial in range(100):
        d = int(g.integers(1, 4))
        ns = [int(g.integers(1, 30)) for _ in range(d)]
        while np.prod(ns) > 1e5:
            ns[int(np.argmax(ns))] //= 2
        pts = [g.dirichlet(np.full(n, g.uniform(0.05, 1.0))) for n in ns]
        N = int(np.prod(ns))
        tau = float(np.exp(g.uniform(np.log(1.0 / N), 0)))
        kb, pb, db = oracle.didx(pts, tau, brute=True)
        kp, pp, dp = oracle.didx(pts, tau)
        # numpy brute force, independent of the oracle's enumeration
        prob = krp_explicit([p[:, None] for p in pts])[:, 0]
        ref = np.nonzero(prob > tau)[0]
        assert list(kp) == list(kb)
        assert set(int(x) for x in kp) <= set(range(N))
        assert abs(dp - db) <= 1e-15
        # numpy's product order equals the canonical order, so sets agree exactly
        assert list(kp) == list(ref)
        assert abs(dp - prob[ref].sum()) <= 1e-10


# ----------------------------------------------------------------- PIN-6/7 SIDX + CIDX
def _raw_draws(pts, s_rnd, tau, seed, step):
    """Independent re-derivation of Alg. 2 from its statement (Python ints)."""
    from synth import philox4x32_10  # the input generator's independent Philox
    import torch
    Cs = []
    for pt in pts:
        q = [int(round(math.ldexp(float(x), 62))) for x in pt]
        Cs.append(np.cumsum(np.array(q, dtype=object)))
    d = len(pts)
    out, a = [], 0
    while len(out) < s_rnd:
        words = []
        for lane in range((d + 1) // 2):
            x = philox4x32_10(torch.tensor([a & 0xFFFFFFFF]), a >> 32, step, lane,
                              seed & 0xFFFFFFFF, seed >> 32)
            words += [int(v) for v in x]
        ii = []
        for j in range(d):
            lo, hi = words[4 * (j // 2) + 2 * (j % 2)], words[4 * (j // 2) + 2 * (j % 2) + 1]
            R = (hi << 32) | lo
            W = int(Cs[j][-1])
            t = (R * W) >> 64
            ii.append(int(np.searchsorted(np.array([int(c) for c in Cs[j]], dtype=object), t, side="right")))
        p = pts[0][ii[0]]
        for j in range(1, d):
            p = p * pts[j][ii[j]]
        if p <= tau:
            key, mult = 0, 1
            for j in range(d):
                key += ii[j] * mult
                mult *= len(pts[j])
            out.append(key)
        a += 1
    return out, a


def test_sidx_cidx_against_rederivation():
    g = rng(9)
    ns = [6, 7]
    pts = [g.dirichlet(np.full(n, 0.4)) for n in ns]
    o = _mk_oracle_with_ptilde(ns, pts)
    s, seed, step = 40, 1234567890123, 17
    tau = 1.0 / s
    info = o.sample(0, s, tau, seed, step)
    smp = o.get_sample()
    kd, pd, pdet = oracle.didx(pts, tau)
    assert info.s_det == len(kd) and abs(info.p_det - pdet) < 1e-15
    raw, att = _raw_draws(pts, s - len(kd), tau, seed, step)
    assert info.attempts == att
    det = smp["keys"][smp["is_det"]]
    assert list(det) == list(kd)
    assert (smp["w2"][smp["is_det"]] == 1.0).all()
    rnd_keys = smp["keys"][~smp["is_det"]]
    uniq, cnt = np.unique(np.array(raw, dtype=np.uint64), return_counts=True)
    assert list(rnd_keys) == list(uniq)
    assert list(smp["counts"][~smp["is_det"]]) == list(cnt)
    assert not set(int(x) for x in rnd_keys) & set(int(x) for x in kd)   # never in D
    s_rnd = s - len(kd)
    p = smp["p"][~smp["is_det"]]
    w2 = smp["w2"][~smp["is_det"]]
    # weight identity (AMB-3)
    np.testing.assert_allclose(w2 * s_rnd * p / ((1 - pdet) * cnt), 1.0, rtol=1e-14)
    # ||Omega_bar x|| = ||Omega x|| for random x
    N = int(np.prod(ns))
    prob = krp_explicit([q[:, None] for q in pts])[:, 0]
    for _ in range(20):
        x = g.standard_normal(N)
        lhs = (smp["w2"] * x[smp["keys"].astype(np.int64)] ** 2).sum()
        rhs = (x[kd.astype(np.int64)] ** 2).sum() + sum(
            (1 - pdet) / (s_rnd * prob[k]) * x[k] ** 2 for k in raw)
        assert abs(lhs - rhs) <= 1e-12 * abs(rhs)


def test_sidx_weight_example():
    ex = GOLD["sidx_weight"]
    o = _mk_oracle_with_ptilde([ex["n"]], [np.full(ex["n"], 1.0 / ex["n"])])
    o.sample(0, ex["s_rnd"], 1.0, 5, 0)
    smp = o.get_sample()
    np.testing.assert_allclose(smp["w2"] / smp["counts"], ex["w2_per_count"], rtol=1e-15)


def test_cidx_weight_example():
    ex = GOLD["cidx_weight"]
    # eq:combo with p_det = 0: w^2 = c/(s p)
    assert abs(ex["c"] / (ex["s"] * ex["p"]) - ex["w2"]) < 1e-15
    # oracle: a point mass of 0.5 on row 0 of a 2-row mode, tau = 1
    o = _mk_oracle_with_ptilde([2], [np.array([0.5, 0.5])])
    o.sample(0, ex["s"], 1.0, 99, 3)
    smp = o.get_sample()
    for c, w2 in zip(smp["counts"], smp["w2"]):
        assert abs(w2 - c / (ex["s"] * ex["p"])) < 1e-15


def test_point_mass_degenerate():
    # all mass on one index -> DIDX keeps it, random phase skipped
    o = _mk_oracle_with_ptilde([3, 4], [np.array([0, 1.0, 0]), np.array([0, 0, 1.0, 0])])
    info = o.sample(0, 16, -1, 1, 0)
    smp = o.get_sample()
    assert info.s_det == 1 and info.skipped_random == 1 and info.s_bar == 1
    assert int(smp["keys"][0]) == 1 + 3 * 2


# ----------------------------------------------------------------- PIN-8 unbiasedness
@pytest.mark.parametrize("tau_mode", ["random", "hybrid"])
def test_unbiasedness_monte_carlo(tau_mode):
    # PAPER.md:302-307 (squared, AMB-2); SPEC acceptance 5
    g = rng(10)
    ns = [16, 16]
    pts = [g.dirichlet(np.full(n, 0.5)) for n in ns]
    o = _mk_oracle_with_ptilde(ns, pts)
    N = 256
    x = g.standard_normal(N)
    s = 32
    tau = 1.0 if tau_mode == "random" else 1.0 / s
    vals = []
    for seed in range(10_000):
        o.sample(0, s, tau, seed, 0)
        smp = o.get_sample()
        vals.append((smp["w2"] * x[smp["keys"].astype(np.int64)] ** 2).sum())
    vals = np.array(vals)
    se = vals.std() / np.sqrt(len(vals))
    assert abs(vals.mean() - (x ** 2).sum()) < 3.5 * se


# ----------------------------------------------------------------- tensors for PIN-9..13
def random_tensor(dims, nnz, seed):
    g = rng(seed)
    N = int(np.prod(dims))
    lin = g.choice(N, size=nnz, replace=False)
    coords = np.stack(np.unravel_index(lin, dims, order="F"), axis=1).astype(np.int64)
    vals = g.standard_normal(nnz)
    return coords, vals


def dense_of(dims, coords, vals):
    X = np.zeros(dims)
    X[tuple(coords.T)] = vals
    return X


def unfold_mttkrp(X, As, k):
    """Dense MTTKRP X_(k) (KRP of others) via einsum (library routine)."""
    D = X.ndim
    letters = "abcdefgh"[:D]
    ops = [X]
    spec = [letters]
    for m in range(D):
        if m != k:
            ops.append(As[m])
            spec.append(letters[m] + "r")
    return np.einsum(",".join(spec) + "->" + letters[k] + "r", *ops)


def test_full_inclusion_equals_exact_als():
    # PIN-9: tau = 0 and s = N_k make every row deterministic with w = 1, so
    # G = *_m A_m^T A_m, RHS = MTTKRP and B = exact ALS.
    dims = (5, 6, 4)
    r = 3
    coords, vals = random_tensor(dims, 60, 11)
    g = rng(12)
    As = [g.uniform(size=(n, r)) for n in dims]
    o = oracle.Oracle(dims, coords, vals, r)
    for k, A in enumerate(As):
        o.set_factor(k, A)
    X = dense_of(dims, coords, vals)
    for k in range(3):
        Nk = int(np.prod([n for m, n in enumerate(dims) if m != k]))
        info = o.sample(k, Nk, 0.0, 1, k)
        assert info.s_det == Nk and info.s_bar == Nk
        cur = [o.get_factor(m)[0] for m in range(3)]
        so = o.solve_mode(k)
        G, M, B = o.last_solve(k)
        V = np.ones((r, r))
        for m in range(3):
            if m != k:
                V *= cur[m].T @ cur[m]
        np.testing.assert_allclose(G, V, rtol=1e-12, atol=1e-13)
        Mref = unfold_mttkrp(X, cur, k)
        np.testing.assert_allclose(M, Mref, rtol=1e-12, atol=1e-13)
        Bref = np.linalg.solve(V, Mref.T).T
        np.testing.assert_allclose(B, Bref, rtol=1e-10, atol=1e-12)
        # and the oracle's own exact-ALS routine agrees
        o2 = oracle.Oracle(dims, coords, vals, r)
        for m in range(3):
            o2.set_factor(m, cur[m])
        o2.als_update(k)
        _, _, B2 = o2.last_solve(k)
        np.testing.assert_allclose(B2, Bref, rtol=1e-10, atol=1e-12)
        A_new, lam = o.get_factor(k)
        np.testing.assert_allclose(lam, np.linalg.norm(Bref, axis=0), rtol=1e-12)
        np.testing.assert_allclose(A_new * lam, Bref, rtol=1e-10, atol=1e-12)


def test_fibers_vs_brute_force_and_example():
    ex = GOLD["tnsr_samp"]
    o = oracle.Oracle(ex["dims"], np.array([ex["coord0"]]), np.array([ex["value"]]), 1)
    o.set_ptilde(0, np.array([0.0, 1.0]))
    o.set_ptilde(1, np.array([1.0, 0.0, 0.0]))
    o.sample(ex["mode"], 1, 1.0, 0, 0)
    smp = o.get_sample()
    assert int(smp["keys"][0]) == ex["key"]
    lens, outs, vals = o.get_fibers()
    assert list(lens) == [1] and list(outs) == [ex["out"]] and list(vals) == [ex["value"]]
    # PIN-10: brute-force scan on a random tensor
    dims = (6, 5, 7, 3)
    coords, vals = random_tensor(dims, 300, 13)
    o = oracle.Oracle(dims, coords, vals, 2)
    g = rng(14)
    for k in range(4):
        for m in range(4):
            o.set_ptilde(m, g.dirichlet(np.ones(dims[m]) * 0.3))
        o.sample(k, 64, -1, 5, k)
        smp = o.get_sample()
        lens, outs, fv = o.get_fibers()
        off = 0
        for key, ln in zip(smp["keys"], lens):
            sel = [e for e in range(len(vals)) if oracle.key(dims, k, coords[e]) == int(key)]
            ref = sorted((int(coords[e, k]), vals[e]) for e in sel)
            got = list(zip(outs[off:off + ln].tolist(), fv[off:off + ln].tolist()))
            assert got == ref
            off += ln


def test_solve_vs_lstsq():
    # PIN-11: numpy.linalg.lstsq on the explicit sketched system
    dims = (8, 9, 10)
    r = 3
    coords, vals = random_tensor(dims, 500, 15)
    g = rng(16)
    o = oracle.Oracle(dims, coords, vals, r)
    As = [g.uniform(size=(n, r)) + 0.1 for n in dims]
    for k, A in enumerate(As):
        o.set_factor(k, A)
    for k in range(3):
        cur = [o.get_factor(m)[0] for m in range(3)]
        o.sample(k, 50, -1, 21, k)
        smp = o.get_sample()
        lens, outs, fv = o.get_fibers()
        others = [m for m in range(3) if m != k]
        Zs = np.zeros((len(smp["keys"]), r))
        Xs = np.zeros((len(smp["keys"]), dims[k]))
        off = 0
        for j, key in enumerate(smp["keys"]):
            idx = oracle.decode(dims, k, int(key))
            z = cur[others[0]][idx[others[0]]] * cur[others[1]][idx[others[1]]]
            w = math.sqrt(smp["w2"][j])
            Zs[j] = w * z
            Xs[j, outs[off:off + lens[j]]] = w * fv[off:off + lens[j]]
            off += lens[j]
        Bref = np.linalg.lstsq(Zs, Xs, rcond=None)[0].T
        o.solve_mode(k)
        _, _, B = o.last_solve(k)
        assert np.linalg.norm(B - Bref) <= 1e-10 * np.linalg.norm(Bref)


def test_fit_identities():
    # PIN-12: three-term identity = dense brute force; model = X -> 1; zero -> 0
    dims = (6, 7, 5)
    r = 2
    coords, vals = random_tensor(dims, 120, 17)
    g = rng(18)
    o = oracle.Oracle(dims, coords, vals, r)
    for k in range(3):
        o.set_factor(k, g.standard_normal((dims[k], r)))
    X = dense_of(dims, coords, vals)
    As = [o.get_factor(k)[0] for k in range(3)]
    M = np.einsum("ir,jr,kr->ijk", *As)
    ref = 1 - np.linalg.norm(X - M) / np.linalg.norm(X)
    assert abs(o.fit() - ref) < 1e-10
    assert abs(o.fit_dense() - ref) < 1e-10
    # exact rank-1 fully populated tensor
    a, b, c = g.uniform(size=6) + .5, g.uniform(size=7) + .5, g.uniform(size=5) + .5
    T = np.einsum("i,j,k->ijk", a, b, c)
    cc = np.array(list(itertools.product(range(6), range(7), range(5))), dtype=np.int64)
    o = oracle.Oracle(dims, cc, T[tuple(cc.T)], 1)
    for k, v in enumerate((a, b, c)):
        o.set_factor(k, v[:, None])
    assert abs(o.fit() - 1.0) < 1e-8
    o.set_factor(0, np.zeros((6, 1)))
    assert abs(o.fit()) < 1e-15


def _c1_dense():
    import synth
    T = synth.make("C1", dense_planted=True, index_dtype=__import__("torch").int64)
    return T


@pytest.mark.slow
def test_planted_rank3_recovery():
    # PIN-13 (BASELINE north_star invariant; AMB-24): fully populated C1.
    import synth
    T = _c1_dense()
    cfg = T.cfg
    init = synth.uniform_init(cfg.dims, cfg.rank, cfg.init_seed)
    o = oracle.Oracle(cfg.dims, T.coords.numpy(), T.vals.numpy(), cfg.rank)
    for k in range(3):
        o.set_factor(k, init[k].numpy())
    for it in range(100):
        for k in range(3):
            o.als_update(k)
    assert o.fit() >= 0.999
    o = oracle.Oracle(cfg.dims, T.coords.numpy(), T.vals.numpy(), cfg.rank)
    for k in range(3):
        o.set_factor(k, init[k].numpy())
    trace = o.run(60, cfg.s, -1, cfg.sample_seed, 1)
    assert np.nanmax(trace) >= 0.999
