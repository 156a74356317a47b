"""Pins of the oracle's estimated fit and stopping rule (
sec:estimating-fit P:964-989; Alg. 3; readings AMB-32/33 in
DESIGN.md).  CPU only.

* the frozen stratified sample is re-derived from its definition with the
  input generator's independent Philox (synth.philox4x32_10): the nonzero
  stratum picks COO entries mulhi(R, nnz), the zero stratum the first
  floor((1-alpha) s) uniform cells that brute force finds absent from X;
* phi weights: nnz / ceil(alpha s) and (prod n - nnz) / floor((1-alpha) s);
* unbiasedness E[F^] = ||X - M||^2 (Monte Carlo over seeds, 4 sigma), with
  the exact residual from the dense brute force;
* an exactly decomposable sparse tensor (support = product of the factor
  supports) has F^ = 0 for every sample, zeros included;
* the stopping rule: tol = +inf stops after exactly pi epochs, tol = -inf
  runs max_epochs; the planted rank-3 tensor stops with fit >= 0.999.
"""
import math

import numpy as np
import pytest

import oracle

from test_oracle_pins import dense_of, random_tensor


def rederive_sample(coords, vals, dims, s_fit, alpha, seed):
    import torch
    from synth import philox4x32_10
    nnz = len(vals)
    nn = math.ceil(alpha * s_fit)
    nz = math.floor((1 - alpha) * s_fit)

    def word(ctr, lane, half):
        x = philox4x32_10(torch.tensor([ctr & 0xFFFFFFFF]), ctr >> 32, 0x46495400, lane,
                          seed & 0xFFFFFFFF, seed >> 32)
        w = [int(v) for v in x]
        return w[2 * half] | (w[2 * half + 1] << 32)

    idx_nz = [(word(i, 0, 0) * nnz) >> 64 for i in range(nn)]
    present = {tuple(int(v) for v in c) for c in coords}
    zeros, a = [], 0
    while len(zeros) < nz:
        cell = tuple((word(a, 1 + m // 2, m % 2) * dims[m]) >> 64 for m in range(len(dims)))
        if cell not in present:
            zeros.append(cell)
        a += 1
    return idx_nz, zeros


@pytest.mark.parametrize("alpha", [0.5, 0.25, 1.0])
def test_fit_sample_against_rederivation(alpha):
    dims = (7, 9, 11)
    coords, vals = random_tensor(dims, 150, 21)
    o = oracle.Oracle(dims, coords, vals, 2)
    s_fit, seed = 37, 123456789012345
    nn, nz = o.fit_sample(s_fit, alpha, seed)
    assert nn == math.ceil(alpha * s_fit) and nz == math.floor((1 - alpha) * s_fit)
    sc, sx, snz = o.get_fit_sample()
    idx_nz, zeros = rederive_sample(coords, vals, dims, s_fit, alpha, seed)
    assert (sc[:nn] == coords[idx_nz]).all() and (sx[:nn] == vals[idx_nz]).all()
    assert [tuple(c) for c in sc[nn:]] == zeros and (sx[nn:] == 0).all()
    assert snz[:nn].all() and not snz[nn:].any()


def test_phi_weights_and_unbiasedness():
    dims = (5, 6, 7)
    coords, vals = random_tensor(dims, 60, 5)
    X = dense_of(dims, coords, vals)
    r = 2
    g = np.random.default_rng(11)
    As = [g.standard_normal((n, r)) for n in dims]
    M = np.einsum("ir,jr,kr->ijk", *As)
    F = float(((X - M) ** 2).sum())
    normX = math.sqrt(float((X ** 2).sum()))
    o = oracle.Oracle(dims, coords, vals, r)
    for k in range(3):
        o.set_factor(k, As[k])          # lambda = 1
    s_fit, alpha = 40, 0.5
    est = []
    for seed in range(3000):
        o.fit_sample(s_fit, alpha, seed)
        f, Fh = o.fit_estimate()
        assert abs(f - (1 - math.sqrt(max(Fh, 0)) / normX)) < 1e-15
        est.append(Fh)
    est = np.array(est)
    # exact phi weights: F^ of a sample whose model is 0 and x = 1 everywhere is sum(phi)
    sc, sx, snz = o.get_fit_sample()
    nn, nz = int(snz.sum()), int((~snz).sum())
    phi_nz, phi_z = 60 / nn, (210 - 60) / nz
    m = np.array([sum(np.prod([As[k][c[k]] for k in range(3)], axis=0)) for c in sc])
    Fh_direct = (phi_nz * ((m[:nn] - sx[:nn]) ** 2)).sum() + (phi_z * ((m[nn:] - sx[nn:]) ** 2)).sum()
    assert abs(Fh_direct - est[-1]) <= 1e-12 * abs(Fh_direct)
    sigma = est.std() / math.sqrt(len(est))
    assert abs(est.mean() - F) <= 4 * sigma, (est.mean(), F, sigma)


def test_exact_sparse_decomposition_gives_zero():
    dims = (6, 5, 7)
    g = np.random.default_rng(3)
    a = [g.standard_normal(n) * (g.random(n) < 0.6) for n in dims]
    X = np.einsum("i,j,k->ijk", *a)
    coords = np.argwhere(X != 0)
    vals = X[tuple(coords.T)]
    o = oracle.Oracle(dims, coords, vals, 1)
    for k in range(3):
        o.set_factor(k, a[k][:, None])
    o.fit_sample(64, 0.5, 7)
    f, Fh = o.fit_estimate()
    assert Fh <= 1e-24 * float((vals ** 2).sum()) and f >= 1 - 1e-10


def test_stopping_rule_extremes():
    dims = (6, 7, 8)
    coords, vals = random_tensor(dims, 120, 8)
    for tol, epochs in ((math.inf, 3), (-math.inf, 6)):
        o = oracle.Oracle(dims, coords, vals, 2)
        g = np.random.default_rng(1)
        for k in range(3):
            o.set_factor(k, g.random((dims[k], 2)))
        o.fit_sample(64, 0.5, 1)
        tr = o.run_until(32, -1.0, 3, eta=2, pi=3, tol=tol, max_epochs=6, estimated=True)
        assert len(tr) == epochs and np.isfinite(tr).all()


@pytest.mark.slow
def test_planted_stops_converged():
    import synth
    import torch
    T = synth.make("C1", dense_planted=True, index_dtype=torch.int64)
    cfg = T.cfg
    init = synth.uniform_init(cfg.dims, cfg.rank, cfg.init_seed)
    o = oracle.Oracle(cfg.dims, T.coords.numpy(), T.vals.numpy(), cfg.rank)
    for k in range(3):
        o.set_factor(k, init[k].numpy())
    tr = o.run_until(cfg.s, -1.0, cfg.sample_seed, eta=5, pi=3, tol=1e-4, max_epochs=30)
    assert tr[-1] >= 0.999 and len(tr) < 30
    # the last pi epochs did not improve on the best by more than tol
    best = np.maximum.accumulate(tr)
    assert all(tr[e] <= best[e - 1] + 1e-4 for e in range(len(tr) - 3, len(tr)))
