"""Pins of the oracle's randomized range finder initialization (SURVEY 8(f)
N4; sec:enron P:1668-1701; reading AMB-34 in DESIGN.md).  CPU only.

* A_k = X_(k)(:, S) Omega checked against the dense mode-k unfolding with the
  fiber draws and Gaussian entries re-derived from their definitions with the
  input generator's independent Philox (synth.philox4x32_10) and numpy's libm;
* Omega is standard normal (moments over many draws);
* lambda = 1 and every column of A_k lies in the span of the sampled fibers.
"""
import math

import numpy as np
import torch

import oracle
from synth import philox4x32_10

from test_oracle_pins import dense_of, random_tensor


def words(seed, j, k, lane):
    x = philox4x32_10(torch.tensor([j & 0xFFFFFFFF]), j >> 32, 0x52524600 + k, lane,
                      seed & 0xFFFFFFFF, seed >> 32)
    return [int(v) for v in x]


def omega(seed, k, j, c):
    w = words(seed, j, k, c // 2)
    a, b = w[0] | (w[1] << 32), w[2] | (w[3] << 32)
    u1 = ((a >> 11) + 1) * 2.0 ** -53
    u2 = (b >> 11) * 2.0 ** -53
    rho = math.sqrt(-2.0 * math.log(u1))
    th = 2.0 * math.pi * u2
    return rho * math.cos(th) if c % 2 == 0 else rho * math.sin(th)


def unfold(X, k):
    """X_(k): rows i_k, columns the canonical key (other modes ascending, first fastest)."""
    other = [m for m in range(X.ndim) if m != k]
    Y = np.transpose(X, [k] + other)
    return Y.reshape(X.shape[k], -1, order="F")


def test_rrf_against_dense_definition():
    dims = (6, 7, 5)
    coords, vals = random_tensor(dims, 90, 13)
    X = dense_of(dims, coords, vals)
    r, s_init, seed = 3, 40, 987654321
    o = oracle.Oracle(dims, coords, vals, r)
    o.init_rrf(s_init, seed)
    for k in range(3):
        Xk = unfold(X, k)
        nonempty = np.flatnonzero(np.abs(Xk).sum(0) > 0)     # ascending canonical key
        S, Om = [], np.zeros((s_init, r))
        for j in range(s_init):
            w = words(seed, j, k, 0xFFFF)
            S.append(nonempty[((w[0] | (w[1] << 32)) * len(nonempty)) >> 64])
            for c in range(r):
                Om[j, c] = omega(seed, k, j, c)
        ref = Xk[:, S] @ Om
        A, lam = o.get_factor(k)
        np.testing.assert_allclose(A, ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())
        assert (lam == 1).all()
        # columns in the span of the sampled fibers
        F = Xk[:, sorted(set(S))]
        res = A - F @ np.linalg.lstsq(F, A, rcond=None)[0]
        assert np.abs(res).max() <= 1e-10 * np.abs(A).max()


def test_rrf_omega_is_standard_normal():
    z = np.array([oracle.lib().or_rrf_omega(5, 1, j, c) for j in range(6000) for c in range(4)])
    n = len(z)
    assert abs(z.mean()) < 4 / math.sqrt(n)
    assert abs(z.var() - 1) < 4 * math.sqrt(2 / n)
    assert abs(np.mean(z ** 4) - 3) < 0.15          # Gaussian kurtosis
