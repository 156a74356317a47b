"""ctypes wrapper of the plain-C CP-ARLS-LEV oracle (oracle/cparls_oracle.c).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` legs may import this module.
The product path (paper_2006_16438_b200) never imports it and shares no code
with it.  Functions cite PAPER.md lines in the C source.

Parity pins: every function here is pinned in tests/test_oracle_*.py against
closed forms, brute force, numpy/LAPACK library routines or the paper's worked
examples.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "cparls_oracle.c")
_LIB = os.path.join(_HERE, "libcparls_oracle.so")


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "cparls_oracle.h"))):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fPIC", "-shared", "-std=gnu11",
                               "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _setup(_lib)
    return _lib


class SampleInfo(C.Structure):
    _fields_ = [("s_det", C.c_int64), ("s_rnd", C.c_int64), ("s_bar", C.c_int64),
                ("attempts", C.c_int64), ("p_det", C.c_double), ("skipped_random", C.c_int32)]


class SolveInfo(C.Structure):
    _fields_ = [("matched_nnz", C.c_int64), ("touched_rows", C.c_int64),
                ("rank_used", C.c_int32), ("chol_fallback", C.c_int32)]


P = C.c_void_p
I64 = C.c_int64
U64 = C.c_uint64
D = C.c_double
I32 = C.c_int


def _setup(L):
    L.or_philox4x32_10.argtypes = [P, P, P]
    L.or_key.argtypes = [I32, P, I32, P]; L.or_key.restype = U64
    L.or_decode.argtypes = [I32, P, I32, U64, P]
    L.or_jacobi_eig.argtypes = [I32, P, P, P]
    L.or_leverage.argtypes = [I64, I32, P, P]; L.or_leverage.restype = I32
    L.or_cdf.argtypes = [I64, P, P]
    L.or_draw.argtypes = [I64, P, U64]; L.or_draw.restype = I64
    L.or_create.argtypes = [I32, P, I64, P, P, I32]; L.or_create.restype = P
    L.or_destroy.argtypes = [P]
    L.or_set_factor.argtypes = [P, I32, P]; L.or_set_factor.restype = I32
    L.or_get_factor.argtypes = [P, I32, P, P]
    L.or_set_ptilde.argtypes = [P, I32, P]
    L.or_get_ptilde.argtypes = [P, I32, P]
    L.or_leverage_mode.argtypes = [P, I32, P]; L.or_leverage_mode.restype = I32
    L.or_sample.argtypes = [P, I32, I64, D, U64, U64, C.POINTER(SampleInfo)]; L.or_sample.restype = I32
    L.or_get_sample.argtypes = [P, I64, P, P, P, P, P]; L.or_get_sample.restype = I64
    L.or_get_fibers.argtypes = [P, I64, P, P, P]; L.or_get_fibers.restype = I64
    L.or_solve_mode.argtypes = [P, I32, C.POINTER(SolveInfo)]; L.or_solve_mode.restype = I32
    L.or_get_last_solve.argtypes = [P, P, P, P]
    L.or_fit.argtypes = [P]; L.or_fit.restype = D
    L.or_fit_dense.argtypes = [P]; L.or_fit_dense.restype = D
    L.or_als_update.argtypes = [P, I32]; L.or_als_update.restype = I32
    L.or_run.argtypes = [P, I32, I64, D, U64, I32, P]; L.or_run.restype = I32
    L.or_didx.argtypes = [I32, P, P, D, I64, P, P, P]; L.or_didx.restype = I64
    L.or_didx_brute.argtypes = [I32, P, P, D, I64, P, P, P]; L.or_didx_brute.restype = I64
    L.or_fit_sample.argtypes = [P, I64, D, U64, P, P]; L.or_fit_sample.restype = I32
    L.or_init_rrf.argtypes = [P, I64, U64]; L.or_init_rrf.restype = I32
    L.or_rrf_omega.argtypes = [U64, I32, U64, I32]; L.or_rrf_omega.restype = D
    L.or_rrf_fiber.argtypes = [U64, I32, U64, I64]; L.or_rrf_fiber.restype = I64
    L.or_get_fit_sample.argtypes = [P, I64, P, P, P]; L.or_get_fit_sample.restype = I64
    L.or_fit_estimate.argtypes = [P, P]; L.or_fit_estimate.restype = D
    L.or_run_until.argtypes = [P, I64, D, U64, I32, I32, D, I32, I32, P, P]; L.or_run_until.restype = I32


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


# ---------------------------------------------------------------- primitives
def philox4x32_10(ctr, key):
    c = np.asarray(ctr, dtype=np.uint32).copy()
    k = np.asarray(key, dtype=np.uint32).copy()
    out = np.zeros(4, dtype=np.uint32)
    lib().or_philox4x32_10(_p(c), _p(k), _p(out))
    return out


def key(dims, k, idx):
    d = np.asarray(dims, dtype=np.int64)
    i = np.asarray(idx, dtype=np.int64)
    return int(lib().or_key(len(d), _p(d), k, _p(i)))


def decode(dims, k, key_):
    d = np.asarray(dims, dtype=np.int64)
    out = np.full(len(d), -1, dtype=np.int64)
    lib().or_decode(len(d), _p(d), k, key_, _p(out))
    return out


def jacobi_eig(G):
    G = np.ascontiguousarray(G, dtype=np.float64)
    r = G.shape[0]
    w = np.zeros(r); V = np.zeros((r, r))
    lib().or_jacobi_eig(r, _p(G), _p(w), _p(V))
    return w, V


def leverage(A):
    A = np.ascontiguousarray(A, dtype=np.float64)
    n, r = A.shape
    ell = np.zeros(n)
    rank = lib().or_leverage(n, r, _p(A), _p(ell))
    return ell, rank


def cdf(pt):
    pt = np.ascontiguousarray(pt, dtype=np.float64)
    Cc = np.zeros(len(pt), dtype=np.uint64)
    lib().or_cdf(len(pt), _p(pt), _p(Cc))
    return Cc


def draw(Cc, R):
    Cc = np.ascontiguousarray(Cc, dtype=np.uint64)
    return int(lib().or_draw(len(Cc), _p(Cc), int(R)))


def _ptarr(pts):
    arrs = [np.ascontiguousarray(p, dtype=np.float64) for p in pts]
    ptrs = (C.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])
    n = np.array([len(a) for a in arrs], dtype=np.int64)
    return arrs, ptrs, n


def didx(pts, tau, cap=1 << 22, brute=False):
    arrs, ptrs, n = _ptarr(pts)
    keys = np.zeros(cap, dtype=np.uint64)
    p = np.zeros(cap)
    pdet = np.zeros(1)
    f = lib().or_didx_brute if brute else lib().or_didx
    cnt = f(len(arrs), _p(n), C.cast(ptrs, C.c_void_p), tau, cap, _p(keys), _p(p), _p(pdet))
    if cnt < 0:
        raise RuntimeError("didx cap exceeded")
    return keys[:cnt], p[:cnt], float(pdet[0])


# ---------------------------------------------------------------- context
class Oracle:
    """The oracle's state machine: tensor + Kruskal model + sample."""

    def __init__(self, dims, coords, vals, rank):
        self.dims = tuple(int(x) for x in dims)
        self.D = len(self.dims)
        self.r = int(rank)
        coords = np.ascontiguousarray(np.asarray(coords), dtype=np.int64)
        vals = np.ascontiguousarray(np.asarray(vals), dtype=np.float64)
        self.nnz = coords.shape[0]
        d = np.array(self.dims, dtype=np.int64)
        self._h = lib().or_create(self.D, _p(d), self.nnz, _p(coords), _p(vals), self.r)
        if not self._h:
            raise ValueError("or_create failed")

    def close(self):
        if self._h:
            lib().or_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_factor(self, k, A):
        A = np.ascontiguousarray(A, dtype=np.float64)
        assert A.shape == (self.dims[k], self.r)
        return lib().or_set_factor(self._h, k, _p(A))

    def get_factor(self, k):
        A = np.zeros((self.dims[k], self.r))
        lam = np.zeros(self.r)
        lib().or_get_factor(self._h, k, _p(A), _p(lam))
        return A, lam

    def set_ptilde(self, k, pt):
        pt = np.ascontiguousarray(pt, dtype=np.float64)
        lib().or_set_ptilde(self._h, k, _p(pt))

    def get_ptilde(self, k):
        pt = np.zeros(self.dims[k])
        lib().or_get_ptilde(self._h, k, _p(pt))
        return pt

    def leverage(self, k):
        ell = np.zeros(self.dims[k])
        rank = lib().or_leverage_mode(self._h, k, _p(ell))
        return ell, rank

    def sample(self, k, s, tau, seed, step):
        info = SampleInfo()
        st = lib().or_sample(self._h, k, s, tau, seed, step, C.byref(info))
        if st:
            raise RuntimeError(f"or_sample status {st}")
        return info

    def get_sample(self):
        n = lib().or_get_sample(self._h, 0, None, None, None, None, None)
        keys = np.zeros(n, dtype=np.uint64); cnt = np.zeros(n, dtype=np.int32)
        w2 = np.zeros(n); p = np.zeros(n); isdet = np.zeros(n, dtype=np.uint8)
        lib().or_get_sample(self._h, n, _p(keys), _p(cnt), _p(w2), _p(p), _p(isdet))
        return dict(keys=keys, counts=cnt, w2=w2, p=p, is_det=isdet.astype(bool))

    def get_fibers(self):
        n = lib().or_get_sample(self._h, 0, None, None, None, None, None)
        lens = np.zeros(n, dtype=np.int64)
        tot = lib().or_get_fibers(self._h, 0, _p(lens), None, None)
        out = np.zeros(tot, dtype=np.int64); val = np.zeros(tot)
        lib().or_get_fibers(self._h, tot, _p(lens), _p(out), _p(val))
        return lens, out, val

    def solve_mode(self, k):
        info = SolveInfo()
        st = lib().or_solve_mode(self._h, k, C.byref(info))
        if st:
            raise RuntimeError(f"or_solve_mode status {st}")
        return info

    def last_solve(self, k):
        G = np.zeros((self.r, self.r)); M = np.zeros((self.dims[k], self.r))
        B = np.zeros((self.dims[k], self.r))
        lib().or_get_last_solve(self._h, _p(G), _p(M), _p(B))
        return G, M, B

    def fit(self):
        return float(lib().or_fit(self._h))

    def fit_dense(self):
        return float(lib().or_fit_dense(self._h))

    def als_update(self, k):
        return lib().or_als_update(self._h, k)

    def init_rrf(self, s_init, seed=0):
        """Randomized range finder initialization of every factor (AMB-34)."""
        st = lib().or_init_rrf(self._h, int(s_init), int(seed))
        if st:
            raise RuntimeError(f"or_init_rrf status {st}")

    def fit_sample(self, s_fit, alpha=0.5, seed=0):
        """Draw and freeze the stratified fit sample (AMB-32)."""
        nn, nz = C.c_int64(), C.c_int64()
        st = lib().or_fit_sample(self._h, int(s_fit), float(alpha), int(seed), C.byref(nn), C.byref(nz))
        if st:
            raise RuntimeError(f"or_fit_sample status {st}")
        return nn.value, nz.value

    def get_fit_sample(self):
        n = lib().or_get_fit_sample(self._h, 0, None, None, None)
        coords = np.zeros((n, self.D), dtype=np.int64); x = np.zeros(n); nz = np.zeros(n, dtype=np.uint8)
        lib().or_get_fit_sample(self._h, n, _p(coords), _p(x), _p(nz))
        return coords, x, nz.astype(bool)

    def fit_estimate(self):
        F = np.zeros(1)
        f = lib().or_fit_estimate(self._h, _p(F))
        return float(f), float(F[0])

    def run_until(self, s, tau, seed, eta=5, pi=3, tol=1e-4, max_epochs=50, estimated=False):
        """Alg. 3 with its stopping rule (AMB-33); returns the per-epoch fit trace."""
        trace = np.full(max_epochs, np.nan)
        ep = C.c_int()
        st = lib().or_run_until(self._h, int(s), float(tau), int(seed), int(eta), int(pi), float(tol),
                                int(max_epochs), 1 if estimated else 0, _p(trace), C.byref(ep))
        if st:
            raise RuntimeError(f"or_run_until status {st}")
        return trace[:ep.value]

    def run(self, iters, s, tau, seed, fit_every=1):
        trace = np.full(iters, np.nan)
        st = lib().or_run(self._h, iters, s, tau, seed, fit_every, _p(trace))
        if st:
            raise RuntimeError(f"or_run status {st}")
        return trace
