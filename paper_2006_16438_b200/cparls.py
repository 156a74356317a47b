"""Thin ctypes binding of libcparls.so (include/cparls.h).

Argument marshalling only: every step of CP-ARLS-LEV runs in the CUDA kernels
of csrc/.  There is no CPU fallback -- if the shared library is missing or
cannot be loaded, or no CUDA device is present, the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# CPARLS_LIB: an alternative in-tree build of the same library (A/B experiments)
LIB_PATH = os.environ.get("CPARLS_LIB") or os.path.join(_HERE, "libcparls.so")

OK, EINVAL, EOOM, ECUDA, ENCCL, ENUMERIC, ESAMPLE, ERANGE, ESTATE = range(9)
_NAMES = ["OK", "EINVAL", "EOOM", "ECUDA", "ENCCL", "ENUMERIC", "ESAMPLE", "ERANGE", "ESTATE"]


class CparlsError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"cparls {_NAMES[status] if 0 <= status < 9 else status}: {msg}")
        self.status = status


class Opts(C.Structure):
    """cparls_opts (include/cparls.h); struct_size versions the layout."""
    _fields_ = [("struct_size", C.c_uint32), ("rank", C.c_int32), ("tau", C.c_double),
                ("value_dtype", C.c_int32), ("index_dtype", C.c_int32), ("stream", C.c_void_p),
                ("world_size", C.c_int32), ("world_rank", C.c_int32), ("comm", C.c_void_p),
                ("didx_cap", C.c_int64), ("attempt_cap", C.c_int64), ("rhs_path", C.c_int32),
                ("fit_samples", C.c_int64), ("fit_alpha", C.c_double), ("fit_seed", C.c_uint64),
                ("sidx_window", C.c_int64), ("sample_sort", C.c_int32), ("fit_mode", C.c_int32),
                ("rhs_hot_rows", C.c_int32)]


class SampleInfo(C.Structure):
    _fields_ = [("s_det", C.c_int64), ("s_rnd", C.c_int64), ("s_bar", C.c_int64),
                ("attempts", C.c_int64), ("p_det", C.c_double), ("skipped_random", C.c_int32)]


class SolveInfo(C.Structure):
    _fields_ = [("matched_nnz", C.c_int64), ("touched_rows", C.c_int64),
                ("rank_used", C.c_int32), ("chol_fallback", C.c_int32)]


class Stats(C.Structure):
    _fields_ = [("struct_size", C.c_uint32), ("reserved0", C.c_uint32)] + [(n, C.c_double) for n in (
        "ms_leverage", "ms_sample", "ms_gram", "ms_lookup", "ms_rhs", "ms_solve", "ms_fit",
        "bytes_leverage", "bytes_sample", "bytes_gram", "bytes_lookup", "bytes_rhs", "bytes_solve",
        "bytes_fit")] + [(n, C.c_int64) for n in (
        "mode_steps", "fits", "kernel_launches", "last_matched_nnz", "last_s_bar", "last_attempts")] + [
        ("touched_rows", C.c_int64 * 8), ("kernel_ms", C.c_double * 4),
        ("kernel_launches_by_id", C.c_int64 * 4), ("sum_matched_nnz", C.c_int64), ("host_syncs", C.c_int64),
        ("bytes_comm", C.c_double), ("create_ms", C.c_double * 4), ("rhs_hot_rows", C.c_int32 * 8),
        ("rhs_hot_share", C.c_double * 8), ("build_ms", C.c_double * 4)]

    KERNELS = ("rhs", "fit", "solve_rows", "lev_rows")

    def as_dict(self):
        d = {n: getattr(self, n) for n, _ in self._fields_}
        d["touched_rows"] = list(self.touched_rows)
        d["create_ms"] = list(self.create_ms)
        d["rhs_hot_rows"] = list(self.rhs_hot_rows)
        d["rhs_hot_share"] = list(self.rhs_hot_share)
        d["build_ms"] = list(self.build_ms)
        d["kernel_ms"] = {k: self.kernel_ms[i] for i, k in enumerate(self.KERNELS)}
        d["kernel_launches_by_id"] = {k: self.kernel_launches_by_id[i] for i, k in enumerate(self.KERNELS)}
        return d


_lib = None


def lib():
    """Load libcparls.so (raises if it is missing: no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run __graft_entry__.build() (nvcc, sm_100a)")
        L = C.CDLL(LIB_PATH)
        P, I32, I64, U64, D = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_double
        sig = {
            "cparls_create": [C.POINTER(P), I32, P, I64, P, P, C.POINTER(Opts), U64],
            "cparls_destroy": [P],
            "cparls_set_factor": [P, I32, P],
            "cparls_get_factor": [P, I32, P, P],
            "cparls_leverage": [P, I32, P, P],
            "cparls_get_ptilde": [P, I32, P],
            "cparls_set_ptilde": [P, I32, P],
            "cparls_sample": [P, I32, I64, U64, U64, C.POINTER(SampleInfo)],
            "cparls_set_tau": [P, D],
            "cparls_get_sample": [P, I64, P, P, P, P, P, P],
            "cparls_get_fibers": [P, I64, P, P, P, P],
            "cparls_solve_mode": [P, I32, C.POINTER(SolveInfo)],
            "cparls_get_last_solve": [P, P, P],
            "cparls_fit": [P, P],
            "cparls_run": [P, I32, I64, U64, I32, I32, P],
            "cparls_fit_estimate": [P, P, P],
            "cparls_get_fit_sample": [P, I64, P, P, P, P],
            "cparls_fit_sample_model": [P, P],
            "cparls_run_until": [P, I64, U64, I32, I32, D, I32, I32, P, P],
            "cparls_als_update": [P, I32],
            "cparls_init_rrf": [P, I64, U64],
            "cparls_run_als": [P, I32, I32, P],
            "cparls_get_stats": [P, P, I64],
            "cparls_reset_stats": [P],
            "cparls_set_profiling": [P, I32],
            "cparls_comm_nccl_unique_id": [P],
            "cparls_comm_create_nccl": [I32, I32, P, C.POINTER(P)],
            "cparls_comm_create_local": [I32, C.POINTER(P)],
            "cparls_comm_destroy": [P],
            "cparls_plan_rows": [I64, P, I32, P, P],
            "cparls_route_nonzeros": [I32, I32, I64, P, I32, P, P, P],
            "cparls_owned_rows": [P, I32, P, P],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = C.c_int
        L.cparls_last_error.argtypes = [P]
        L.cparls_last_error.restype = C.c_char_p
        L.cparls_opts_init.argtypes = [P]
        L.cparls_opts_init.restype = None
        L.cparls_version.argtypes = []
        L.cparls_version.restype = C.c_char_p
        _lib = L
    return _lib


EXPORTED = ["cparls_create", "cparls_destroy", "cparls_set_factor", "cparls_get_factor",
            "cparls_leverage", "cparls_get_ptilde", "cparls_set_ptilde", "cparls_sample",
            "cparls_set_tau", "cparls_get_sample", "cparls_get_fibers", "cparls_solve_mode",
            "cparls_get_last_solve", "cparls_fit", "cparls_run", "cparls_fit_estimate",
            "cparls_get_fit_sample", "cparls_fit_sample_model", "cparls_run_until", "cparls_init_rrf", "cparls_als_update",
            "cparls_run_als", "cparls_get_stats",
            "cparls_reset_stats", "cparls_set_profiling", "cparls_last_error", "cparls_version",
            "cparls_comm_nccl_unique_id", "cparls_comm_create_nccl", "cparls_comm_create_local",
            "cparls_comm_destroy", "cparls_plan_rows", "cparls_owned_rows", "cparls_opts_init",
            "cparls_route_nonzeros"]


def _ptr(x):
    """Raw pointer of a numpy array or torch tensor (host or device)."""
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        assert x.flags["C_CONTIGUOUS"]
        return x.ctypes.data
    return x.data_ptr()   # torch.Tensor (contiguous, checked by caller)


class Cparls:
    """One CP-ARLS-LEV context (the C ABI's cparls_ctx)."""

    def __init__(self, dims, coords, vals, rank, tau=-1.0, init_seed=2, stream=None,
                 didx_cap=0, attempt_cap=0, comm=None, world_size=1, world_rank=0, rhs_path=0,
                 fit_samples=0, fit_alpha=0.5, fit_seed=0, sidx_window=0, sample_sort=0, fit_mode=-1,
                 rhs_hot_rows=-1):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("cparls needs a CUDA device (B200); no CPU fallback exists")
        L = lib()
        self.dims = tuple(int(d) for d in dims)
        self.D = len(self.dims)
        self.r = int(rank)
        self._keep = []
        if isinstance(coords, np.ndarray):
            coords = np.ascontiguousarray(coords)
            vals = np.ascontiguousarray(vals)
            idt = 1 if coords.dtype == np.int64 else 0
            vdt = 1 if vals.dtype == np.float32 else 0
            assert coords.dtype in (np.int32, np.int64) and vals.dtype in (np.float32, np.float64)
        else:
            coords = coords.contiguous()
            vals = vals.contiguous()
            idt = 1 if coords.dtype == torch.int64 else 0
            vdt = 1 if vals.dtype == torch.float32 else 0
            assert coords.dtype in (torch.int32, torch.int64) and vals.dtype in (torch.float32, torch.float64)
        nnz = int(coords.shape[0]) if coords.ndim else 0
        if stream is None:
            stream = torch.cuda.current_stream().cuda_stream
        self.stream = stream
        o = Opts(struct_size=C.sizeof(Opts), rank=self.r, tau=float(tau), value_dtype=vdt, index_dtype=idt,
                 stream=C.c_void_p(stream), world_size=int(world_size), world_rank=int(world_rank),
                 comm=(comm.handle if comm is not None else None),
                 didx_cap=int(didx_cap), attempt_cap=int(attempt_cap), rhs_path=int(rhs_path),
                 fit_samples=int(fit_samples), fit_alpha=float(fit_alpha), fit_seed=int(fit_seed),
                 sidx_window=int(sidx_window), sample_sort=int(sample_sort), fit_mode=int(fit_mode),
                 rhs_hot_rows=int(rhs_hot_rows))
        d = np.array(self.dims, dtype=np.int64)
        h = C.c_void_p()
        st = L.cparls_create(C.byref(h), self.D, d.ctypes.data, nnz, _ptr(coords), _ptr(vals),
                             C.byref(o), int(init_seed))
        if st != OK:
            raise CparlsError(st, L.cparls_last_error(None).decode())
        self._h = h

    # ------------------------------------------------------------------
    def _check(self, st):
        if st != OK:
            raise CparlsError(st, lib().cparls_last_error(self._h).decode())

    def close(self):
        if getattr(self, "_h", None):
            lib().cparls_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_factor(self, k, A):
        A = np.ascontiguousarray(A, dtype=np.float64)
        assert A.shape == (self.dims[k], self.r)
        self._check(lib().cparls_set_factor(self._h, k, A.ctypes.data))

    def get_factor(self, k, out=None, lam_out=None):
        """Factor k (n_k x r fp64) and lambda.  out / lam_out: optional caller
        arrays (C-contiguous fp64; e.g. numpy views of pinned torch tensors,
        which the library copies into without staging)."""
        A = np.zeros((self.dims[k], self.r)) if out is None else out
        lam = np.zeros(self.r) if lam_out is None else lam_out
        if A.shape != (self.dims[k], self.r) or A.dtype != np.float64 or not A.flags.c_contiguous:
            raise ValueError("out must be a C-contiguous float64 array of shape (n_k, r)")
        if lam.shape != (self.r,) or lam.dtype != np.float64 or not lam.flags.c_contiguous:
            raise ValueError("lam_out must be a C-contiguous float64 array of shape (r,)")
        self._check(lib().cparls_get_factor(self._h, k, A.ctypes.data, lam.ctypes.data))
        return A, lam

    def leverage(self, k):
        ell = np.zeros(self.dims[k])
        rank = C.c_int32()
        self._check(lib().cparls_leverage(self._h, k, ell.ctypes.data, C.byref(rank)))
        return ell, rank.value

    def get_ptilde(self, k):
        pt = np.zeros(self.dims[k])
        self._check(lib().cparls_get_ptilde(self._h, k, pt.ctypes.data))
        return pt

    def set_ptilde(self, k, pt):
        pt = np.ascontiguousarray(pt, dtype=np.float64)
        self._check(lib().cparls_set_ptilde(self._h, k, pt.ctypes.data))

    def set_tau(self, tau):
        self._check(lib().cparls_set_tau(self._h, float(tau)))

    def sample(self, k, s, seed, step):
        info = SampleInfo()
        self._check(lib().cparls_sample(self._h, k, int(s), int(seed), int(step), C.byref(info)))
        return info

    def get_sample(self):
        n = C.c_int64()
        self._check(lib().cparls_get_sample(self._h, 0, None, None, None, None, None, C.byref(n)))
        n = n.value
        keys = np.zeros(n, dtype=np.uint64); cnt = np.zeros(n, dtype=np.int32)
        w2 = np.zeros(n); p = np.zeros(n); isdet = np.zeros(n, dtype=np.uint8)
        m = C.c_int64()
        self._check(lib().cparls_get_sample(self._h, n, keys.ctypes.data, cnt.ctypes.data,
                                            w2.ctypes.data, p.ctypes.data, isdet.ctypes.data,
                                            C.byref(m)))
        return dict(keys=keys, counts=cnt, w2=w2, p=p, is_det=isdet.astype(bool))

    def get_fibers(self):
        n = C.c_int64()
        self._check(lib().cparls_get_sample(self._h, 0, None, None, None, None, None, C.byref(n)))
        lens = np.zeros(n.value, dtype=np.int64)
        mk = C.c_int64()
        self._check(lib().cparls_get_fibers(self._h, 0, lens.ctypes.data, None, None, C.byref(mk)))
        out = np.zeros(mk.value, dtype=np.int64); val = np.zeros(mk.value)
        self._check(lib().cparls_get_fibers(self._h, mk.value, lens.ctypes.data, out.ctypes.data,
                                            val.ctypes.data, C.byref(mk)))
        return lens, out, val

    def get_fiber_lengths(self):
        """Per-sample fiber lengths of the current sample (canonical order)."""
        n = C.c_int64()
        self._check(lib().cparls_get_sample(self._h, 0, None, None, None, None, None, C.byref(n)))
        lens = np.zeros(n.value, dtype=np.int64)
        mk = C.c_int64()
        self._check(lib().cparls_get_fibers(self._h, 0, lens.ctypes.data, None, None, C.byref(mk)))
        return lens

    def solve_mode(self, k):
        info = SolveInfo()
        self._check(lib().cparls_solve_mode(self._h, k, C.byref(info)))
        return info

    def last_solve(self, k):
        G = np.zeros((self.r, self.r)); B = np.zeros((self.dims[k], self.r))
        self._check(lib().cparls_get_last_solve(self._h, G.ctypes.data, B.ctypes.data))
        return G, B

    def fit(self):
        f = C.c_double()
        self._check(lib().cparls_fit(self._h, C.byref(f)))
        return f.value

    def fit_estimate(self):
        """Estimated fit over the frozen stratified sample: (fit, F^)."""
        f, F = C.c_double(), C.c_double()
        self._check(lib().cparls_fit_estimate(self._h, C.byref(f), C.byref(F)))
        return f.value, F.value

    def get_fit_sample(self):
        n = C.c_int64()
        self._check(lib().cparls_get_fit_sample(self._h, 0, None, None, None, C.byref(n)))
        m = n.value
        coords = np.zeros((m, self.D), dtype=np.int64); x = np.zeros(m); nz = np.zeros(m, dtype=np.uint8)
        self._check(lib().cparls_get_fit_sample(self._h, m, coords.ctypes.data, x.ctypes.data, nz.ctypes.data,
                                                C.byref(n)))
        return coords, x, nz.astype(bool)

    def fit_sample_model(self):
        """m_i of the current model at every fit-sample position (diagnostics)."""
        n = C.c_int64()
        self._check(lib().cparls_get_fit_sample(self._h, 0, None, None, None, C.byref(n)))
        m = np.zeros(n.value)
        self._check(lib().cparls_fit_sample_model(self._h, m.ctypes.data))
        return m

    def run_until(self, s, seed, eta=5, pi=3, tol=1e-4, max_epochs=50, estimated=False):
        """Alg. 3 with its stopping rule (AMB-33): the per-epoch fit trace."""
        trace = np.full(max(max_epochs, 1), np.nan)
        ep = C.c_int32()
        self._check(lib().cparls_run_until(self._h, int(s), int(seed), int(eta), int(pi), float(tol),
                                           int(max_epochs), 1 if estimated else 0, trace.ctypes.data,
                                           C.byref(ep)))
        return trace[:ep.value]

    def init_rrf(self, s_init, seed=0):
        """Randomized range finder initialization of every factor (AMB-34)."""
        self._check(lib().cparls_init_rrf(self._h, int(s_init), int(seed)))

    def als_update(self, k):
        """One exact CP-ALS mode update."""
        self._check(lib().cparls_als_update(self._h, int(k)))

    def run_als(self, iters, fit_every=1):
        trace = np.full(max(iters, 1), np.nan)
        self._check(lib().cparls_run_als(self._h, int(iters), int(fit_every), trace.ctypes.data))
        return trace[:iters]

    def run(self, iters, s, seed, iter0=0, fit_every=1):
        trace = np.full(max(iters, 1), np.nan)
        self._check(lib().cparls_run(self._h, int(iters), int(s), int(seed), int(iter0),
                                     int(fit_every), trace.ctypes.data))
        return trace[:iters]

    def owned_rows(self, k):
        lo, hi = C.c_int64(), C.c_int64()
        self._check(lib().cparls_owned_rows(self._h, k, C.byref(lo), C.byref(hi)))
        return lo.value, hi.value

    def stats(self):
        s = Stats()
        self._check(lib().cparls_get_stats(self._h, C.byref(s), C.sizeof(s)))
        return s.as_dict()

    def reset_stats(self):
        self._check(lib().cparls_reset_stats(self._h))

    def set_profiling(self, on=True):
        self._check(lib().cparls_set_profiling(self._h, 1 if on else 0))


class Comm:
    """A cparls_comm: NCCL (one process per GPU) or an in-process local group
    (shard simulator: world_size shards on the current GPU, one host thread
    each)."""

    def __init__(self, handle, kind):
        self.handle = handle
        self.kind = kind

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        st = lib().cparls_comm_nccl_unique_id(buf)
        if st != OK:
            raise CparlsError(st, "ncclGetUniqueId failed")
        return bytes(buf)

    @classmethod
    def nccl(cls, world_size, rank, uid: bytes):
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        h = C.c_void_p()
        st = lib().cparls_comm_create_nccl(int(world_size), int(rank), buf, C.byref(h))
        if st != OK:
            raise CparlsError(st, "ncclCommInitRank failed")
        return cls(h, "nccl")

    @classmethod
    def local(cls, world_size):
        h = C.c_void_p()
        st = lib().cparls_comm_create_local(int(world_size), C.byref(h))
        if st != OK:
            raise CparlsError(st, "local group creation failed")
        return cls(h, "local")

    def close(self):
        if self.handle:
            lib().cparls_comm_destroy(self.handle)
            self.handle = None


def plan_rows(deg, world_size, with_heavy=False):
    """Row blocks (world_size + 1 bounds) balanced by the per-row counts deg
    (host-only library call; cparls_plan_rows); with_heavy also returns the
    heavy-row flags (rows whose nonzeros are spread over all ranks)."""
    deg = np.ascontiguousarray(deg, dtype=np.uint64)
    bound = np.zeros(int(world_size) + 1, dtype=np.int64)
    heavy = np.zeros(len(deg), dtype=np.uint8)
    st = lib().cparls_plan_rows(len(deg), deg.ctypes.data, int(world_size), bound.ctypes.data, heavy.ctypes.data)
    if st != OK:
        raise CparlsError(st, "plan_rows")
    return (bound, heavy.astype(bool)) if with_heavy else bound


def route_nonzeros(coords, mode, world_size, bound, heavy=None):
    """Rank of each nonzero in the sharded build of `mode` (host-only library
    call; cparls_route_nonzeros): the row owner, or a hash for heavy rows."""
    coords = np.ascontiguousarray(coords, dtype=np.int64)
    bound = np.ascontiguousarray(bound, dtype=np.int64)
    hv = None if heavy is None else np.ascontiguousarray(heavy, dtype=np.uint8)
    out = np.zeros(coords.shape[0], dtype=np.int32)
    st = lib().cparls_route_nonzeros(coords.shape[1], int(mode), coords.shape[0], coords.ctypes.data,
                                     int(world_size), bound.ctypes.data, None if hv is None else hv.ctypes.data,
                                     out.ctypes.data)
    if st != OK:
        raise CparlsError(st, "route_nonzeros")
    return out


def version():
    return lib().cparls_version().decode()
