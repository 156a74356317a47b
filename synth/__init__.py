"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the CPU oracle.

This module holds NONE of CP-ARLS-LEV's arithmetic (no leverage, no sampling of
KRP rows, no solve).  It only manufactures sparse COO tensors with the shapes,
nonzero counts and value types of the paper's workloads (PAPER.md:1007-1027,
Table 6.1) and the planted tiny case of BASELINE.json configs[0].  The FROSTT
tensors themselves are not available; these seeded Zipf tensors stand in for
them.

Everything is integer arithmetic on int64 torch tensors (Philox4x32-10 with
16-bit partial products so nothing overflows, inverse-CDF draws by
``searchsorted`` on exact integer tables), so the same call produces the same
bytes on CPU and on CUDA.  Floating point enters only through host-side tables
(Zipf pmf, log(1+c) values) built once with numpy and through the tiny C1
planted values, which are always built on the CPU.
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional, Sequence

import numpy as np
import torch

M32 = 0xFFFFFFFF
_PH_M0 = 0xD2511F53
_PH_M1 = 0xCD9E8D57
_PH_W0 = 0x9E3779B9
_PH_W1 = 0xBB67AE85

TWO62 = 1 << 62


# --------------------------------------------------------------------------
# Philox4x32-10 on int64 tensors (values kept in [0, 2^32)).
# --------------------------------------------------------------------------
def _mulhilo(a: torch.Tensor, m: int):
    """(hi, lo) 32-bit halves of a*m for a in [0,2^32), m a 32-bit constant."""
    m_lo = m & 0xFFFF
    m_hi = m >> 16
    p1 = a * m_lo                      # < 2^48
    t = a * m_hi + (p1 >> 16)          # < 2^49
    hi = t >> 16
    lo = ((t & 0xFFFF) << 16) | (p1 & 0xFFFF)
    return hi, lo


def philox4x32_10(c0, c1, c2, c3, k0: int, k1: int):
    """Philox4x32 with 10 rounds (Salmon et al. 2011).  Counters are int64
    tensors (or ints broadcastable to them) holding 32-bit values."""
    dev = c0.device if isinstance(c0, torch.Tensor) else None
    shape = None
    for c in (c0, c1, c2, c3):
        if isinstance(c, torch.Tensor):
            shape = c.shape
            dev = c.device
    def t(x):
        if isinstance(x, torch.Tensor):
            return x.to(torch.int64)
        return torch.full(shape, int(x), dtype=torch.int64, device=dev)
    x0, x1, x2, x3 = t(c0), t(c1), t(c2), t(c3)
    ka, kb = k0 & M32, k1 & M32
    for r in range(10):
        if r > 0:
            ka = (ka + _PH_W0) & M32
            kb = (kb + _PH_W1) & M32
        hi0, lo0 = _mulhilo(x0, _PH_M0)
        hi1, lo1 = _mulhilo(x2, _PH_M1)
        x0, x1, x2, x3 = hi1 ^ x1 ^ ka, lo1, hi0 ^ x3 ^ kb, lo0
    return x0, x1, x2, x3


def _word62(lo32: torch.Tensor, hi32: torch.Tensor) -> torch.Tensor:
    """Top 62 bits of the 64-bit word (hi<<32|lo): a uniform integer in [0,2^62)."""
    return (hi32 << 30) | (lo32 >> 2)


def _word53(lo32: torch.Tensor, hi32: torch.Tensor) -> torch.Tensor:
    return (hi32 << 21) | (lo32 >> 11)


# --------------------------------------------------------------------------
# Integer inverse-CDF tables
# --------------------------------------------------------------------------
def int_cdf_from_pmf(pmf: np.ndarray) -> np.ndarray:
    """Inclusive integer CDF with total exactly 2^62 (rounding slack put on
    the largest entry).  Returned as int64 numpy array."""
    pmf = np.asarray(pmf, dtype=np.float64)
    pmf = pmf / pmf.sum()
    q = np.rint(np.ldexp(pmf, 62)).astype(np.int64)
    q[int(np.argmax(q))] += TWO62 - int(q.sum(dtype=np.int64))
    assert int(q.sum(dtype=np.int64)) == TWO62 and (q >= 0).all()
    return np.cumsum(q, dtype=np.int64)


def zipf_cdf(n: int, alpha: float) -> np.ndarray:
    ranks = np.arange(1, n + 1, dtype=np.float64)
    return int_cdf_from_pmf(ranks ** (-alpha))


def uniform_cdf(n: int) -> np.ndarray:
    return int_cdf_from_pmf(np.ones(n))


def geometric_table(p: float, gmax: int = 200) -> np.ndarray:
    """Ascending thresholds so that G = searchsorted(T, u, right=True) for a
    uniform u in [0,2^62) gives P(G >= g) = (1-p)^g (Geometric on {0,1,..})."""
    g = np.arange(gmax, 0, -1, dtype=np.float64)              # gmax..1
    thr = np.floor(np.ldexp((1.0 - p) ** g, 62)).astype(np.int64)
    # P(G >= g) = P(u < thr_g); G = #{g : u < thr_g}.  Use ascending table of
    # thresholds: G = #entries > u = len - searchsorted(right=True).
    return thr  # ascending (small g last => largest threshold last)


def _permutation(n: int, seed: int, mode: int, device) -> torch.Tensor:
    """Seeded random permutation (rank -> index), AMB-25: argsort of Philox
    hashes of 0..n-1 (stable, so ties cannot make it device dependent)."""
    i = torch.arange(n, dtype=torch.int64, device=device)
    x0, x1, _, _ = philox4x32_10(i & M32, i >> 32, 0x9E77, mode, seed, 0x5045524D)
    h = (x1 << 31) | (x0 >> 1)                                # 63-bit, >= 0
    return torch.argsort(h, stable=True)


# --------------------------------------------------------------------------
# Configs (BASELINE.json configs[0..4])
# --------------------------------------------------------------------------
@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    dims: tuple
    nnz: int
    alpha: Optional[float]        # Zipf exponent; None = uniform cells (C1)
    value: str                    # 'planted', 'geom', 'loggeom'
    geom_p: float
    value_dtype: str              # 'f64' or 'f32'
    rank: int
    s: int
    iters: int
    coord_seed: int = 0
    value_seed: int = 1
    init_seed: int = 2
    sample_seed: int = 3


CONFIGS = {
    # configs[0]: planted rank-3, 2000 distinct uniform cells
    "C1": Config("C1", (30, 40, 50), 2000, None, "planted", 0.0, "f64", 3, 256, 20),
    # configs[1]: Uber-shaped
    "C2": Config("C2", (183, 24, 1140, 1717), 3_309_490, 1.1, "geom", 0.5, "f64", 25, 1 << 17, 20),
    # configs[2]: Enron-shaped
    "C3": Config("C3", (6066, 5699, 244268, 1176), 54_202_099, 1.2, "geom", 0.3, "f64", 25, 1 << 17, 20),
    # configs[3]: Amazon-shaped, fp32 values
    "C4": Config("C4", (4_821_207, 1_774_269, 1_805_187), 1_741_809_018, 1.1, "geom", 0.5, "f32", 25, 1 << 17, 10),
    # configs[4]: Reddit-shaped, log(1+c) values, fp32
    "C5": Config("C5", (8_211_298, 176_962, 8_116_559), 4_687_474_081, 1.2, "loggeom", 0.4, "f32", 25, 1 << 17, 10),
}


def packed_key_layout(dims: Sequence[int]):
    """Bit layout of the 64-bit dedup key: mixed radix of modes 0..D-2 in the
    low `lo_bits`, last mode above it.  Returns lo_bits."""
    prod = 1
    for n in dims[:-1]:
        prod *= int(n)
    lo_bits = max(1, (prod - 1).bit_length())
    hi_bits = max(1, (int(dims[-1]) - 1).bit_length())
    if lo_bits + hi_bits > 64:
        raise ValueError("tensor too large for 64-bit packed keys")
    return lo_bits


def _pack(coords: List[torch.Tensor], dims, lo_bits):
    lo = torch.zeros_like(coords[0])
    mult = 1
    for c, n in zip(coords[:-1], dims[:-1]):
        lo = lo + c * mult
        mult *= int(n)
    return lo | (coords[-1] << lo_bits)


def _unpack(keys: torch.Tensor, dims, lo_bits):
    lo = keys & ((1 << lo_bits) - 1)
    hi = (keys >> lo_bits) & ((1 << (64 - lo_bits)) - 1)   # logical shift
    out = []
    for n in dims[:-1]:
        out.append(lo % int(n))
        lo = lo // int(n)
    out.append(hi)
    return out


def _draw_coords(first: int, count: int, cdfs, perms, seed: int, device):
    """Coordinates of draws [first, first+count): slot j uses Philox lane j//2,
    64-bit word j%2 of that lane (counter = (draw lo, draw hi, 0x5A1F, lane))."""
    D = len(cdfs)
    a = torch.arange(first, first + count, dtype=torch.int64, device=device)
    lo, hi = a & M32, a >> 32
    out = []
    lanes = {}
    for j in range(D):
        lane = j // 2
        if lane not in lanes:
            lanes[lane] = philox4x32_10(lo, hi, 0x5A1F, lane, seed, 0x5A1F0000)
        x = lanes[lane]
        w = j % 2
        u = _word62(x[2 * w], x[2 * w + 1])
        r = torch.searchsorted(cdfs[j], u, right=True)
        out.append(perms[j][r] if perms[j] is not None else r)
    return out


_NB = 8           # dedup buckets (key & 7): keeps every sort below torch's INT_MAX limit
_CH = 1 << 30     # scan chunk for first-occurrence selection


def _first_unique_positions(parts, total, target, device):
    """Positions (ascending) of the first `target` distinct keys by first
    occurrence, from draw-ordered key chunks.  Returns None if fewer exist."""
    first = torch.zeros(total, dtype=torch.bool, device=device)
    for b in range(_NB):
        ks, ps = [], []
        base = 0
        for k in parts:
            m = (k & (_NB - 1)) == b
            ks.append(k[m])
            ps.append(torch.nonzero(m).squeeze(1) + base)
            base += k.numel()
        kb = torch.cat(ks)
        pb = torch.cat(ps)
        del ks, ps
        if kb.numel() == 0:
            continue
        sk, order = torch.sort(kb, stable=True)
        f = torch.ones_like(sk, dtype=torch.bool)
        f[1:] = sk[1:] != sk[:-1]
        first[pb[order[f]]] = True
        del kb, pb, sk, order, f
    out, have = [], 0
    for c0 in range(0, total, _CH):
        idx = torch.nonzero(first[c0:c0 + _CH]).squeeze(1) + c0
        take = min(idx.numel(), target - have)
        out.append(idx[:take])
        have += take
        if have >= target:
            break
    if have < target:
        return None
    return torch.cat(out)


def generate_coords(cfg: Config, device="cpu", chunk: int = 1 << 27, out_dtype=torch.int64, part: int = 0,
                    parts: int = 1) -> torch.Tensor:
    """nnz x D int64 coordinates (0-based), distinct, in first-draw order.
    parts > 1: only the cells at first-draw positions part, part + parts, ...
    (a rank's chunk of the same tensor; the draws and the dedup are the same
    on every rank, only the materialized coordinates are 1/parts)."""
    dims = cfg.dims
    D = len(dims)
    lo_bits = packed_key_layout(dims)
    cdfs, perms = [], []
    for m, n in enumerate(dims):
        if cfg.alpha is None:
            c = uniform_cdf(n)
            perms.append(None)
        else:
            c = zipf_cdf(n, cfg.alpha)
            perms.append(_permutation(n, cfg.coord_seed, m, device))
        cdfs.append(torch.from_numpy(c).to(device))
    target = cfg.nnz
    total = int(target * 1.05) + 64
    keys = []
    drawn = 0
    while True:
        while drawn < total:
            cnt = min(chunk, total - drawn)
            cs = _draw_coords(drawn, cnt, cdfs, perms, cfg.coord_seed, device)
            keys.append(_pack(cs, dims, lo_bits))
            del cs
            drawn += cnt
        pos = _first_unique_positions(keys, drawn, target, device)
        if pos is not None:
            break
        total = int(total * 1.25) + 1024
    if parts > 1:   # this rank's chunk: every parts-th cell in first-draw order
        pos = pos[part::parts].contiguous()
    target = pos.numel()
    # gather the selected keys chunk by chunk (positions ascending)
    sel = torch.empty(target, dtype=torch.int64, device=device)
    base = 0
    for k in keys:
        n = k.numel()
        lo_i = torch.searchsorted(pos, torch.tensor([base, base + n], device=device))
        a_, b_ = int(lo_i[0]), int(lo_i[1])
        sel[a_:b_] = k[pos[a_:b_] - base]
        base += n
    del keys, pos
    out = torch.empty((target, D), dtype=out_dtype, device=device)
    for c0 in range(0, target, chunk):
        cs = _unpack(sel[c0:c0 + chunk], dims, lo_bits)
        out[c0:c0 + chunk] = torch.stack(cs, dim=1).to(out_dtype)
    return out


def _uniform53(c0, c1, c2, c3, seed):
    x = philox4x32_10(c0, c1, c2, c3, seed, 0x55AA)
    return _word53(x[0], x[1]).to(torch.float64) * (2.0 ** -53), x


def planted_factors(cfg: Config, seed: int):
    """U[0,1) factors, entry (m, i, c) from Philox(counter=(i, c, m, 0x9A47))."""
    out = []
    for m, n in enumerate(cfg.dims):
        i = torch.arange(n, dtype=torch.int64).repeat_interleave(cfg.rank)
        c = torch.arange(cfg.rank, dtype=torch.int64).repeat(n)
        u, _ = _uniform53(i, c, m, 0x9A47, seed)
        out.append(u.reshape(n, cfg.rank))
    return out


def uniform_init(dims, rank, seed, device="cpu"):
    """Initial factors U[0,1) (AMB-21), same construction as planted_factors."""
    out = []
    for m, n in enumerate(dims):
        i = torch.arange(n, dtype=torch.int64, device=device).repeat_interleave(rank)
        c = torch.arange(rank, dtype=torch.int64, device=device).repeat(n)
        u, _ = _uniform53(i, c, m, 0x1417, seed)
        out.append(u.reshape(n, rank))
    return out


def generate_values(cfg: Config, coords: torch.Tensor, chunk: int = 1 << 27) -> torch.Tensor:
    device = coords.device
    dims = cfg.dims
    if cfg.value == "planted":
        assert device.type == "cpu", "planted values are built on the CPU"
        facs = planted_factors(cfg, cfg.value_seed)
        v = torch.ones(coords.shape[0], cfg.rank, dtype=torch.float64)
        for m in range(len(dims)):
            v = v * facs[m][coords[:, m]]
        v = v.sum(dim=1)
        # N(0, sigma=1e-4) noise (AMB-23) by Box-Muller on separate lane
        n = coords.shape[0]
        j = torch.arange(n, dtype=torch.int64)
        x = philox4x32_10(j, 0, 0x40153, 1, cfg.value_seed, 0x4E4F)
        u1 = (_word53(x[0], x[1]).to(torch.float64) + 1.0) * (2.0 ** -53)   # (0,1]
        u2 = _word53(x[2], x[3]).to(torch.float64) * (2.0 ** -53)
        z = torch.sqrt(-2.0 * torch.log(u1)) * torch.cos(2.0 * math.pi * u2)
        return v + 1e-4 * z
    lo_bits = packed_key_layout(dims)
    thr = torch.from_numpy(geometric_table(cfg.geom_p)).to(device)
    tab = None
    if cfg.value == "loggeom":   # fp32(log(1+c)) from a host table (no device libm)
        tab = torch.tensor([math.log1p(float(k)) for k in range(thr.numel() + 2)],
                           dtype=torch.float64).to(device)
    out_dtype = torch.float32 if cfg.value_dtype == "f32" else torch.float64
    out = torch.empty(coords.shape[0], dtype=out_dtype, device=device)
    for c0 in range(0, coords.shape[0], chunk):
        cc = coords[c0:c0 + chunk].to(torch.int64)
        keys = _pack([cc[:, m] for m in range(len(dims))], dims, lo_bits)
        x = philox4x32_10(keys & M32, (keys >> 32) & M32, 0x7A1E, 0, cfg.value_seed, 0x7A1E0000)
        u = _word62(x[0], x[1])
        g = thr.numel() - torch.searchsorted(thr, u, right=True)      # #thr > u
        c = 1 + g
        vals = c.to(torch.float64) if tab is None else tab[c]
        out[c0:c0 + chunk] = vals.to(out_dtype)
    return out


@dataclasses.dataclass
class Tensor:
    cfg: Config
    dims: tuple
    coords: torch.Tensor     # nnz x D int64 (or int32 if requested)
    vals: torch.Tensor


def make(name_or_cfg, device="cpu", index_dtype=torch.int32, dense_planted=False, part: int = 0,
         parts: int = 1) -> Tensor:
    """The config's tensor; parts > 1 gives rank `part`'s chunk of it (cells
    part, part + parts, ... in first-draw order) without materializing the
    rest (multi-GPU bench: every rank builds only its share)."""
    cfg = CONFIGS[name_or_cfg] if isinstance(name_or_cfg, str) else name_or_cfg
    if dense_planted:
        # fully populated C1 variant for the recovery invariant (AMB-24)
        grids = torch.meshgrid(*[torch.arange(n) for n in cfg.dims], indexing="ij")
        coords = torch.stack([g.reshape(-1) for g in grids], dim=1).to(torch.int64)
        cfg = dataclasses.replace(cfg, nnz=coords.shape[0])
    else:
        coords = generate_coords(cfg, device=device, out_dtype=index_dtype, part=part, parts=parts)
    vals = generate_values(cfg, coords)
    if coords.dtype != index_dtype:
        out = torch.empty(coords.shape, dtype=index_dtype, device=coords.device)
        for c0 in range(0, coords.shape[0], 1 << 27):
            out[c0:c0 + (1 << 27)] = coords[c0:c0 + (1 << 27)].to(index_dtype)
        del coords
        coords = out
    return Tensor(cfg, tuple(cfg.dims), coords, vals)


def scaled(cfg_name: str, nnz: int, dims=None, **kw) -> Config:
    """A smaller instance of a config (same generator), for fast tests."""
    base = CONFIGS[cfg_name]
    return dataclasses.replace(base, name=f"{cfg_name}-small", nnz=nnz,
                               dims=tuple(dims) if dims else base.dims, **kw)
