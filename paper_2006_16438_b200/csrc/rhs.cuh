// rhs.cuh -- K8 sampled right-hand side M = Xs^T diag(w^2) Z_S (P:949-958,
// AMB-14): M(out_e,:) += w_j^2 x_e z_j for every matched nonzero e of every
// sampled fiber j.
//
// Warps walk the concatenated matched entries (fiber after fiber, so z_j stays
// in registers across a fiber); lanes = columns, so one entry is one r-wide
// reduction into M's row: int64 fixed point by default (AMB-35: z_j is
// pre-scaled by 2^e_c, one rounding per term, order-free sums), fp64 `red`
// with rhs_path 3 or when the scales are out of range.  The L2's reduction
// rate bounds this kernel: bench.py measures it for k_rhs's own row stream
// (cparls_peak_red_idx) and k_rhs runs at ~100% of it.  Entries reach the
// lanes through a per-warp shared buffer (one 16-byte broadcast load per
// entry); addresses are one IMAD.WIDE.U32 from a per-lane column base.
// (Privatizing the heaviest rows in shared memory was measured and dropped:
// the top 64 rows hold < 1% of the entries on the Zipf workloads, and shared
// atomics on spread addresses are no faster than L2 reductions.)
//
// M (n_k x ld) is far larger than L2 for the big modes, so random reductions
// would each be a DRAM read-modify-write.  The entries are therefore visited
// in output-row windows of ~96 MB of M: each fiber is sorted by output row, so
// its entries inside window w are the sub-range found by k_win_bounds; the
// (window, fiber) segments are concatenated window-major and warps take
// chunks from a global counter, so the rows being reduced stay in L2.
#pragma once
#include <algorithm>

#include "common.cuh"

namespace cparls {

constexpr int kRhsThreads = 256;

// One matched entry as the warp shares it: w_j^2 x_e, its output row and its
// sample.  Lanes publish their entries to a per-warp shared buffer once per
// 32-entry group and every lane reads entry u with one 16-byte broadcast load
// (three shuffles per entry before).
struct RhsEnt {
  double cx;
  int32_t o;
  int32_t j;
};

// FX: int64 fixed point, zs = z * 2^e_c (exact power-of-two scaling), one
// rounding to the integer per term; else fp64 reductions of cx * z.  The
// reduction is predicated (no branch per lane); addr already holds the lane's
// column.
template <bool FX>
__device__ __forceinline__ void rhs_red(char *addr, double cx, double zs, unsigned on) {
  if (FX) {
    const long long q = __double2ll_rn(cx * zs);
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p red.global.add.u64 [%0], %1;\n\t}"
                 :: "l"(addr), "l"(q), "r"(on) : "memory");
  } else {
    const double v = cx * zs;
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p red.global.add.f64 [%0], %1;\n\t}"
                 :: "l"(addr), "d"(v), "r"(on) : "memory");
  }
}

// Hot rows (round 2).  A Zipf head row holds 8-24% of a C2/C3 mode's
// nonzeros, so its entries' reductions pile up on the same L2 addresses,
// where they serialize.  The HOT variant sums the entries of the mode's hot
// rows (the H rows of largest degree, chosen at create; all rows when n_k <= H)
// per CTA in shared memory and adds each CTA's nonzero partial rows to M once
// at the end.  An int64 accumulator is two 32-bit words (shared 64-bit atomics
// are a CAS loop): the low word's atomic add returns the old value, so each
// carry into the high word is exact and the pair holds the same sum modulo
// 2^64 as the L2 reductions: M is bit-identical with or without hot rows.
struct HotAcc {
  uint32_t *lo, *hi;   // [H][r] words in shared memory
  int r;
};

__device__ __forceinline__ void hot_add(const HotAcc &h, int slot, int lane, double cx, double zs, unsigned on) {
  if (!on) return;
  const unsigned long long q = (unsigned long long)__double2ll_rn(cx * zs);
  const uint32_t qlo = (uint32_t)q, qhi = (uint32_t)(q >> 32);
  const int i = slot * h.r + lane;
  const uint32_t old = atomicAdd(h.lo + i, qlo);
  atomicAdd(h.hi + i, qhi + (uint32_t)(old + qlo < old));
}

template <typename VT, bool HI, bool FX, bool HOT = false>
__device__ __forceinline__ void rhs_body(const int64_t *__restrict__ off, const int64_t *__restrict__ lo,
                                         const int32_t *__restrict__ seg_j, int64_t nseg, int64_t mk,
                                         unsigned long long *__restrict__ work, const int32_t *__restrict__ outidx,
                                         const VT *__restrict__ vals, const double *__restrict__ sw2,
                                         const double *__restrict__ Z, int r, int ld, double *__restrict__ M,
                                         int64_t per_warp, double sc0, double sc1, RhsEnt *we,
                                         const int32_t *__restrict__ hot_slot = nullptr, HotAcc hacc = {}) {
  const int lane = threadIdx.x & 31;
  const uint64_t pstream = l2_evict_first();
  {
    // chunk size from m_k (on the device): about 4 chunks per warp, a multiple
    // of 32 in [32, per_warp].  A warp's groups run one after another (each
    // waits on its index loads), so small m_k (C2/C3) needs small chunks to
    // spread over every warp; large m_k keeps per_warp (fewer chunk searches).
    const int64_t nw4 = 4 * (int64_t)gridDim.x * (blockDim.x >> 5);
    const int64_t pw = ((mk + nw4 - 1) / nw4 + 31) & ~int64_t(31);
    per_warp = max((int64_t)32, min(per_warp, pw));
  }
  // row address = lane's column base + out * row bytes (one IMAD.WIDE.U32)
  char *const Mb0 = reinterpret_cast<char *>(M + lane);
  char *const Mb1 = reinterpret_cast<char *>(M + lane + 32);
  const uint32_t rowb = (uint32_t)ld * 8u;
  const unsigned on0 = lane < r, on1 = HI && lane + 32 < r;
  while (true) {
    int64_t t0 = 0;
    if (lane == 0) t0 = (int64_t)atomicAdd(work, (unsigned long long)per_warp);
    t0 = __shfl_sync(0xffffffffu, t0, 0);
    if (t0 >= mk) break;
    const int64_t t1 = min(mk, t0 + per_warp);
    // segment containing entry t0: last g with off[g] <= t0 (off[0] = 0),
    // 32-ary search (one coalesced probe per level; empty segments share
    // their successor's offset and are skipped)
    int64_t a = 0, b = nseg;   // answer in [a, b)
    while (b - a > 1) {
      const int64_t step = (b - a + 31) >> 5;
      const int64_t g = a + (int64_t)lane * step;
      const bool le = g < b && __ldg(off + g) <= t0;
      const int c = __popc(__ballot_sync(0xffffffffu, le));   // >= 1: lane 0 probes a
      b = min(b, a + (int64_t)c * step);
      a += (int64_t)(c - 1) * step;
    }
    int64_t jcur = a;       // segment of the first entry of the current 32-group
    int32_t jz = -1;        // sample whose (scaled) z row is loaded
    double z0 = 0.0, z1 = 0.0;
    for (int64_t t = t0; t < t1; t += 32) {
      const int64_t tmax = min(t + 31, t1 - 1);
      const int64_t tt = min(t + lane, tmax);
      const bool valid = t + lane < t1;
      // this lane's segment: last g with off[g] <= tt, found 32 segment
      // starts per coalesced load (runs of empty fibers cost one load per 32)
      int64_t jj = jcur;
      for (int64_t jb = jcur;; jb += 32) {
        const int64_t g = jb + 1 + lane;
        const int64_t og = g < nseg ? __ldg(off + g) : INT64_MAX;
        int c = 0;   // #{k < 32 : og_k <= tt} (og ascending over the lanes)
#pragma unroll
        for (int stp = 16; stp >= 1; stp >>= 1)
          if (__shfl_sync(0xffffffffu, og, c + stp - 1) <= tt) c += stp;
        const int64_t last = __shfl_sync(0xffffffffu, og, 31);
        if (last <= tt) c = 32;
        if (c > 0) jj = jb + c;
        if (last > tmax) break;
      }
      RhsEnt me = {0.0, 0, -1};
      if (valid) {
        me.j = seg_j ? __ldg(seg_j + jj) : (int32_t)jj;
        const int64_t e = __ldg(lo + jj) + (tt - __ldg(off + jj));
        me.o = ld_stream(outidx + e, pstream);
        me.cx = __ldg(sw2 + me.j) * (double)ld_stream(vals + e, pstream);
        if (HOT) {   // hot row: o = ~slot (negative)
          const int32_t slot = hot_slot ? __ldg(hot_slot + me.o) : me.o;
          if (slot >= 0) me.o = ~slot;
        }
      }
      const int cnt = (int)min((int64_t)32, t1 - t);
      __syncwarp();   // the previous group's reads of we[] are done
      *reinterpret_cast<double2 *>(we + lane) =
          make_double2(me.cx, __longlong_as_double(((long long)me.j << 32) | (uint32_t)me.o));
      __syncwarp();
      const int32_t j0 = __shfl_sync(0xffffffffu, me.j, 0);
      auto load_z = [&](int32_t j) {
        jz = j;
        z0 = lane < r ? __ldg(Z + (int64_t)j * ld + lane) * sc0 : 0.0;
        if (HI) z1 = lane + 32 < r ? __ldg(Z + (int64_t)j * ld + lane + 32) * sc1 : 0.0;
      };
      if (__all_sync(0xffffffffu, !valid || me.j == j0)) {
        // whole group inside one fiber: one z row for all of its entries
        if (j0 != jz) load_z(j0);
#pragma unroll 4
        for (int u = 0; u < cnt; ++u) {
          const double2 ev = *reinterpret_cast<const double2 *>(we + u);
          const int32_t o = (int32_t)__double_as_longlong(ev.y);
          if (HOT && o < 0) { hot_add(hacc, ~o, lane, ev.x, z0, on0); continue; }
          const uint64_t rb = (uint64_t)(uint32_t)o * rowb;
          rhs_red<FX>(Mb0 + rb, ev.x, z0, on0);
          if (HI) rhs_red<FX>(Mb1 + rb, ev.x, z1, on1);
        }
      } else {
        // several fibers (short fibers: C2/C3): the z rows of 8 entries are
        // loaded before their 8 reductions, so the loads overlap instead of
        // each fiber change waiting for its own (entries of one fiber hit L1)
        constexpr int ZB = 4;
        for (int u0 = 0; u0 < cnt; u0 += ZB) {
          double za[ZB], zb[ZB];
#pragma unroll
          for (int v = 0; v < ZB; ++v) {
            const int u = min(u0 + v, cnt - 1);
            const int64_t zr = (int64_t)we[u].j * ld;
            za[v] = lane < r ? __ldg(Z + zr + lane) * sc0 : 0.0;
            if (HI) zb[v] = lane + 32 < r ? __ldg(Z + zr + lane + 32) * sc1 : 0.0;
          }
#pragma unroll
          for (int v = 0; v < ZB; ++v) {
            if (u0 + v >= cnt) break;
            const double2 ev = *reinterpret_cast<const double2 *>(we + u0 + v);
            const int32_t o = (int32_t)__double_as_longlong(ev.y);
            if (HOT && o < 0) { hot_add(hacc, ~o, lane, ev.x, za[v], on0); continue; }
            const uint64_t rb = (uint64_t)(uint32_t)o * rowb;
            rhs_red<FX>(Mb0 + rb, ev.x, za[v], on0);
            if (HI) rhs_red<FX>(Mb1 + rb, ev.x, zb[v], on1);
          }
        }
        jz = -1;
      }
      jcur = __shfl_sync(0xffffffffu, jj, 31);   // segment of tmax
    }
  }
}

template <typename VT, bool HI, bool FIXED>
__global__ void __launch_bounds__(kRhsThreads, HI ? 6 : 8) k_rhs(const int64_t *__restrict__ off, const int64_t *__restrict__ lo,
                                                    const int32_t *__restrict__ seg_j, int64_t nseg,
                                                    const int64_t *__restrict__ mk_ptr,
                                                    unsigned long long *__restrict__ work,
                                                    const int32_t *__restrict__ outidx, const VT *__restrict__ vals,
                                                    const double *__restrict__ sw2, const double *__restrict__ Z,
                                                    int r, int ld, double *__restrict__ M, int64_t per_warp,
                                                    const double *__restrict__ fscale,
                                                    const int64_t *nseg_dev = nullptr, const StepCtl *ctl = nullptr) {
  CPARLS_GUARD(ctl);
  nseg = dcount(nseg, nseg_dev);
  __shared__ __align__(16) RhsEnt ents[kRhsThreads];
  RhsEnt *we = ents + (threadIdx.x & ~31);
  const int lane = threadIdx.x & 31;
  const int64_t mk = *mk_ptr;
  // FIXED: the scales' flag (k_fixed_scales) picks the loop once per warp;
  // an out-of-range bound falls back to fp64 reductions
  if (FIXED && fscale[2 * kMaxRank] != 0.0) {
    const double sc0 = lane < r ? fscale[lane] : 0.0;
    const double sc1 = HI && lane + 32 < r ? fscale[lane + 32] : 0.0;
    rhs_body<VT, HI, true>(off, lo, seg_j, nseg, mk, work, outidx, vals, sw2, Z, r, ld, M, per_warp, sc0, sc1, we);
  } else {
    rhs_body<VT, HI, false>(off, lo, seg_j, nseg, mk, work, outidx, vals, sw2, Z, r, ld, M, per_warp, 1.0, 1.0, we);
  }
}

// k_rhs with hot rows (see HotAcc): one CTA of kRhsHotThreads per SM, H rows
// x r int64 accumulators in dynamic shared memory.  Only with the fixed-point
// reductions and r <= 32; when the scales' flag selects the fp64 fallback the
// kernel reduces every entry into M directly.
constexpr int kRhsHotThreads = 1024;

template <typename VT>
__global__ void __launch_bounds__(kRhsHotThreads, 1)
    k_rhs_hot(const int64_t *__restrict__ off, const int64_t *__restrict__ lo, const int32_t *__restrict__ seg_j,
              int64_t nseg, const int64_t *__restrict__ mk_ptr, unsigned long long *__restrict__ work,
              const int32_t *__restrict__ outidx, const VT *__restrict__ vals, const double *__restrict__ sw2,
              const double *__restrict__ Z, int r, int ld, double *__restrict__ M, int64_t per_warp,
              const double *__restrict__ fscale, const int32_t *__restrict__ hot_slot,
              const int32_t *__restrict__ hot_rows, int H, const int64_t *nseg_dev = nullptr,
              const StepCtl *ctl = nullptr) {
  CPARLS_GUARD(ctl);
  nseg = dcount(nseg, nseg_dev);
  __shared__ __align__(16) RhsEnt ents[kRhsHotThreads];
  extern __shared__ uint32_t hot_words[];
  RhsEnt *we = ents + (threadIdx.x & ~31);
  const int lane = threadIdx.x & 31;
  const int64_t mk = *mk_ptr;
  if (fscale[2 * kMaxRank] == 0.0) {
    rhs_body<VT, false, false>(off, lo, seg_j, nseg, mk, work, outidx, vals, sw2, Z, r, ld, M, per_warp, 1.0, 1.0,
                               we);
    return;
  }
  const HotAcc h{hot_words, hot_words + H * r, r};
  for (int i = threadIdx.x; i < 2 * H * r; i += blockDim.x) hot_words[i] = 0u;
  __syncthreads();
  const double sc0 = lane < r ? fscale[lane] : 0.0;
  rhs_body<VT, false, true, true>(off, lo, seg_j, nseg, mk, work, outidx, vals, sw2, Z, r, ld, M, per_warp, sc0, 0.0,
                                  we, hot_slot, h);
  __syncthreads();
  // this CTA's partial hot rows into M (int64 adds modulo 2^64, any order)
  for (int i = threadIdx.x; i < H * r; i += blockDim.x) {
    const unsigned long long v = ((unsigned long long)h.hi[i] << 32) | h.lo[i];
    if (v == 0ull) continue;
    const int slot = i / r, col = i - slot * r;
    const int64_t row = hot_rows ? (int64_t)__ldg(hot_rows + slot) : (int64_t)slot;
    asm volatile("red.global.add.u64 [%0], %1;" ::"l"(M + row * ld + col), "l"(v) : "memory");
  }
}

// Degree of every row of mode k in this rank's copy (hot-row choice, create).
__global__ void k_row_degree(const int32_t *__restrict__ outidx, int64_t nnz, uint32_t *__restrict__ deg) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(deg + outidx[e], 1u);
}

// hot_slot[hot_rows[s]] = s for the H hottest rows (the rest stay -1).
__global__ void k_hot_slots(const int32_t *__restrict__ rows, int H, int32_t *__restrict__ hot_slot) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < H) hot_slot[rows[s]] = s;
}

// For every (window w, sample j): the sub-range of fiber j whose output rows
// fall in [w*RW, (w+1)*RW) (fibers are sorted by output row).
__global__ void k_win_bounds(const int64_t *__restrict__ lo, const int64_t *__restrict__ len, int64_t sbar,
                             const int32_t *__restrict__ outidx, int nwin, int64_t RW,
                             int64_t *__restrict__ seg_lo, int64_t *__restrict__ seg_len,
                             int32_t *__restrict__ seg_j, const int64_t *sbar_dev = nullptr,
                             int64_t *nseg_out = nullptr, const StepCtl *ctl = nullptr) {
  CPARLS_GUARD(ctl);
  sbar = dcount(sbar, sbar_dev);
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g == 0 && nseg_out) *nseg_out = (int64_t)nwin * sbar;
  if (g >= (int64_t)nwin * sbar) return;
  const int w = (int)(g / sbar);
  const int64_t j = g - (int64_t)w * sbar;
  const int64_t f0 = lo[j], f1 = f0 + len[j];
  auto lb = [&](int64_t o) {   // first e in [f0, f1) with outidx[e] >= o
    int64_t a = f0, n = f1 - f0;
    while (n > 0) {
      int64_t h = n >> 1;
      if (__ldg(outidx + a + h) < o) { a += h + 1; n -= h + 1; }
      else n = h;
    }
    return a;
  };
  const int64_t b0 = (w == 0) ? f0 : lb((int64_t)w * RW);
  const int64_t b1 = (w == nwin - 1) ? f1 : lb((int64_t)(w + 1) * RW);
  seg_lo[g] = b0;
  seg_len[g] = b1 - b0;
  seg_j[g] = (int32_t)j;
}

}  // namespace cparls
