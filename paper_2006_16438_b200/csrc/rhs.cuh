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

template <typename VT, bool HI, bool FX>
__device__ __forceinline__ void rhs_body(const int64_t *__restrict__ off, const int64_t *__restrict__ lo,
                                         const int32_t *__restrict__ seg_j, int64_t nseg, int64_t mk,
                                         unsigned long long *__restrict__ work, const int32_t *__restrict__ outidx,
                                         const VT *__restrict__ vals, const double *__restrict__ sw2,
                                         const double *__restrict__ Z, int r, int ld, double *__restrict__ M,
                                         int64_t per_warp, double sc0, double sc1, RhsEnt *we) {
  const int lane = threadIdx.x & 31;
  const uint64_t pstream = l2_evict_first();
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
    // segment containing entry t0: last g with off[g] <= t0 (skips empty ones)
    int64_t a = 0, len = nseg;
    while (len > 0) {
      int64_t half = len >> 1;
      if (__ldg(off + a + half) <= t0) { a += half + 1; len -= half + 1; }
      else len = half;
    }
    int64_t jcur = a - 1;   // segment of the first entry of the current 32-group
    int32_t jz = -1;        // sample whose (scaled) z row is loaded
    double z0 = 0.0, z1 = 0.0;
    for (int64_t t = t0; t < t1; t += 32) {
      const int64_t tt = t + lane;
      const bool valid = tt < t1;
      int64_t jj = jcur;
      while (jj + 1 < nseg && __ldg(off + jj + 1) <= tt) ++jj;
      RhsEnt me = {0.0, 0, -1};
      if (valid) {
        me.j = seg_j ? __ldg(seg_j + jj) : (int32_t)jj;
        const int64_t e = __ldg(lo + jj) + (tt - __ldg(off + jj));
        me.o = ld_stream(outidx + e, pstream);
        me.cx = __ldg(sw2 + me.j) * (double)ld_stream(vals + e, pstream);
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
          const uint64_t rb = (uint64_t)(uint32_t)__double_as_longlong(ev.y) * rowb;
          rhs_red<FX>(Mb0 + rb, ev.x, z0, on0);
          if (HI) rhs_red<FX>(Mb1 + rb, ev.x, z1, on1);
        }
      } else {
        for (int u = 0; u < cnt; ++u) {
          const double2 ev = *reinterpret_cast<const double2 *>(we + u);
          const long long bits = __double_as_longlong(ev.y);
          const int32_t ju = (int32_t)(bits >> 32);
          if (ju != jz) load_z(ju);
          const uint64_t rb = (uint64_t)(uint32_t)bits * rowb;
          rhs_red<FX>(Mb0 + rb, ev.x, z0, on0);
          if (HI) rhs_red<FX>(Mb1 + rb, ev.x, z1, on1);
        }
      }
      jcur = __shfl_sync(0xffffffffu, jj, 31);
    }
  }
}

template <typename VT, bool HI, bool FIXED>
__global__ void __launch_bounds__(kRhsThreads) k_rhs(const int64_t *__restrict__ off, const int64_t *__restrict__ lo,
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
