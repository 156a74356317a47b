// rhs.cuh -- K8 sampled right-hand side M = Xs^T diag(w^2) Z_S (P:949-958,
// AMB-14): M(out_e,:) += w_j^2 x_e z_j for every matched nonzero e of every
// sampled fiber j.
//
// Warps walk the concatenated matched entries (fiber after fiber, so z_j and
// w_j^2 stay in registers across a fiber); lanes = columns, so one entry is one
// r-wide fp64 reduction into M's row.  Global fp64 `red` (no f64 vector red on
// sm_100a) bounds this kernel: bench.py measures the ceiling of exactly this
// pattern (r-lane reds into random rows of an L2-sized window) with
// libcparls_peaks.so and k_rhs runs at ~97% of it.  (Privatizing the heaviest
// rows in shared memory was measured and dropped: the top 64 rows hold < 1% of
// the entries on the Zipf workloads, and the smem cost halved occupancy.)
//
// M (n_k x ld fp64) is far larger than L2 for the big modes, so random reds
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

__device__ __forceinline__ void red_fixed(double *addr, double v, double sc) {
  const long long q = __double2ll_rn(v * sc);   // v * 2^e exact; the only rounding is to the integer
  if (q != 0) atomicAdd(reinterpret_cast<unsigned long long *>(addr), (unsigned long long)q);
}

template <typename VT, bool HI, bool FIXED>
__global__ void __launch_bounds__(kRhsThreads) k_rhs(const int64_t *__restrict__ off, const int64_t *__restrict__ lo,
                                                    const int32_t *__restrict__ seg_j, int64_t nseg,
                                                    const int64_t *__restrict__ mk_ptr,
                                                    unsigned long long *__restrict__ work,
                                                    const int32_t *__restrict__ outidx, const VT *__restrict__ vals,
                                                    const double *__restrict__ sw2, const double *__restrict__ Z,
                                                    int r, int ld, double *__restrict__ M, int64_t per_warp,
                                                    const double *__restrict__ fscale) {
  const int lane = threadIdx.x & 31;
  const bool fx = FIXED && fscale[2 * kMaxRank] != 0.0;   // else: out-of-range bound, fp64 reductions
  const double sc0 = FIXED && lane < r ? fscale[lane] : 0.0;
  const double sc1 = FIXED && HI && lane + 32 < r ? fscale[lane + 32] : 0.0;
  const int64_t mk = *mk_ptr;
  const uint64_t pstream = l2_evict_first();
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
    int64_t jz = -1;        // sample whose z row is loaded
    double z0 = 0.0, z1 = 0.0;
    for (int64_t t = t0; t < t1; t += 32) {
      const int64_t tt = t + lane;
      const bool valid = tt < t1;
      int64_t jj = jcur;
      while (jj + 1 < nseg && __ldg(off + jj + 1) <= tt) ++jj;
      int64_t j_l = -1;
      int32_t o_l = 0;
      double cx_l = 0.0;     // w_j^2 * x_e
      if (valid) {
        j_l = seg_j ? (int64_t)__ldg(seg_j + jj) : jj;
        const int64_t e = __ldg(lo + jj) + (tt - __ldg(off + jj));
        o_l = ld_stream(outidx + e, pstream);
        cx_l = __ldg(sw2 + j_l) * (double)ld_stream(vals + e, pstream);
      }
      const int cnt = (int)min((int64_t)32, t1 - t);
      const int64_t j0 = __shfl_sync(0xffffffffu, j_l, 0);
      if (__all_sync(0xffffffffu, !valid || j_l == j0)) {
        // whole group inside one fiber: one z row for all 32 entries
        if (j0 != jz) {
          jz = j0;
          z0 = lane < r ? __ldg(Z + j0 * ld + lane) : 0.0;
          if (HI) z1 = lane + 32 < r ? __ldg(Z + j0 * ld + lane + 32) : 0.0;
        }
#pragma unroll 4
        for (int u = 0; u < cnt; ++u) {
          const int o = __shfl_sync(0xffffffffu, o_l, u);
          const double cx = __shfl_sync(0xffffffffu, cx_l, u);
          if (lane < r) {
            if (fx) red_fixed(M + (int64_t)o * ld + lane, cx * z0, sc0);
            else atomicAdd(M + (int64_t)o * ld + lane, cx * z0);
          }
          if (HI && lane + 32 < r) {
            if (fx) red_fixed(M + (int64_t)o * ld + lane + 32, cx * z1, sc1);
            else atomicAdd(M + (int64_t)o * ld + lane + 32, cx * z1);
          }
        }
      } else {
        for (int u = 0; u < cnt; ++u) {
          const int o = __shfl_sync(0xffffffffu, o_l, u);
          const double cx = __shfl_sync(0xffffffffu, cx_l, u);
          const int64_t ju = __shfl_sync(0xffffffffu, j_l, u);
          if (ju != jz) {
            jz = ju;
            z0 = lane < r ? __ldg(Z + ju * ld + lane) : 0.0;
            if (HI) z1 = lane + 32 < r ? __ldg(Z + ju * ld + lane + 32) : 0.0;
          }
          if (lane < r) {
            if (fx) red_fixed(M + (int64_t)o * ld + lane, cx * z0, sc0);
            else atomicAdd(M + (int64_t)o * ld + lane, cx * z0);
          }
          if (HI && lane + 32 < r) {
            if (fx) red_fixed(M + (int64_t)o * ld + lane + 32, cx * z1, sc1);
            else atomicAdd(M + (int64_t)o * ld + lane + 32, cx * z1);
          }
        }
      }
      jcur = __shfl_sync(0xffffffffu, jj, 31);
    }
  }
}

// For every (window w, sample j): the sub-range of fiber j whose output rows
// fall in [w*RW, (w+1)*RW) (fibers are sorted by output row).
__global__ void k_win_bounds(const int64_t *__restrict__ lo, const int64_t *__restrict__ len, int64_t sbar,
                             const int32_t *__restrict__ outidx, int nwin, int64_t RW,
                             int64_t *__restrict__ seg_lo, int64_t *__restrict__ seg_len,
                             int32_t *__restrict__ seg_j) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
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
