// rhs_bucket.cuh -- K8+K9 without global fp64 reductions: the sampled RHS
// M = Xs^T diag(w^2) Z_S (AMB-14) and B = M G^+  for large
// modes.
//
// k_rhs (rhs.cuh) issues one r-lane fp64 red per matched entry and runs at
// ~97% of the measured red ceiling of that pattern; the only way past it is to
// stop reducing in L2.  Here the matched entries (fiber-major) are first
// placed into buckets of kBktRows consecutive output rows (one counting pass
// and one placing pass; the per-bucket counters take one integer atomic per
// distinct bucket in a warp, not per entry and column), then one CTA owns a
// bucket at a time: a warp owns a bucket of 32 rows and accumulates its
// records into shared memory with plain fp64 adds, then writes the finished
// rows of M (every row: no zeroing pass).  B = M G^+ follows in
// k_solve_rows_t as on the atomic path.
#pragma once
#include "common.cuh"

namespace cparls {

constexpr int kBktShift = 5;                 // 32 output rows per bucket: one warp owns a bucket
constexpr int kBktRows = 1 << kBktShift;
constexpr int kBktThreads = 256;             // 8 warps
constexpr int kBktJBits = 32 - kBktShift;    // record key = (j << kBktShift) | row-in-bucket
constexpr int64_t kBktMaxSbar = int64_t(1) << kBktJBits;

// Walks the matched entries t in [0, mk) (fiber j's entries are
// [off[j], off[j] + len_j) of the concatenation, stored at lo[j] + ...):
// warps take per_warp-entry chunks from *work and call op(valid, j, e) once per
// 32-entry group (lane-parallel; the whole warp calls op).
template <typename Op>
__device__ __forceinline__ void for_matched(const int64_t *__restrict__ off, const int64_t *__restrict__ lo,
                                            int64_t nseg, int64_t mk, unsigned long long *work, int64_t per_warp,
                                            Op &op) {
  const int lane = threadIdx.x & 31;
  while (true) {
    int64_t t0 = 0;
    if (lane == 0) t0 = (int64_t)atomicAdd(work, (unsigned long long)per_warp);
    t0 = __shfl_sync(0xffffffffu, t0, 0);
    if (t0 >= mk) break;
    const int64_t t1 = min(mk, t0 + per_warp);
    int64_t a = 0, len = nseg;   // last segment with off <= t0
    while (len > 0) {
      const int64_t half = len >> 1;
      if (__ldg(off + a + half) <= t0) { a += half + 1; len -= half + 1; }
      else len = half;
    }
    int64_t jcur = a - 1;
    for (int64_t t = t0; t < t1; t += 32) {
      const int64_t tt = t + lane;
      const bool valid = tt < t1;
      int64_t jj = jcur;
      while (jj + 1 < nseg && __ldg(off + jj + 1) <= tt) ++jj;
      const int64_t e = valid ? __ldg(lo + jj) + (tt - __ldg(off + jj)) : 0;
      op(valid, jj, e);
      jcur = __shfl_sync(0xffffffffu, jj, 31);
    }
  }
}

struct BktCountOp {
  const int32_t *outidx;
  int64_t row0;
  unsigned long long *cnt;
  uint64_t pol;
  __device__ __forceinline__ void operator()(bool valid, int64_t, int64_t e) {
    const int b = valid ? (int)((ld_stream(outidx + e, pol) - row0) >> kBktShift) : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, b);
    const int lane = threadIdx.x & 31;
    if (valid && lane == __ffs(peers) - 1) atomicAdd(cnt + b, (unsigned long long)__popc(peers));
  }
};

template <typename VT>
struct BktPlaceOp {
  const int32_t *outidx;
  const VT *vals;
  const double *sw2;
  int64_t row0;
  unsigned long long *cursor;
  uint32_t *rec;
  double *recc;
  uint64_t pol;
  __device__ __forceinline__ void operator()(bool valid, int64_t j, int64_t e) {
    const int lane = threadIdx.x & 31;
    int row = 0, b = -1;
    double cx = 0.0;
    if (valid) {
      row = (int)(ld_stream(outidx + e, pol) - row0);
      b = row >> kBktShift;
      cx = __ldg(sw2 + j) * (double)ld_stream(vals + e, pol);   // w_j^2 x_e, as k_rhs forms it
    }
    const unsigned peers = __match_any_sync(0xffffffffu, b);
    const int leader = __ffs(peers) - 1;
    unsigned long long base = 0;
    if (valid && lane == leader) base = atomicAdd(cursor + b, (unsigned long long)__popc(peers));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (valid) {
      const unsigned long long pos = base + __popc(peers & lanemask_lt());
      rec[pos] = ((uint32_t)j << kBktShift) | (uint32_t)(row & (kBktRows - 1));
      recc[pos] = cx;
    }
  }
};

__global__ void __launch_bounds__(256) k_bkt_count(const int64_t *__restrict__ off, const int64_t *__restrict__ lo,
                                                   int64_t nseg, const int64_t *__restrict__ mk_ptr,
                                                   unsigned long long *work, int64_t per_warp,
                                                   const int32_t *__restrict__ outidx, int64_t row0,
                                                   unsigned long long *__restrict__ cnt) {
  BktCountOp op{outidx, row0, cnt, l2_evict_first()};
  for_matched(off, lo, nseg, *mk_ptr, work, per_warp, op);
}

template <typename VT>
__global__ void __launch_bounds__(256) k_bkt_place(const int64_t *__restrict__ off, const int64_t *__restrict__ lo,
                                                   int64_t nseg, const int64_t *__restrict__ mk_ptr,
                                                   unsigned long long *work, int64_t per_warp,
                                                   const int32_t *__restrict__ outidx, const VT *__restrict__ vals,
                                                   const double *__restrict__ sw2, int64_t row0,
                                                   unsigned long long *__restrict__ cursor,
                                                   uint32_t *__restrict__ rec, double *__restrict__ recc) {
  BktPlaceOp<VT> op{outidx, vals, sw2, row0, cursor, rec, recc, l2_evict_first()};
  for_matched(off, lo, nseg, *mk_ptr, work, per_warp, op);
}

__global__ void k_bkt_cursor(const int64_t *__restrict__ start, int64_t nb, unsigned long long *__restrict__ cursor) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nb) cursor[i] = (unsigned long long)start[i];
}

// One 32-row bucket per warp (grid-stride over buckets): the warp's 32 rows of
// M live in a private shared tile.  Records are read 32 at a time (coalesced,
// the next batch prefetched into registers); a step is 4 records, one per
// 8-lane sub-warp (4 columns per lane, 16-byte accesses), and the z rows of 4
// steps are loaded before any of them is used.  A step whose 4 records hit
// two equal rows is replayed one record at a time, so every row is updated by
// plain fp64 adds.  The finished rows are written to M (all of them: no
// zeroing pass), and k_solve_rows_t forms B = M G^+ as on the atomic path.
template <int U>
__global__ void __launch_bounds__(kBktThreads, 3) k_bkt_accum(const int64_t *__restrict__ start, int64_t nbkt,
                                                             const uint32_t *__restrict__ rec,
                                                             const double *__restrict__ recc,
                                                             const double *__restrict__ Z, int64_t nrows, int ld,
                                                             double *__restrict__ M) {
  extern __shared__ __align__(16) double bsm[];   // 8 tiles of 32 x ld
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int sw = lane >> 3, sl = lane & 7, c0 = 4 * sl;
  const bool colok = c0 < ld;
  double *acc = bsm + (size_t)w * kBktRows * ld;
  const int64_t nwarps = (int64_t)gridDim.x * (kBktThreads / 32);
  for (int64_t b = (int64_t)blockIdx.x * (kBktThreads / 32) + w; b < nbkt; b += nwarps) {
    for (int i = lane; i < kBktRows * ld; i += 32) acc[i] = 0.0;
    __syncwarp();
    const uint32_t s0 = (uint32_t)__ldg(start + b), s1 = (uint32_t)__ldg(start + b + 1);
    uint32_t nkey = (s0 + lane < s1) ? __ldg(rec + s0 + lane) : 0xffffffffu;
    double ncc = (s0 + lane < s1) ? __ldg(recc + s0 + lane) : 0.0;
    for (uint32_t k0 = s0; k0 < s1; k0 += 32) {
      const uint32_t key = nkey;
      const double ccl = ncc;
      if (k0 + 32 < s1) {
        const uint32_t kn = k0 + 32 + lane;
        nkey = kn < s1 ? __ldg(rec + kn) : 0xffffffffu;
        ncc = kn < s1 ? __ldg(recc + kn) : 0.0;
      }
      const int n = (int)min(32u, s1 - k0);
      // lane l holds record l of the batch; records 4t..4t+3 form step t
      const int rowl = lane < n ? (int)(key & (kBktRows - 1)) : kBktRows + (lane & 3);
      int d = 0;
#pragma unroll
      for (int x = 1; x < 4; x <<= 1) d |= (__shfl_xor_sync(0xffffffffu, rowl, x, 4) == rowl);
      d |= (__shfl_xor_sync(0xffffffffu, rowl, 3, 4) == rowl);
      const unsigned dupl = __ballot_sync(0xffffffffu, d != 0);
      for (int t0 = 0; t0 < (n + 3) / 4; t0 += U) {
        double2 z0[U], z1[U];
        uint32_t kk[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int src = 4 * (t0 + u) + sw;
          kk[u] = __shfl_sync(0xffffffffu, key, src & 31);
          z0[u] = make_double2(0.0, 0.0);
          z1[u] = make_double2(0.0, 0.0);
          if (src < n && colok) {
            const double2 *zr = reinterpret_cast<const double2 *>(Z + (int64_t)(kk[u] >> kBktShift) * ld + c0);
            z0[u] = __ldg(zr);
            z1[u] = __ldg(zr + 1);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int t = t0 + u;
          if (4 * t >= n) break;
          const int src = 4 * t + sw;
          const double cc = __shfl_sync(0xffffffffu, ccl, src & 31);
          const bool mine = src < n && colok;
          double2 *ar = reinterpret_cast<double2 *>(acc + (int)(kk[u] & (kBktRows - 1)) * ld + c0);
          if (((dupl >> (4 * t)) & 0xfu) == 0u) {
            if (mine) {
              double2 a01 = ar[0], a23 = ar[1];
              a01.x += cc * z0[u].x; a01.y += cc * z0[u].y; a23.x += cc * z1[u].x; a23.y += cc * z1[u].y;
              ar[0] = a01; ar[1] = a23;
            }
          } else {
            for (int q = 0; q < 4; ++q) {
              if (sw == q && mine) {
                double2 a01 = ar[0], a23 = ar[1];
                a01.x += cc * z0[u].x; a01.y += cc * z0[u].y; a23.x += cc * z1[u].x; a23.y += cc * z1[u].y;
                ar[0] = a01; ar[1] = a23;
              }
              __syncwarp();
            }
          }
        }
      }
    }
    __syncwarp();
    // the bucket's rows of M (padding columns stay 0)
    const int64_t rbase = b * kBktRows;
    const int nr = (int)max((int64_t)0, min((int64_t)kBktRows, nrows - rbase));
    double2 *dst = reinterpret_cast<double2 *>(M + rbase * ld);
    const double2 *srct = reinterpret_cast<const double2 *>(acc);
    for (int i = lane; i < nr * ld / 2; i += 32) dst[i] = srct[i];
    __syncwarp();
  }
}

inline size_t bkt_accum_smem(int ld) { return sizeof(double) * (size_t)(kBktThreads / 32) * kBktRows * ld; }

}  // namespace cparls
