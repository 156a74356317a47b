// fit.cuh -- K10 exact fit (eq:fit P:867-875): the inner product <X, M> of the
// tensor with the Kruskal model, streamed over the fit mode k*'s sorted copy.
//
// Nonzeros of one fiber share the other-mode rows, so per fiber the leader
// lane forms h = lambda * A_{m_1}(i_1,:) * ... * A_{m_d}(i_d,:) once (into a
// per-lane shared slot) and every nonzero then needs only its own
// A_{k*}(out,:) row: <X,M> = sum_e x_e <h_fiber(e), A_{k*}(out_e,:)>.  Keys
// are decoded with an fp64 reciprocal plus an exact integer correction.
#pragma once
#include "common.cuh"

namespace cparls {

constexpr int kFitThreads = 256;

struct FitDecode {
  int d;
  int64_t n[kMaxModes];
  double inv[kMaxModes];      // 1.0 / n
  const double *A[kMaxModes];
  int fast;                   // keys < 2^53: reciprocal path exact after correction
};

// q = key / n, key -= q*n ... returns quotient, writes remainder
__device__ __forceinline__ uint64_t divmod_fast(uint64_t key, int64_t n, double inv, uint64_t &rem, int fast) {
  if (!fast) {
    uint64_t q = key / (uint64_t)n;
    rem = key - q * (uint64_t)n;
    return q;
  }
  int64_t q = (int64_t)((double)key * inv);
  int64_t rr = (int64_t)key - q * n;
  if (rr < 0) { --q; rr += n; }
  if (rr >= n) { ++q; rr -= n; }
  rem = (uint64_t)rr;
  return (uint64_t)q;
}

// Thread per nonzero (grid-stride over 32-nonzero warp tiles).  Each thread
// issues its A_{k*}(out,:) row loads first; the fiber's leader lane (first lane
// of a run of equal keys) forms h = lambda * A_{m_1}(i_1,:) * ... into its
// shared slot; every lane then dots its row with its fiber's h.
template <typename VT, int RMAX>
__global__ void __launch_bounds__(kFitThreads, 2) k_fit_thread(const uint64_t *__restrict__ keys,
                                                           const int32_t *__restrict__ outidx,
                                                           const VT *__restrict__ vals, int64_t nnz, FitDecode fd,
                                                           const double *__restrict__ Ak,
                                                           const double *__restrict__ lam, int r, int ld,
                                                           dd *__restrict__ part) {
  extern __shared__ double hbuf[];   // kFitThreads slots of RS doubles
  __shared__ double lam_s[kMaxRank + 1];
  const int RS = r | 1;              // odd slot stride: conflict-free 8-byte accesses
  for (int c = threadIdx.x; c <= kMaxRank; c += blockDim.x) lam_s[c] = c < r ? lam[c] : 0.0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  double *hw = hbuf + (size_t)(threadIdx.x & ~31) * RS;
  dd acc = {0.0, 0.0};
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e0 = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); e0 < nnz; e0 += stride) {
    const int64_t e = e0 + lane;
    const bool valid = e < nnz;
    const uint64_t key = valid ? keys[e] : ~0ull;
    const int32_t o = valid ? outidx[e] : 0;
    const double x = valid ? (double)vals[e] : 0.0;
    double2 a[RMAX / 2];
    const double2 *ar = reinterpret_cast<const double2 *>(Ak + (int64_t)o * ld);
#pragma unroll
    for (int c2 = 0; c2 < RMAX / 2; ++c2)
      a[c2] = (valid && 2 * c2 < r) ? __ldg(ar + c2) : make_double2(0.0, 0.0);
    uint64_t prev = __shfl_up_sync(0xffffffffu, key, 1);
    if (lane == 0) prev = ~key;
    const bool lead = valid && key != prev;
    const unsigned lm = __ballot_sync(0xffffffffu, lead);
    if (lead) {
      double *h = hw + lane * RS;
      for (int c = 0; c < r; ++c) h[c] = lam_s[c];
      uint64_t t = key;
      for (int m = 0; m < fd.d; ++m) {
        uint64_t rem;
        t = divmod_fast(t, fd.n[m], fd.inv[m], rem, fd.fast);
        const double2 *row = reinterpret_cast<const double2 *>(fd.A[m] + rem * ld);
        double2 v[RMAX / 2];
#pragma unroll
        for (int c2 = 0; c2 < RMAX / 2; ++c2) v[c2] = (2 * c2 < r) ? __ldg(row + c2) : make_double2(0.0, 0.0);
#pragma unroll
        for (int c2 = 0; c2 < RMAX / 2; ++c2) {
          if (2 * c2 < r) h[2 * c2] *= v[c2].x;
          if (2 * c2 + 1 < r) h[2 * c2 + 1] *= v[c2].y;
        }
      }
    }
    __syncwarp();
    if (valid) {
      const int src = 31 - __clz(lm & (0xffffffffu >> (31 - lane)));   // last leader at or before lane
      const double *h = hw + src * RS;
      double mv = 0.0;
#pragma unroll
      for (int c2 = 0; c2 < RMAX / 2; ++c2) {
        if (2 * c2 < r) mv += h[2 * c2] * a[c2].x;
        if (2 * c2 + 1 < r) mv += h[2 * c2 + 1] * a[c2].y;
      }
      acc = dd_add_d(acc, x * mv);
    }
    __syncwarp();
  }
  acc = warp_sum_dd(acc);
  __shared__ dd ws[kFitThreads / 32];
  if (lane == 0) ws[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    dd t = {0.0, 0.0};
    for (int i = 0; i < kFitThreads / 32; ++i) t = dd_add(t, ws[i]);
    part[blockIdx.x] = t;
  }
}

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit_wait() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

// As k_fit_thread, but each warp stages the 32 A_{k*}(out,:) rows of its tile
// into shared memory with coalesced 16-byte cp.async chunks (about 2.3 rows per
// instruction instead of one row per lane), overlapping the fiber leaders' h
// computation; lanes then read their own row from shared memory.
template <typename VT, int RMAX>
__global__ void __launch_bounds__(kFitThreads) k_fit_stage(const uint64_t *__restrict__ keys,
                                                          const int32_t *__restrict__ outidx,
                                                          const VT *__restrict__ vals, int64_t nnz, FitDecode fd,
                                                          const double *__restrict__ Ak,
                                                          const double *__restrict__ lam, int r, int ld,
                                                          dd *__restrict__ part) {
  extern __shared__ __align__(16) double fsm[];
  const int S = ld + 2;              // even (16-byte aligned rows), 2-way conflicts at most
  const int RS = r | 1;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double *tile = fsm + (size_t)w * 32 * S;                                   // 32 rows x S
  double *hw = fsm + (size_t)(kFitThreads / 32) * 32 * S + (size_t)w * 32 * RS;   // 32 slots x RS
  __shared__ double lam_s[kMaxRank + 1];
  for (int c = threadIdx.x; c <= kMaxRank; c += blockDim.x) lam_s[c] = c < r ? lam[c] : 0.0;
  __syncthreads();
  const int H = ld / 2;              // 16-byte chunks per row
  const uint64_t pstream = l2_evict_first();
  dd acc = {0.0, 0.0};
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e0 = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); e0 < nnz; e0 += stride) {
    const int64_t e = e0 + lane;
    const bool valid = e < nnz;
    const int n = (int)min((int64_t)32, nnz - e0);
    const uint64_t key = valid ? ld_stream(keys + e, pstream) : ~0ull;
    const int32_t o = valid ? ld_stream(outidx + e, pstream) : 0;
    const double x = valid ? (double)ld_stream(vals + e, pstream) : 0.0;
    // stage A rows: chunk f = lane + 32q  ->  row rho = f / H, part = f % H
    {
      int rho = lane / H, part = lane - (lane / H) * H;
      for (int f = lane; f < 32 * H; f += 32) {
        const int orow = __shfl_sync(0xffffffffu, o, rho & 31);
        if (rho < n) cp_async16(tile + rho * S + 2 * part, Ak + (int64_t)orow * ld + 2 * part);
        part += 32;
        while (part >= H) { part -= H; ++rho; }
      }
      asm volatile("cp.async.commit_group;\n" ::: "memory");
    }
    uint64_t prev = __shfl_up_sync(0xffffffffu, key, 1);
    if (lane == 0) prev = ~key;
    const bool lead = valid && key != prev;
    const unsigned lm = __ballot_sync(0xffffffffu, lead);
    if (lead) {
      double *h = hw + lane * RS;
      for (int c = 0; c < r; ++c) h[c] = lam_s[c];
      uint64_t t = key;
      for (int m = 0; m < fd.d; ++m) {
        uint64_t rem;
        t = divmod_fast(t, fd.n[m], fd.inv[m], rem, fd.fast);
        const double2 *row = reinterpret_cast<const double2 *>(fd.A[m] + rem * ld);
        double2 v[RMAX / 2];
#pragma unroll
        for (int c2 = 0; c2 < RMAX / 2; ++c2) v[c2] = (2 * c2 < r) ? __ldg(row + c2) : make_double2(0.0, 0.0);
#pragma unroll
        for (int c2 = 0; c2 < RMAX / 2; ++c2) {
          if (2 * c2 < r) h[2 * c2] *= v[c2].x;
          if (2 * c2 + 1 < r) h[2 * c2 + 1] *= v[c2].y;
        }
      }
    }
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncwarp();
    if (valid) {
      const int src = 31 - __clz(lm & (0xffffffffu >> (31 - lane)));   // last leader at or before lane
      const double *h = hw + src * RS;
      const double *a = tile + lane * S;
      double mv = 0.0;
#pragma unroll
      for (int c = 0; c < RMAX; ++c)
        if (c < r) mv += h[c] * a[c];
      acc = dd_add_d(acc, x * mv);
    }
    __syncwarp();
  }
  acc = warp_sum_dd(acc);
  __shared__ dd ws[kFitThreads / 32];
  if (lane == 0) ws[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    dd tt = {0.0, 0.0};
    for (int i = 0; i < kFitThreads / 32; ++i) tt = dd_add(tt, ws[i]);
    part[blockIdx.x] = tt;
  }
}

inline size_t fit_stage_smem(int r, int ld) {
  return sizeof(double) * ((size_t)kFitThreads * (ld + 2) + (size_t)kFitThreads * (r | 1)) + 16;
}

// <X,M> from block partials; ||M||^2 = lambda^T (*_m G_m) lambda with the
// factors' Grams G_m (P:146-148 structure); fit = 1 - sqrt(max(0, ||X||^2 -
// 2<X,M> + ||M||^2)) / ||X|| (AMB-16).
struct FitModes {
  int D;
  const double *GA[kMaxModes];
};

__global__ void k_fit_final(const dd *__restrict__ part, int nb, FitModes fm, const double *__restrict__ lam, int r,
                            double normX2, double *out) {
  __shared__ dd red[256];
  dd inner = {0.0, 0.0}, nm = {0.0, 0.0};
  for (int i = threadIdx.x; i < nb; i += blockDim.x) inner = dd_add(inner, part[i]);
  for (int i = threadIdx.x; i < r * r; i += blockDim.x) {
    const int p = i / r, q = i % r;
    double h = lam[p] * lam[q];
    for (int m = 0; m < fm.D; ++m) h *= fm.GA[m][i];
    nm = dd_add_d(nm, h);
  }
  red[threadIdx.x] = inner;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] = dd_add(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  const dd in_ = red[0];
  __syncthreads();
  red[threadIdx.x] = nm;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] = dd_add(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double inner_v = in_.hi + in_.lo, nm_v = red[0].hi + red[0].lo;
    double resid2 = normX2 - 2.0 * inner_v + nm_v;
    if (resid2 < 0.0) resid2 = 0.0;
    out[0] = 1.0 - sqrt(resid2) / sqrt(normX2);
    out[1] = inner_v;
    out[2] = nm_v;
  }
}

// number of distinct keys (fibers) of a sorted key array, per-block counts
__global__ void k_count_fibers(const uint64_t *__restrict__ keys, int64_t nnz, unsigned long long *cnt) {
  unsigned long long c = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x)
    c += (i == 0 || keys[i] != keys[i - 1]);
  c = warp_sum<unsigned long long>(c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(cnt, c);
}

}  // namespace cparls
