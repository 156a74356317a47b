// fit.cuh -- K10 exact fit (eq:fit P:867-875): the inner product <X, M> of the
// tensor with the Kruskal model, streamed over the fit mode k*'s sorted copy.
//
// Nonzeros of one fiber share the other-mode rows, so per fiber
// h = lambda * A_{m_1}(i_1,:) * ... * A_{m_d}(i_d,:) is formed once and every
// nonzero then needs only its own A_{k*}(out,:) row:
// <X,M> = sum_e x_e <h_fiber(e), A_{k*}(out_e,:)>.  k_fit_sub (D <= 4) maps one
// entry to a sub-warp of ld/4 lanes; k_fit_thread (D > 4) maps one entry to a
// thread.  Keys are decoded with an fp64 reciprocal plus an exact integer
// correction.
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
                                                           dd *__restrict__ part, const StepCtl *ctl = nullptr) {
  CPARLS_GUARD(ctl);
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

// Work is taken in kFitChunk-entry chunks from a global counter; h depends only
// on the key, so a fiber split across chunks is simply restarted.
constexpr int kFitChunk = 2048;
#ifndef CPARLS_FIT_U
#define CPARLS_FIT_U 4   // entries per sub-warp issued before any is consumed
#endif
// Resident CTAs per SM the register budget is sized for.  Measured on C4
// (r = 25): U4/2 CTAs 69.1 ms, U2/3 83.1, U2/4 79.9, U4/3 85.0 (spills), U8/2
// 75.6; 256-bit row loads (LDG.E.ENL2.256) instead of 2 x 16 B: 71.0.
#ifndef CPARLS_FIT_LD256
#define CPARLS_FIT_LD256 1   // one 256-bit load per lane per row (C4: 65.7 -> 64.5 ms with 256-byte rows)
#endif
#ifndef CPARLS_FIT_MINB
#define CPARLS_FIT_MINB 2
#endif

// Sub-warp fit: SW lanes per entry, 4 columns per lane (two 16-byte loads; ld
// is a multiple of 4, so a row is ld/4 lanes), NS = 32/SW entries per warp
// step.  (k_fit_cols, one column per lane, spent ~45 warp instructions per
// nonzero and was issue-bound.)  A warp takes a kFitChunk-entry chunk; sub-warp
// s walks its own contiguous 1/NS of it, SW entries per batch loaded by its
// own lanes, so a fiber is only restarted at a sub-range start.  Per fiber
// h = g * A_{m_1}(i_1,:) * ... * A_{m_{d-1}}(i_{d-1},:) where g = lambda *
// A_{m_d}(i_d,:) is cached per sub-warp: m_d is the slowest key mode, so the
// copy is sorted by it and g changes only every ~nnz/n_{m_d} entries.
// acc_c += x_e * A_{k*}(out_e,c) * h_c per lane: plain fp64 within a chunk,
// folded into a double-double per chunk (AMB-16).
template <typename VT, int SW, int DM, int U>
__global__ void __launch_bounds__(kFitThreads, CPARLS_FIT_MINB) k_fit_sub(const uint64_t *__restrict__ keys,
                                                          const int32_t *__restrict__ outidx,
                                                          const VT *__restrict__ vals, int64_t nnz, FitDecode fd,
                                                          const double *__restrict__ Ak,
                                                          const double *__restrict__ lam, int r, int ld,
                                                          dd *__restrict__ part,
                                                          unsigned long long *__restrict__ work,
                                                          const StepCtl *ctl = nullptr) {
  CPARLS_GUARD(ctl);
  static_assert(SW >= 2 && SW <= 32 && (SW & (SW - 1)) == 0, "SW power of two");
  constexpr int NS = 32 / SW;
  constexpr int SUB = kFitChunk / NS;    // entries per sub-warp per chunk (multiple of SW)
  const int lane = threadIdx.x & 31;
  const int sl = lane & (SW - 1);        // lane within the sub-warp
  const int sbase = lane & ~(SW - 1);
  const int c0 = 4 * sl;
  const bool colok = c0 < ld;            // ld % 4 == 0: all 4 columns in bounds
  double lam4[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) lam4[q] = (c0 + q < r) ? lam[c0 + q] : 0.0;
  const uint64_t pstream = l2_evict_first();
  const double *Aslow = fd.A[DM - 1];
  dd acc = {0.0, 0.0};
  while (true) {
    int64_t cb = 0;
    if (lane == 0) cb = (int64_t)atomicAdd(work, (unsigned long long)kFitChunk);
    cb = __shfl_sync(0xffffffffu, cb, 0);
    if (cb >= nnz) break;
    const int64_t s0 = cb + (int64_t)(lane / SW) * SUB;
    const int64_t s1 = min(nnz, s0 + SUB);
    double h[4] = {0.0, 0.0, 0.0, 0.0};
    double g[4] = {0.0, 0.0, 0.0, 0.0};
    double cacc[4] = {0.0, 0.0, 0.0, 0.0};
    uint64_t last_key = ~0ull;
    uint32_t cur_slow = 0xffffffffu;
    // the next batch's stream entries are loaded while this batch's rows are
    // in flight (register double buffer)
    uint64_t nkey = (s0 + sl < s1) ? ld_stream(keys + s0 + sl, pstream) : ~0ull;
    int32_t no = (s0 + sl < s1) ? ld_stream(outidx + s0 + sl, pstream) : 0;
    VT nx = (s0 + sl < s1) ? ld_stream(vals + s0 + sl, pstream) : VT(0);
    for (int64_t b0 = 0; b0 < SUB; b0 += SW) {
      // warp-uniform trip count; a sub-warp past its end has no valid entries
      const int64_t e = s0 + b0 + sl;
      const bool valid = e < s1;
      const uint64_t key = nkey;
      const int32_t o = no;
      const double x = (double)nx;
      {
        const int64_t en = e + SW;
        const bool vn = en < s1 && b0 + SW < SUB;
        nkey = vn ? ld_stream(keys + en, pstream) : ~0ull;
        no = vn ? ld_stream(outidx + en, pstream) : 0;
        nx = vn ? ld_stream(vals + en, pstream) : VT(0);
      }
      uint64_t prev = __shfl_up_sync(0xffffffffu, key, 1, SW);
      if (sl == 0) prev = last_key;
      const bool lead = valid && key != prev;
      const unsigned lm = __ballot_sync(0xffffffffu, lead);
      const unsigned vm = __ballot_sync(0xffffffffu, valid);
      if (vm == 0u) break;
      uint32_t id[DM];
      {
        uint64_t t = key;
#pragma unroll
        for (int m = 0; m < DM; ++m) {
          uint64_t rem;
          t = divmod_fast(t, fd.n[m], fd.inv[m], rem, fd.fast);
          id[m] = (uint32_t)rem;
        }
      }
      last_key = __shfl_sync(0xffffffffu, key, sbase + SW - 1);
#pragma unroll
      for (int t0 = 0; t0 < SW; t0 += U) {
        double av[U][4];
        double hv[U][DM > 1 ? DM - 1 : 1][4];
        double gv[U][4];
        bool lead_[U], slow_[U];
        uint32_t sid[U];
        double xv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int src = sbase + t0 + u;
          const bool ok = (vm >> src) & 1u;
          lead_[u] = (lm >> src) & 1u;
          const int ou = __shfl_sync(0xffffffffu, o, src);
          xv[u] = __shfl_sync(0xffffffffu, x, src);
          const double2 *row = reinterpret_cast<const double2 *>(Ak + (int64_t)ou * ld + c0);
          double2 p0 = make_double2(0.0, 0.0), p1 = make_double2(0.0, 0.0);
#if CPARLS_FIT_LD256
          if (ok && colok)
            asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
                : "=d"(p0.x), "=d"(p0.y), "=d"(p1.x), "=d"(p1.y) : "l"(row));
#else
          if (ok && colok) { p0 = __ldg(row); p1 = __ldg(row + 1); }
#endif
          av[u][0] = p0.x; av[u][1] = p0.y; av[u][2] = p1.x; av[u][3] = p1.y;
#pragma unroll
          for (int m = 0; m + 1 < DM; ++m) {
            const uint32_t im = __shfl_sync(0xffffffffu, id[m], src);
            const double2 *hr = reinterpret_cast<const double2 *>(fd.A[m] + (int64_t)im * ld + c0);
            double2 q0 = make_double2(0.0, 0.0), q1 = make_double2(0.0, 0.0);
#if CPARLS_FIT_LD256
            if (lead_[u] && colok)
              asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
                  : "=d"(q0.x), "=d"(q0.y), "=d"(q1.x), "=d"(q1.y) : "l"(hr));
#else
            if (lead_[u] && colok) { q0 = __ldg(hr); q1 = __ldg(hr + 1); }
#endif
            hv[u][m][0] = q0.x; hv[u][m][1] = q0.y; hv[u][m][2] = q1.x; hv[u][m][3] = q1.y;
          }
          sid[u] = __shfl_sync(0xffffffffu, id[DM - 1], src);
          slow_[u] = lead_[u] && sid[u] != (u == 0 ? cur_slow : sid[u - 1]);
          {
            const double2 *gr = reinterpret_cast<const double2 *>(Aslow + (int64_t)sid[u] * ld + c0);
            double2 q0 = make_double2(0.0, 0.0), q1 = make_double2(0.0, 0.0);
            if (slow_[u] && colok) { q0 = __ldg(gr); q1 = __ldg(gr + 1); }
            gv[u][0] = q0.x; gv[u][1] = q0.y; gv[u][2] = q1.x; gv[u][3] = q1.y;
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (slow_[u]) {
#pragma unroll
            for (int q = 0; q < 4; ++q) g[q] = lam4[q] * gv[u][q];
          }
          if (lead_[u]) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              double hh = g[q];
#pragma unroll
              for (int m = 0; m + 1 < DM; ++m) hh *= hv[u][m][q];
              h[q] = hh;
            }
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) cacc[q] = fma(xv[u] * av[u][q], h[q], cacc[q]);
        }
        // g now belongs to the fiber of the batch's last entry
        if ((vm >> (sbase + t0 + U - 1)) & 1u) cur_slow = sid[U - 1];
      }
    }
    acc = dd_add_d(acc, (cacc[0] + cacc[1]) + (cacc[2] + cacc[3]));
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

// <X,M> from block partials; ||M||^2 = lambda^T (*_m G_m) lambda with the
// factors' Grams G_m (P:146-148 structure); fit = 1 - sqrt(max(0, ||X||^2 -
// 2<X,M> + ||M||^2)) / ||X|| (AMB-16).
struct FitModes {
  int D;
  const double *GA[kMaxModes];
};

__global__ void k_fit_final(const dd *__restrict__ part, int nb, FitModes fm, const double *__restrict__ lam, int r,
                            double normX2, double *out, const StepCtl *ctl = nullptr) {
  CPARLS_GUARD(ctl);
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
