// rows.cuh -- row-streaming kernels over n_k x r fp64 factor-shaped matrices:
// factor Gram, leverage/p~/q (K1/K2), B = M G^+ with B^T B (K9), and the
// sampled-KRP Gram (K6).  Rows are staged through shared memory with
// coalesced loads, then held in registers (RMAX-templated, fully unrolled), so
// the r x r products read only broadcast shared-memory operands.
#pragma once
#include "common.cuh"
#include "prims.cuh"
#include "syrk.cuh"

namespace cparls {

constexpr int kRowThreads = 256;   // rows per tile = threads per block

// stage rows [base, base+rows) of a (ld-strided) matrix into tile (stride S);
// 4 independent 16-byte loads in flight per thread
__device__ __forceinline__ void stage_rows(const double *__restrict__ src, int rows, int ld, double *tile, int S) {
  const double2 *s2 = reinterpret_cast<const double2 *>(src);
  const int n2 = rows * ld / 2;
  const int B = blockDim.x;
  for (int i0 = threadIdx.x; i0 < n2; i0 += 4 * B) {
    double2 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u * B;
      v[u] = i < n2 ? __ldg(s2 + i) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u * B;
      if (i < n2) {
        const int e = 2 * i, row = e / ld, c = e - row * ld;
        tile[row * S + c] = v[u].x;
        tile[row * S + c + 1] = v[u].y;
      }
    }
  }
}

__device__ __forceinline__ void store_rows(double *__restrict__ dst, int rows, int ld, const double *tile, int S) {
  double2 *d2 = reinterpret_cast<double2 *>(dst);
  const int n2 = rows * ld / 2;
  for (int i = threadIdx.x; i < n2; i += blockDim.x) {
    const int e = 2 * i, row = e / ld, c = e - row * ld;
    d2[i] = make_double2(tile[row * S + c], tile[row * S + c + 1]);
  }
}

// ---------------------------------------------------------------- factor Gram
template <int RMAX>
__global__ void __launch_bounds__(kRowThreads) k_gram_rows_t(const double *__restrict__ A, int64_t n, int r, int ld,
                                                            double *__restrict__ part) {
  extern __shared__ double smem[];
  const int S = ld + 1;
  double *tile = smem;
  Syrk<RMAX> sy;
  sy.init(r);
  const int64_t ntiles = ceil_div(n, kRowThreads);
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t base = t * kRowThreads;
    const int rows = (int)min((int64_t)kRowThreads, n - base);
    __syncthreads();
    stage_rows(A + base * ld, rows, ld, tile, S);
    __syncthreads();
    sy.accumulate(tile, rows, S, nullptr);
  }
  __syncthreads();
  sy.finish(r, smem, part + (int64_t)blockIdx.x * r * r);
}

// ---------------------------------------------------------------- leverage rows
// l_i = ||a_i W||^2 (W = L^{-T} upper triangular, or V_kept mu^{-1/2}),
// p~_i = l_i / rank (AMB-11), q_i = rint(p~_i 2^62) (AMB-9)
// written to C (CDF pass 1), per-tile q sums, alpha = max p~, drawable count.
// lam != nullptr: normalize A in place first, a_i = b_i / lambda.
template <int RMAX>
__global__ void __launch_bounds__(kRowThreads) k_lev_rows_t(double *__restrict__ A, int64_t n, int r, int ld,
                                                           const double *__restrict__ lam,
                                                           const ModeDev *__restrict__ md, double *__restrict__ pt,
                                                           uint64_t *__restrict__ C, uint64_t *__restrict__ tile_sum,
                                                           double *alpha_out, unsigned long long *drawable_out) {
  extern __shared__ double smem[];
  const int S = ld + 1;
  double *W = smem;
  double *lam_s = smem + r * r;
  double *tile = lam_s + RMAX;
  const int tri = md->tri, rank = md->rank;
  for (int i = threadIdx.x; i < r * r; i += blockDim.x) W[i] = md->W[i];
  for (int i = threadIdx.x; i < RMAX; i += blockDim.x) lam_s[i] = (lam != nullptr && i < r) ? lam[i] : 1.0;
  double pmax = 0.0;
  unsigned long long dcnt = 0;
  __shared__ unsigned long long wq[kRowThreads / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t ntiles = ceil_div(n, kRowThreads);
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t base = t * kRowThreads;
    const int rows = (int)min((int64_t)kRowThreads, n - base);
    __syncthreads();
    stage_rows(A + base * ld, rows, ld, tile, S);
    __syncthreads();
    if (lam != nullptr) {
      for (int i = threadIdx.x; i < rows * ld; i += blockDim.x) {
        int row = i / ld, c = i - row * ld;
        if (c < r) {
          double l = lam_s[c];
          tile[row * S + c] = l > 0.0 ? tile[row * S + c] / l : 0.0;
        }
      }
      __syncthreads();
      store_rows(A + base * ld, rows, ld, tile, S);
    }
    uint64_t q = 0;
    if (threadIdx.x < rows) {
      const double *x = tile + threadIdx.x * S;
      double a[RMAX];
#pragma unroll
      for (int c = 0; c < RMAX; ++c) a[c] = (c < r) ? x[c] : 0.0;
      double l = 0.0;
      if (rank > 0) {
        // outer loop over output columns stays rolled (keeps W loads inside it);
        // the inner loop is unrolled so a[] lives in registers
        for (int c = 0; c < r; ++c) {
          const double *Wc = W + c;
          double s = 0.0;
#pragma unroll
          for (int k = 0; k < RMAX; ++k)
            if (k < r && (!tri || k <= c)) s += a[k] * Wc[k * r];
          l += s * s;
        }
      }
      double p = rank > 0 ? l / (double)rank : 0.0;
      q = __double2ull_rn(p * kTwo62);
      pt[base + threadIdx.x] = p;
      C[base + threadIdx.x] = q;
      pmax = fmax(pmax, p);
      dcnt += (p > 1.0842021724855044e-19);
    }
    unsigned long long qs = warp_sum<unsigned long long>(q);
    if (lane == 0) wq[w] = qs;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long s = 0;
      for (int i = 0; i < kRowThreads / 32; ++i) s += wq[i];
      tile_sum[t] = s;
    }
  }
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) pmax = fmax(pmax, __shfl_xor_sync(0xffffffffu, pmax, m));
  dcnt = warp_sum<unsigned long long>(dcnt);
  if (lane == 0) {
    atomic_max_nonneg(alpha_out, pmax);
    if (dcnt) atomicAdd(drawable_out, dcnt);
  }
}

// ---------------------------------------------------------------- solve rows
// B_i = M_i G^+ (rows with M_i = 0 give 0), M zeroed behind the read,
// block partial of B^T B (column norms lambda, and the normalized
// factor's Gram).
template <int RMAX>
__global__ void __launch_bounds__(kRowThreads) k_solve_rows_t(double *__restrict__ M, int64_t n, int r, int ld,
                                                             const SolveDev *__restrict__ sd, double *__restrict__ B,
                                                             double *__restrict__ part,
                                                             unsigned long long *__restrict__ touched) {
  extern __shared__ double smem[];
  const int S = ld + 1;
  double *Gi = smem;
  double *tile = smem + r * r;
  for (int i = threadIdx.x; i < r * r; i += blockDim.x) Gi[i] = sd->Ginv[i];
  Syrk<RMAX> sy;
  sy.init(r);
  unsigned long long ntouch = 0;
  const int64_t ntiles = ceil_div(n, kRowThreads);
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t base = t * kRowThreads;
    const int rows = (int)min((int64_t)kRowThreads, n - base);
    __syncthreads();
    stage_rows(M + base * ld, rows, ld, tile, S);
    {
      double2 *d2 = reinterpret_cast<double2 *>(M + base * ld);   // keep M zero for the next RHS
      for (int i = threadIdx.x; i < rows * ld / 2; i += blockDim.x) d2[i] = make_double2(0.0, 0.0);
    }
    __syncthreads();
    if (threadIdx.x < rows) {
      double *x = tile + threadIdx.x * S;
      double m[RMAX];
      bool nz = false;
#pragma unroll
      for (int c = 0; c < RMAX; ++c) {
        m[c] = (c < r) ? x[c] : 0.0;
        nz |= (m[c] != 0.0);
      }
      if (nz) {
        ++ntouch;
        for (int c = 0; c < r; ++c) {
          const double *Gc = Gi + c;
          double s = 0.0;
#pragma unroll
          for (int p = 0; p < RMAX; ++p)
            if (p < r) s += m[p] * Gc[p * r];
          x[c] = s;
        }
      }
    }
    __syncthreads();
    store_rows(B + base * ld, rows, ld, tile, S);
    sy.accumulate(tile, rows, S, nullptr);
  }
  unsigned long long nt = warp_sum<unsigned long long>(ntouch);
  if ((threadIdx.x & 31) == 0 && nt) atomicAdd(touched, nt);
  __syncthreads();
  sy.finish(r, smem, part + (int64_t)blockIdx.x * r * r);
}

// ---------------------------------------------------------------- KrpSamp + Gram
// z_j = A_{m_1}(i_1,:) * ... * A_{m_d}(i_d,:) (eq:Zrow P:214, left to right),
// Z (s_bar x ld, padding zero) and the block partial of sum_j w_j^2 z_j z_j^T.
template <int RMAX>
__global__ void __launch_bounds__(kRowThreads) k_krp_gram_t(const uint64_t *__restrict__ skey,
                                                           const double *__restrict__ sw2, int64_t sbar,
                                                           OtherModes om, int r, int ld, double *__restrict__ Z,
                                                           double *__restrict__ part) {
  extern __shared__ double smem[];
  const int S = ld + 1;
  double *tile = smem;
  double *wt = smem + kRowThreads * S;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  Syrk<RMAX> sy;
  sy.init(r);
  const int64_t ntiles = ceil_div(sbar, kRowThreads);
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t base = t * kRowThreads;
    const int rows = (int)min((int64_t)kRowThreads, sbar - base);
    __syncthreads();
    for (int jj = w; jj < rows; jj += kRowThreads / 32) {
      const int64_t j = base + jj;
      uint64_t key = skey[j];
      double z0 = 1.0, z1 = 1.0;
      for (int m = 0; m < om.d; ++m) {
        uint64_t i = key % (uint64_t)om.n[m];
        key /= (uint64_t)om.n[m];
        const double *row = om.A[m] + i * ld;
        if (lane < r) {
          double a = __ldg(row + lane);
          z0 = (m == 0) ? a : z0 * a;
        }
        if (lane + 32 < r) {
          double a = __ldg(row + lane + 32);
          z1 = (m == 0) ? a : z1 * a;
        }
      }
      double *x = tile + jj * S;
      if (lane < ld) x[lane] = lane < r ? z0 : 0.0;
      if (lane + 32 < ld) x[lane + 32] = lane + 32 < r ? z1 : 0.0;
      if (lane == 0) wt[jj] = sw2[j];
    }
    __syncthreads();
    store_rows(Z + base * ld, rows, ld, tile, S);
    sy.accumulate(tile, rows, S, wt);
  }
  __syncthreads();
  sy.finish(r, smem, part + (int64_t)blockIdx.x * r * r);
}

}  // namespace cparls
