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

// 16-byte variants for an even tile stride S (rows 16-byte aligned; ld is a
// multiple of 4): one 16-byte shared store / load per 16-byte global access
__device__ __forceinline__ void stage_rows_v(const double *__restrict__ src, int rows, int ld, double *tile, int S) {
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
        *reinterpret_cast<double2 *>(tile + row * S + c) = v[u];
      }
    }
  }
}

__device__ __forceinline__ void store_rows_v(double *__restrict__ dst, int rows, int ld, const double *tile, int S) {
  double2 *d2 = reinterpret_cast<double2 *>(dst);
  const int n2 = rows * ld / 2;
  for (int i = threadIdx.x; i < n2; i += blockDim.x) {
    const int e = 2 * i, row = e / ld, c = e - row * ld;
    d2[i] = *reinterpret_cast<const double2 *>(tile + row * S + c);
  }
}

// ---------------------------------------------------------------- factor Gram
// Block partials of sum_i w_i a_i a_i^T over the rows of A (w = null: unit
// weights): the factor Gram, and the sampled Gram Z^T diag(w^2) Z (P:683,
// P:900-901) with n = s_bar read on the device.
template <int RMAX>
__global__ void __launch_bounds__(kRowThreads) k_gram_rows_t(const double *__restrict__ A, int64_t n, int r, int ld,
                                                            double *__restrict__ part,
                                                            const double *__restrict__ w = nullptr,
                                                            const int64_t *n_dev = nullptr,
                                                            const StepCtl *ctl = nullptr) {
  CPARLS_GUARD(ctl);
  n = dcount(n, n_dev);
  extern __shared__ double smem[];
  const int S = ld + 1;
  double *tile = smem;
  double *wt = smem + kRowThreads * S;
  Syrk<RMAX> sy;
  sy.init(r);
  const int64_t ntiles = ceil_div(n, kRowThreads);
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t base = t * kRowThreads;
    const int rows = (int)min((int64_t)kRowThreads, n - base);
    __syncthreads();
    stage_rows(A + base * ld, rows, ld, tile, S);
    if (w && (int)threadIdx.x < rows) wt[threadIdx.x] = w[base + threadIdx.x];
    __syncthreads();
    sy.accumulate(tile, rows, S, w ? wt : nullptr);
  }
  __syncthreads();
  sy.finish(r, smem, part + (int64_t)blockIdx.x * r * r);
}

// ---------------------------------------------------------------- solve rows
// B_i = M_i G^+ (rows with M_i = 0 give 0), M zeroed behind the read,
// block partial of B^T B (column norms lambda, and the normalized
// factor's Gram).
template <int RMAX>
__global__ void __launch_bounds__(kRowThreads) k_solve_rows_t(double *__restrict__ M, int64_t n, int r, int ld,
                                                             const SolveDev *__restrict__ sd, double *__restrict__ B,
                                                             double *__restrict__ part,
                                                             unsigned long long *__restrict__ touched,
                                                             int zero_m, const double *__restrict__ fscale,
                                                             const StepCtl *ctl = nullptr) {
  CPARLS_GUARD(ctl);
  extern __shared__ __align__(16) double smem[];
  const int S = ld + 2;              // even: 16-byte aligned rows, conflict-free 16-byte row accesses
  double *Gi = smem;                 // G^+ with row stride ld (zero padded): 16-byte operand loads
  double *tile = smem + r * ld;
  for (int i = threadIdx.x; i < r * ld; i += blockDim.x) {
    const int p = i / ld, c = i - p * ld;
    Gi[i] = c < r ? sd->Ginv[p * r + c] : 0.0;
  }
  const bool fixed = fscale != nullptr && fscale[2 * kMaxRank] != 0.0;
  Syrk<RMAX> sy;
  sy.init(r);
  unsigned long long ntouch = 0;
  const int64_t ntiles = ceil_div(n, kRowThreads);
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t base = t * kRowThreads;
    const int rows = (int)min((int64_t)kRowThreads, n - base);
    __syncthreads();
    stage_rows_v(M + base * ld, rows, ld, tile, S);
    if (zero_m) {   // keep M zero for the next atomic RHS (the bucketed RHS overwrites every row)
      double2 *d2 = reinterpret_cast<double2 *>(M + base * ld);
      for (int i = threadIdx.x; i < rows * ld / 2; i += blockDim.x) d2[i] = make_double2(0.0, 0.0);
    }
    __syncthreads();
    if (threadIdx.x < rows) {
      double *x = tile + threadIdx.x * S;
      double m[RMAX];
      bool nz = false;
#pragma unroll
      for (int c = 0; c < RMAX; c += 2) {
        const double2 v2 = *reinterpret_cast<const double2 *>(x + c);
        double v0 = (c < r) ? v2.x : 0.0, v1 = (c + 1 < r) ? v2.y : 0.0;
        if (fixed) {   // fixed-point RHS: int64 count of 2^-e_c
          if (c < r) v0 = (double)__double_as_longlong(v0) * fscale[kMaxRank + c];
          if (c + 1 < r) v1 = (double)__double_as_longlong(v1) * fscale[kMaxRank + c + 1];
        }
        m[c] = v0;
        if (c + 1 < RMAX) m[c + 1] = v1;
        nz |= (v0 != 0.0) | (v1 != 0.0);
      }
      if (nz) {
        ++ntouch;
        // four output columns per pass: four independent FMA chains
        for (int c = 0; c < r; c += 4) {
          double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
          for (int p = 0; p < RMAX; ++p)
            if (p < r) {
              const double2 g01 = *reinterpret_cast<const double2 *>(Gi + p * ld + c);
              const double2 g23 = *reinterpret_cast<const double2 *>(Gi + p * ld + c + 2);
              s0 += m[p] * g01.x;
              s1 += m[p] * g01.y;
              s2 += m[p] * g23.x;
              s3 += m[p] * g23.y;
            }
          // columns >= r come out 0 (zero-padded G^+): the padding stays zero
          *reinterpret_cast<double2 *>(x + c) = make_double2(s0, s1);
          *reinterpret_cast<double2 *>(x + c + 2) = make_double2(s2, s3);
        }
      }
    }
    __syncthreads();
    store_rows_v(B + base * ld, rows, ld, tile, S);
    sy.accumulate_v(tile, rows, S);
  }
  unsigned long long nt = warp_sum<unsigned long long>(ntouch);
  if ((threadIdx.x & 31) == 0 && nt) atomicAdd(touched, nt);
  __syncthreads();
  sy.finish(r, smem, part + (int64_t)blockIdx.x * r * r);
}

// ---------------------------------------------------------------- warp-tiled row passes
// The leverage pass (normalize, l_i, p~, q) has no cross-row reduction besides
// integer/max atomics, so every warp owns 32-row tiles end to end: coalesced
// 16-byte loads of 32 contiguous rows into a private smem tile, thread-per-row
// compute, coalesced stores, no block barriers inside the loop (the
// block-synchronous stage -> compute -> store version reached ~13% of HBM
// bandwidth: every phase waited for the slowest warp).
constexpr int kWarpRows = 32;

// Tiles use stride S = ld + 2 (even, so 16-byte aligned rows; conflict-free
// 16-byte loads when lane t reads row t) and the r x r operands use row stride
// ld (a multiple of 4), so every shared-memory access below is 16 bytes wide.
__host__ __device__ constexpr int warp_tile_stride(int ld) { return ld + 2; }

// contiguous rows [0, rows) of an ld-strided matrix <-> a warp's tile (stride S).
// 16-byte chunk i = lane + 32u holds doubles e = 2i, 2i+1 of row e / ld; the
// (row, column) of the next chunk of a lane advances by 64 doubles, so it is
// updated incrementally instead of dividing by the runtime ld.
struct ChunkWalk {
  int row, c, drow, dc, ld;
  __device__ __forceinline__ ChunkWalk(int lane, int ld_) : ld(ld_) {
    row = (2 * lane) / ld; c = 2 * lane - row * ld;
    drow = 64 / ld; dc = 64 - drow * ld;
  }
  __device__ __forceinline__ void next() {
    row += drow; c += dc;
    if (c >= ld) { c -= ld; ++row; }
  }
};

__device__ __forceinline__ void warp_stage(const double *__restrict__ src, int rows, int ld, double *tile, int S,
                                           double *zero_after) {
  const int lane = threadIdx.x & 31;
  const double2 *s2 = reinterpret_cast<const double2 *>(src);
  const int n2 = rows * ld / 2;
  constexpr int U = 7;
  ChunkWalk cw(lane, ld);
  for (int i0 = lane; i0 < n2; i0 += 32 * U) {
    double2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 + 32 * u;
      v[u] = i < n2 ? __ldg(s2 + i) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 + 32 * u;
      if (i < n2) {
        *reinterpret_cast<double2 *>(tile + cw.row * S + cw.c) = v[u];
        if (zero_after) reinterpret_cast<double2 *>(zero_after)[i] = make_double2(0.0, 0.0);
      }
      cw.next();
    }
  }
}
__device__ __forceinline__ void warp_store(double *__restrict__ dst, int rows, int ld, const double *tile, int S) {
  const int lane = threadIdx.x & 31;
  double2 *d2 = reinterpret_cast<double2 *>(dst);
  const int n2 = rows * ld / 2;
  ChunkWalk cw(lane, ld);
  for (int i = lane; i < n2; i += 32) {
    d2[i] = *reinterpret_cast<const double2 *>(tile + cw.row * S + cw.c);
    cw.next();
  }
}

// The tile of warp_stage as 16-byte cp.async copies (no registers, the data
// lands while the warp computes on its other tile); chunks past `rows` rows
// are not copied (the consumers read rows < rows only).
__device__ __forceinline__ void warp_stage_async(const double *__restrict__ src, int rows, int ld, double *tile,
                                                 int S) {
  const int lane = threadIdx.x & 31;
  const double2 *s2 = reinterpret_cast<const double2 *>(src);
  const int n2 = rows * ld / 2;
  ChunkWalk cw(lane, ld);
  for (int i = lane; i < n2; i += 32) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(tile + cw.row * S + cw.c);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(s2 + i) : "memory");
    cw.next();
  }
}
__device__ __forceinline__ void warp_zero(double *__restrict__ dst, int rows, int ld) {
  const int lane = threadIdx.x & 31;
  double2 *d2 = reinterpret_cast<double2 *>(dst);
  const int n2 = rows * ld / 2;
  for (int i = lane; i < n2; i += 32) d2[i] = make_double2(0.0, 0.0);
}

// p~_i = ||a_i W||^2 / rank of one normalized row x (16-byte aligned, r columns)
// with W (RMAX x RMAX, zero padded; zero below the diagonal if tri): s_c =
// sum_{k < r} a_k W_kc, l = sum_c s_c^2.  One definition for the leverage pass
// and the fused solve + leverage pass, so both give the same bits.
template <int RMAX>
__device__ __forceinline__ double lev_of_row(const double *x, int r, const double *W, int tri, int rank) {
  if (tri == 2) return 1.0 / (double)rank;   // full row rank, nk < r: the hat matrix is I
  double a[RMAX];
#pragma unroll
  for (int c = 0; c < RMAX; c += 2) {
    const double2 v = *reinterpret_cast<const double2 *>(x + c);
    a[c] = (c < r) ? v.x : 0.0;
    if (c + 1 < RMAX) a[c + 1] = (c + 1 < r) ? v.y : 0.0;
  }
  double l = 0.0;
  if (rank > 0) {
    // s_c = sum_{k < r} a_k W_kc over the zero-padded W (an upper
    // triangular W's zeros below the diagonal leave the sums unchanged)
    for (int c = 0; c < r; c += 4) {
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
      for (int k = 0; k < RMAX; ++k)
        if (k < r && (!tri || k <= c + 3)) {
          const double2 w01 = *reinterpret_cast<const double2 *>(W + k * RMAX + c);
          const double2 w23 = *reinterpret_cast<const double2 *>(W + k * RMAX + c + 2);
          s0 += a[k] * w01.x;
          s1 += a[k] * w01.y;
          s2 += a[k] * w23.x;
          s3 += a[k] * w23.y;
        }
      l += s0 * s0;
      if (c + 1 < r) l += s1 * s1;
      if (c + 2 < r) l += s2 * s2;
      if (c + 3 < r) l += s3 * s3;
    }
  }
  return rank > 0 ? l / (double)rank : 0.0;
}

// l_i = ||a_i W||^2, p~_i = l_i / rank, q_i = rint(p~_i 2^62) into C, q summed
// into the 256-row tile sums of the CDF scan (integer adds: order-free, exact);
// lam != nullptr normalizes A in place first (a_ic = b_ic * (1/lambda_c),
// within 1 ulp of the division, which cost ~10 FP64 instructions per element).
#ifndef CPARLS_LEV_MINB
#define CPARLS_LEV_MINB 2   // resident CTAs per SM the leverage pass is compiled for
#endif
#ifndef CPARLS_SOLVE_MINB
#define CPARLS_SOLVE_MINB 2   // resident CTAs per SM the DMMA solve pass is compiled for
#endif
template <int RMAX>
__global__ void __launch_bounds__(kRowThreads, CPARLS_LEV_MINB) k_lev_rows_w(double *__restrict__ A, int64_t n, int r, int ld,
                                                              const double *__restrict__ lam,
                                                              const ModeDev *__restrict__ md, double *__restrict__ pt,
                                                              uint64_t *__restrict__ C,
                                                              unsigned long long *__restrict__ tile_sum,
                                                              double *alpha_out,
                                                              unsigned long long *drawable_out,
                                                              const StepCtl *ctl = nullptr) {
  CPARLS_GUARD(ctl);
  extern __shared__ __align__(16) double smem[];
  const int S = warp_tile_stride(ld);
  double *W = smem;                  // RMAX x RMAX, zero padded (and zero below the diagonal if tri)
  double *lam_s = smem + RMAX * RMAX;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double *tile = lam_s + kMaxRank + (size_t)w * kWarpRows * S;
  const int tri = md->tri, rank = md->rank;
  for (int i = threadIdx.x; i < RMAX * RMAX; i += blockDim.x) {
    const int k = i / RMAX, c = i - k * RMAX;
    W[i] = (k < r && c < r && tri < 2 && (!tri || k <= c)) ? md->W[k * r + c] : 0.0;
  }
  // 1 / lambda_c (0 for a zero column): one multiply per element instead of a division
  for (int i = threadIdx.x; i < RMAX; i += blockDim.x)
    lam_s[i] = (lam != nullptr && i < r) ? (lam[i] > 0.0 ? 1.0 / lam[i] : 0.0) : 1.0;
  __syncthreads();
  double pmax = 0.0;
  unsigned long long dcnt = 0;
  const int64_t ntiles = ceil_div(n, kWarpRows);
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t t = (int64_t)blockIdx.x * (blockDim.x >> 5) + w; t < ntiles; t += nwarps) {
    const int64_t base = t * kWarpRows;
    const int rows = (int)min((int64_t)kWarpRows, n - base);
    warp_stage(A + base * ld, rows, ld, tile, S, nullptr);
    __syncwarp();
    if (lam != nullptr) {
      for (int i = lane; i < rows * ld; i += 32) {
        const int row = i / ld, c = i - row * ld;
        if (c < r) tile[row * S + c] *= lam_s[c];
      }
      __syncwarp();
      warp_store(A + base * ld, rows, ld, tile, S);
    }
    uint64_t q = 0;
    if (lane < rows) {
      const double p = lev_of_row<RMAX>(tile + lane * S, r, W, tri, rank);
      q = __double2ull_rn(p * kTwo62);
      pt[base + lane] = p;
      C[base + lane] = q;
      pmax = fmax(pmax, p);
      dcnt += (p > 1.0842021724855044e-19);
    }
    const unsigned long long qs = warp_sum<unsigned long long>(q);
    if (lane == 0 && qs) atomicAdd(tile_sum + (base >> 8), qs);   // 256-row CDF tiles (kLevThreads)
    __syncwarp();
  }
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) pmax = fmax(pmax, __shfl_xor_sync(0xffffffffu, pmax, m));
  dcnt = warp_sum<unsigned long long>(dcnt);
  if (lane == 0) {
    atomic_max_nonneg(alpha_out, pmax);
    if (dcnt) atomicAdd(drawable_out, dcnt);
  }
}

// ---------------------------------------------------------------- solve on FP64 tensor cores
// B = M G^+ and the block partial of B^T B with DMMA (mma.sync m8n8k4 f64)
// for ld = 8 NT <= 32 (r in 5..32).  k_solve_rows_t streams G^+ operands from
// shared memory for every row and FMA (ncu: LSU/smem wavefronts ~70%, FP64
// pipe ~23%); here a warp owns 32-row tiles: per 8-row slab the M fragments
// are loaded once (fixed-point M converted on load), D = M G^+ takes
// 2 NT^2 x 4 DMMAs with G^+ fragments read from shared memory, and the SYRK
// B^T B accumulates the NT(NT+1)/2 upper 8x8 tiles in registers (one DMMA per
// tile per 4 rows).  Fragment layout (m8n8k4, f64): A[g][t], B[t][g],
// C[g][2t..2t+1] with g = lane/4, t = lane%4.  Per-warp partials are summed in
// a fixed order: the result is deterministic.
__device__ __forceinline__ void dmma_884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// PIPE (round 2): two tiles per warp, the next one's M rows in flight
// (cp.async) while the current one is multiplied and stored; one CTA per SM
// (the tiles take ~140 KB of shared memory), grid = SMs.  C4: 0.611 -> 0.566
// ms per launch.  (The same pipeline in k_lev_rows_w measured slower, 0.514 ->
// 0.622 ms: its per-row quadratic forms want the 16 warps per SM of two CTAs.)
#ifndef CPARLS_SOLVE_PIPE
#define CPARLS_SOLVE_PIPE 1
#endif
__host__ __device__ constexpr size_t solve_dmma_smem_d(int LD, bool pipe = false) {
  return (size_t)LD * LD + LD + (pipe ? 2 : 1) * (size_t)(kRowThreads / 32) * kWarpRows * (LD + 2) + 64;
}

template <int NT, bool PIPE = false>
__global__ void __launch_bounds__(kRowThreads, PIPE ? 1 : CPARLS_SOLVE_MINB) k_solve_dmma(double *__restrict__ M, int64_t n, int r, int ld,
                                                               const SolveDev *__restrict__ sd,
                                                               double *__restrict__ B, double *__restrict__ part,
                                                               unsigned long long *__restrict__ touched, int zero_m,
                                                               const double *__restrict__ fscale,
                                                               const StepCtl *ctl = nullptr) {
  CPARLS_GUARD(ctl);
  constexpr int LD = NT * 8, KS = NT * 2, NP = NT * (NT + 1) / 2;
  constexpr int S = LD + 2;   // even: 16-byte aligned tile rows
  extern __shared__ __align__(16) double smem[];
  double *Gs = smem;          // LD x LD, G^+ zero padded
  double *fs = Gs + LD * LD;  // 2^-e_c (fixed-point RHS) or 1
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, gid = lane >> 2, tig = lane & 3;
  double *tile0 = fs + LD + (size_t)w * (PIPE ? 2 : 1) * kWarpRows * S;
  double *tile = tile0;
  const bool fixed = fscale != nullptr && fscale[2 * kMaxRank] != 0.0;
  for (int i = threadIdx.x; i < LD * LD; i += blockDim.x) {
    const int p = i / LD, c = i - p * LD;
    Gs[i] = (p < r && c < r) ? sd->Ginv[p * r + c] : 0.0;
  }
  for (int i = threadIdx.x; i < LD; i += blockDim.x) fs[i] = (fixed && i < r) ? fscale[kMaxRank + i] : 1.0;
  __syncthreads();
  double sacc[NP][2];
#pragma unroll
  for (int q = 0; q < NP; ++q) sacc[q][0] = sacc[q][1] = 0.0;
  unsigned long long ntouch = 0;
  const int64_t ntiles = ceil_div(n, kWarpRows);
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t tfirst = (int64_t)blockIdx.x * (blockDim.x >> 5) + w;
  if (PIPE && tfirst < ntiles) {
    warp_stage_async(M + tfirst * kWarpRows * ld, (int)min((int64_t)kWarpRows, n - tfirst * kWarpRows), ld, tile0, S);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  }
  int buf = 0;
  for (int64_t t = tfirst; t < ntiles; t += nwarps) {
    const int64_t base = t * kWarpRows;
    const int rows = (int)min((int64_t)kWarpRows, n - base);
    if (PIPE) {
      tile = tile0 + (size_t)buf * kWarpRows * S;
      const int64_t tn = t + nwarps;
      if (tn < ntiles)
        warp_stage_async(M + tn * kWarpRows * ld, (int)min((int64_t)kWarpRows, n - tn * kWarpRows), ld,
                         tile0 + (size_t)(buf ^ 1) * kWarpRows * S, S);
      asm volatile("cp.async.commit_group;\n" ::: "memory");
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");   // this tile's rows have landed
      __syncwarp();
      if (zero_m) warp_zero(M + base * ld, rows, ld);
      buf ^= 1;
    } else {
      warp_stage(M + base * ld, rows, ld, tile, S, zero_m ? M + base * ld : nullptr);
    }
    __syncwarp();
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const int row = m * 8 + gid;
      double a[KS];
      bool nzr = false;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const int c = ks * 4 + tig;
        double v = row < rows ? tile[row * S + c] : 0.0;
        if (fixed) v = (double)__double_as_longlong(v) * fs[c];
        a[ks] = v;
        nzr |= (v != 0.0);
      }
      unsigned f = nzr;
      f |= __shfl_xor_sync(0xffffffffu, f, 1);
      f |= __shfl_xor_sync(0xffffffffu, f, 2);
      if (tig == 0 && f) ++ntouch;
      double d[NT][2];
#pragma unroll
      for (int nn = 0; nn < NT; ++nn) d[nn][0] = d[nn][1] = 0.0;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks)
#pragma unroll
        for (int nn = 0; nn < NT; ++nn) dmma_884(d[nn], a[ks], Gs[(ks * 4 + tig) * LD + nn * 8 + gid]);
      __syncwarp();   // every lane has read its M fragments of this slab
#pragma unroll
      for (int nn = 0; nn < NT; ++nn)
        *reinterpret_cast<double2 *>(tile + row * S + nn * 8 + 2 * tig) = make_double2(d[nn][0], d[nn][1]);
    }
    __syncwarp();
    warp_store(B + base * ld, rows, ld, tile, S);
    // B^T B over this tile's rows (rows >= `rows` are zero)
#pragma unroll
    for (int ks = 0; ks < kWarpRows / 4; ++ks) {
      const double *xr = tile + (ks * 4 + tig) * S + gid;
      double v[NT];
#pragma unroll
      for (int tq = 0; tq < NT; ++tq) v[tq] = xr[tq * 8];
      int pi = 0;
#pragma unroll
      for (int p = 0; p < NT; ++p)
#pragma unroll
        for (int q = p; q < NT; ++q) dmma_884(sacc[pi++], v[p], v[q]);
    }
    __syncwarp();
  }
  if (PIPE) asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  unsigned long long nt = warp_sum<unsigned long long>(ntouch);
  if (lane == 0 && nt) atomicAdd(touched, nt);
  __syncthreads();
  // per-warp partials -> block partial (upper triangle), fixed summation order
  double *red = smem;   // 8 x LD x LD (fits in the tiles' space)
  {
    int pi = 0;
#pragma unroll
    for (int p = 0; p < NT; ++p)
#pragma unroll
      for (int q = p; q < NT; ++q, ++pi) {
        double *dst = red + (size_t)w * LD * LD + (p * 8 + gid) * LD + q * 8 + 2 * tig;
        dst[0] = sacc[pi][0];
        dst[1] = sacc[pi][1];
      }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < r * r; i += blockDim.x) {
    const int p = i / r, q = i - p * r;
    if (p > q) continue;
    double sum = 0.0;
    for (int ww = 0; ww < (int)(blockDim.x >> 5); ++ww) sum += red[(size_t)ww * LD * LD + p * LD + q];
    part[(int64_t)blockIdx.x * r * r + i] = sum;
  }
}


// ---------------------------------------------------------------- KrpSamp
// z_j = A_{m_1}(i_1,:) * ... * A_{m_d}(i_d,:) (eq:Zrow P:214, left to right)
// into Z (s_bar x ld, padding zero), and the block partial of the column sums
// sum_j w_j^2 |z_j| (fixed-point RHS scales, k_gram_scales).  A warp forms QR
// rows at once: all QR x d index decodes first, then all QR x d row loads in
// flight together, then the products (DM >= d modes, unrolled).  Low register
// use, so 64 warps per SM hide the gather latency; the sampled Gram
// sum_j w_j^2 z_j z_j^T is a separate streaming pass over Z (k_gram_rows_t).
constexpr int kKrpThreads = 256;
constexpr int kKrpBlocks = 148 * 4;   // upper bound of k_krp_rows' grid (cpart partials)

template <int DM, int QR, bool HI>
__global__ void __launch_bounds__(kKrpThreads, DM * QR > 8 ? 3 : 4) k_krp_rows(const uint64_t *__restrict__ skey,
                                                         const double *__restrict__ sw2, int64_t sbar,
                                                         OtherModes om, int r, int ld, double *__restrict__ Z,
                                                         double *__restrict__ cpart, const int64_t *sbar_dev,
                                                         const StepCtl *ctl, const double *__restrict__ zg) {
  CPARLS_GUARD(ctl);
  sbar = dcount(sbar, sbar_dev);
  __shared__ double cabs_red[kKrpThreads / 32][64];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t nw = (int64_t)gridDim.x * (kKrpThreads / 32);
  double ca0 = 0.0, ca1 = 0.0;   // this lane's column sums of w^2 |z|
  const int d = om.d;
  for (int64_t j0 = ((int64_t)blockIdx.x * (kKrpThreads / 32) + w) * QR; j0 < sbar; j0 += nw * QR) {
    const double *rowp[QR][DM];
#pragma unroll
    for (int q = 0; q < QR; ++q) {
      const int64_t j = min(j0 + q, sbar - 1);
      uint64_t key = skey[j];
#pragma unroll
      for (int m = 0; m < DM; ++m) {
        if (m < d) {
          uint64_t i;
          key = fastdivmod(key, om.div[m], i);
          // sharded run: the rows come from their owners (zg, sample-major, d rows per sample)
          rowp[q][m] = zg ? zg + (j * (int64_t)d + m) * ld : om.A[m] + i * ld;
        }
      }
    }
    double a0[QR][DM], a1[QR][HI ? DM : 1];
#pragma unroll
    for (int q = 0; q < QR; ++q)
#pragma unroll
      for (int m = 0; m < DM; ++m) {
        a0[q][m] = m < d && lane < r ? __ldg(rowp[q][m] + lane) : 1.0;
        if (HI) a1[q][HI ? m : 0] = m < d && lane + 32 < r ? __ldg(rowp[q][m] + lane + 32) : 1.0;
      }
#pragma unroll
    for (int q = 0; q < QR; ++q) {
      const int64_t j = j0 + q;
      if (j >= sbar) break;
      double z0 = a0[q][0], z1 = HI ? a1[q][0] : 0.0;
#pragma unroll
      for (int m = 1; m < DM; ++m)
        if (m < d) { z0 *= a0[q][m]; if (HI) z1 *= a1[q][HI ? m : 0]; }
      z0 = lane < r ? z0 : 0.0;
      z1 = lane + 32 < r ? z1 : 0.0;
      if (lane < ld) Z[j * ld + lane] = z0;
      if (lane + 32 < ld) Z[j * ld + lane + 32] = z1;
      if (cpart) {
        const double wq = __ldg(sw2 + j);
        ca0 += wq * fabs(z0);
        ca1 += wq * fabs(z1);
      }
    }
  }
  if (cpart) {   // block partial of sum_j w_j^2 |z_j| per column, warps in order
    cabs_red[w][lane] = ca0;
    cabs_red[w][lane + 32] = ca1;
    __syncthreads();
    if (threadIdx.x < r) {
      double t = 0.0;
      for (int g = 0; g < kKrpThreads / 32; ++g) t += cabs_red[g][threadIdx.x];
      cpart[(int64_t)blockIdx.x * r + threadIdx.x] = t;
    }
  }
}

}  // namespace cparls
