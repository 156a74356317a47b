// kernels.cuh -- CP-ARLS-LEV hot-path kernels for sm_100a (B200).
// "P:L" cites /root/reference/PAPER.md line L; AMB-n cites DESIGN.md readings.
#pragma once
#include "common.cuh"
#include "prims.cuh"

namespace cparls {

// Per-mode device state written by the leverage preparation.
struct ModeDev {
  double alpha;            // max p~
  long long drawable;      // #{i : p~_i > 2^-63}  (rows whose integer weight q_i > 0)
  int rank;                // kept rank (AMB-11)
  int tri;                 // 1: W upper triangular (Cholesky); 0: full (eigen);
                           // 2: l_i = 1 (nk < r rows, full row rank; W unused)
  double W[kMaxRank * kMaxRank];   // l_i = || a_i W ||^2
  double GA[kMaxRank * kMaxRank];  // Gram of the (normalized) factor
};

// Per-solve device scalars.
struct SolveDev {
  double G[kMaxRank * kMaxRank];     // sampled Gram Z~^T Z~
  double Ginv[kMaxRank * kMaxRank];  // (pseudo-)inverse used for B = M G^+
  double BtB[kMaxRank * kMaxRank];
  double lambda[kMaxRank];
  double lambda_inv[kMaxRank];       // unused (division is used)
  int rank_used;
  int chol_fallback;
  long long touched;
};

__host__ __device__ constexpr int npairs(int r) { return r * (r + 1) / 2; }

// ======================================================================
// Small dense r x r linear algebra, single block (r <= 64)
// ======================================================================

// Parallel cyclic Jacobi eigensolver (round-robin ordering: R/2 disjoint
// rotations per round, A <- J^T A J, V <- V J), whole block.  a, V: shared
// r x r (row stride r).  Eigenvalues end on diag(a), vectors in V's columns.
// Convergence test as the oracle's: off^2 <= 1e-34 diag^2.
constexpr int kPrepThreads = 256;     // block of the single-block r x r kernels (k_*_prep)
constexpr double kCholSafe = 1e-6;   // Cholesky fast path only if every pivot > kCholSafe * max_diag

__device__ int block_jacobi(int r, double *a, double *V) {   // returns the sweeps taken
  __shared__ double cs[kMaxRank / 2 + 1], sn[kMaxRank / 2 + 1];
  __shared__ int pp[kMaxRank / 2 + 1], qq[kMaxRank / 2 + 1];
  __shared__ int done;
  const int R = (r + 1) & ~1;
  const int H = R / 2;
  for (int i = threadIdx.x; i < r * r; i += blockDim.x) V[i] = (i / r == i % r) ? 1.0 : 0.0;
  __syncthreads();
  __shared__ double red_off[32], red_diag[32];
  double prev_off = 0.0;
  int sweep = 0;
  for (; sweep < 60; ++sweep) {
    // off / diag: squared off-diagonal (upper) and diagonal sums, block-wide
    double off = 0.0, diag = 0.0;
    for (int i = threadIdx.x; i < r * r; i += blockDim.x) {
      const int p = i / r, q = i % r;
      const double x = a[i];
      if (p == q) diag += x * x;
      else if (q > p) off += x * x;
    }
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) {
      off += __shfl_xor_sync(0xffffffffu, off, m);
      diag += __shfl_xor_sync(0xffffffffu, diag, m);
    }
    if ((threadIdx.x & 31) == 0) { red_off[threadIdx.x >> 5] = off; red_diag[threadIdx.x >> 5] = diag; }
    __syncthreads();
    if (threadIdx.x == 0) {
      off = 0.0; diag = 0.0;
      for (int w = 0; w < (int)(blockDim.x + 31) / 32; ++w) { off += red_off[w]; diag += red_diag[w]; }
      // converged, or stagnating at the rounding floor (a rank-deficient G's
      // null-space block keeps off ~ (eps |G|)^2 from reaching 1e-34 |G|^2;
      // quadratic convergence otherwise cuts off far below a quarter per sweep)
      done = (off <= 1e-34 * diag || off == 0.0 || (sweep > 0 && off <= 1e-26 * diag && off > 0.25 * prev_off));
      prev_off = off;
    }
    __syncthreads();
    if (done) break;
    for (int t = 0; t < R - 1; ++t) {
      for (int i = threadIdx.x; i < H; i += blockDim.x) {
        int x = (i == 0) ? 0 : ((i - 1 + t) % (R - 1)) + 1;
        int yi = R - 1 - i;
        int y = ((yi - 1 + t) % (R - 1)) + 1;
        int p = min(x, y), q = max(x, y);
        double c = 1.0, sv = 0.0;
        if (q < r) {
          const double apq = a[p * r + q];
          if (apq != 0.0) {
            // t = tan of the angle zeroing a_pq: sgn(theta) / (|theta| + sqrt(theta^2 + 1))
            // with theta = d / (2 a_pq), d = a_qq - a_pp, as 2 a_pq sgn(d) / (|d| +
            // sqrt(d^2 + 4 a_pq^2)): one division and one square root
            const double d = a[q * r + q] - a[p * r + p], two = 2.0 * apq;
            const double tt = (d >= 0.0 ? two : -two) / (fabs(d) + sqrt(fma(d, d, two * two)));
            c = rsqrt(fma(tt, tt, 1.0));
            sv = tt * c;
          }
        }
        pp[i] = p; qq[i] = q; cs[i] = c; sn[i] = sv;
      }
      __syncthreads();
      // A <- J^T A J as independent 2x2 blocks (rows {p_i, q_i} x columns
      // {p_j, q_j}: row rotation i, then column rotation j, the same
      // operations as a row pass followed by a column pass) and V <- V J:
      // one pass, one barrier per round
      const int nblk = H * H;
      for (int idx = threadIdx.x; idx < nblk + H * r; idx += blockDim.x) {
        if (idx < nblk) {
          const int i = idx / H, j = idx - i * H;
          const int pi = pp[i], qi = qq[i], pj = pp[j], qj = qq[j];
          const bool vi = qi < r, vj = qj < r;   // q = r: the dummy of an odd r
          const bool ri = vi && sn[i] != 0.0, rj = vj && sn[j] != 0.0;
          if (!ri && !rj) continue;
          double x00 = a[pi * r + pj], x01 = vj ? a[pi * r + qj] : 0.0;
          double x10 = vi ? a[qi * r + pj] : 0.0, x11 = vi && vj ? a[qi * r + qj] : 0.0;
          if (ri) {
            const double c = cs[i], sv = sn[i];
            const double y00 = c * x00 - sv * x10, y10 = sv * x00 + c * x10;
            const double y01 = c * x01 - sv * x11, y11 = sv * x01 + c * x11;
            x00 = y00; x10 = y10; x01 = y01; x11 = y11;
          }
          if (rj) {
            const double c = cs[j], sv = sn[j];
            const double y00 = c * x00 - sv * x01, y01 = sv * x00 + c * x01;
            const double y10 = c * x10 - sv * x11, y11 = sv * x10 + c * x11;
            x00 = y00; x01 = y01; x10 = y10; x11 = y11;
          }
          a[pi * r + pj] = x00;
          if (vj) a[pi * r + qj] = x01;
          if (vi) a[qi * r + pj] = x10;
          if (vi && vj) a[qi * r + qj] = x11;
        } else {
          const int t2 = idx - nblk, j = t2 / r, k = t2 - j * r;
          const int p = pp[j], q = qq[j];
          if (q < r && sn[j] != 0.0) {
            const double c = cs[j], sv = sn[j];
            const double vkp = V[k * r + p], vkq = V[k * r + q];
            V[k * r + p] = c * vkp - sv * vkq;
            V[k * r + q] = sv * vkp + c * vkq;
          }
        }
      }
      __syncthreads();
    }
  }
  return sweep;
}

// Cholesky G = L L^T in shared memory.  Fast path of G^+ only: accepted when
// every pivot > kCholSafe * max_diag (G well conditioned, where Cholesky and the
// eigen pseudo-inverse agree to kappa*eps); otherwise the caller takes the
// eigen path whose cutoff mu_j > r*eps*mu_max defines the rank (AMB-11/12).
// Returns 1 on success.  L lower (row stride r).
// Whole block participates.
__device__ int block_cholesky(int r, const double *G, double *L, int *ok_flag) {
  // right-looking: L's lower triangle starts as G's and every column's
  // trailing update runs in parallel (O(r) barriers, O(1) work per thread per
  // step).  Entry (i, l) receives the subtractions L(i,q) L(l,q) for q = 0, 1,
  // ... in the same order and form as the column-by-column (left-looking)
  // formula, so the factor is bit-identical to it.
  __shared__ double maxdiag;
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int j = 0; j < r; ++j) m = fmax(m, G[j * r + j]);
    maxdiag = m;
    *ok_flag = m > 0.0;
  }
  for (int i = threadIdx.x; i < r * r; i += blockDim.x) L[i] = (i % r <= i / r) ? G[i] : 0.0;
  __syncthreads();
  for (int j = 0; j < r; ++j) {
    if (threadIdx.x == 0 && *ok_flag) {
      const double dj = L[j * r + j];
      if (!(dj > kCholSafe * maxdiag)) *ok_flag = 0;
      else L[j * r + j] = sqrt(dj);
    }
    __syncthreads();
    if (!*ok_flag) return 0;
    const double ljj = L[j * r + j];
    for (int i = j + 1 + threadIdx.x; i < r; i += blockDim.x) L[i * r + j] = L[i * r + j] / ljj;
    __syncthreads();
    const int t = r - j - 1;   // trailing block rows/cols j+1 .. r-1 (lower triangle)
    for (int idx = threadIdx.x; idx < t * t; idx += blockDim.x) {
      const int i = j + 1 + idx / t, l = j + 1 + idx % t;
      if (l <= i) L[i * r + l] -= L[i * r + j] * L[l * r + j];
    }
    __syncthreads();
  }
  return 1;
}

// Lower-triangular inverse Linv = L^{-1} (row stride r) by row-oriented
// forward substitution with all r right-hand sides in parallel (O(r)
// barriers).  Entry (l, c) receives its subtractions in the order q = 0, 1, ...
// (the q < c ones are exact zeros), so Linv is bit-identical to the
// column-by-column formula.
__device__ void block_tri_inverse(int r, const double *L, double *Linv) {
  for (int i = threadIdx.x; i < r * r; i += blockDim.x) Linv[i] = (i / r == i % r) ? 1.0 : 0.0;
  __syncthreads();
  for (int i = 0; i < r; ++i) {
    for (int c = threadIdx.x; c <= i; c += blockDim.x) Linv[i * r + c] = Linv[i * r + c] / L[i * r + i];
    __syncthreads();
    const int t = r - i - 1;
    for (int idx = threadIdx.x; idx < t * (i + 1); idx += blockDim.x) {
      const int l = i + 1 + idx / (i + 1), c = idx % (i + 1);
      Linv[l * r + c] -= L[l * r + i] * Linv[i * r + c];
    }
    __syncthreads();
  }
}

// Block Cholesky + lower-triangular inverse for r <= 32 with kPrepThreads =
// 256 threads as 32 columns x 8 row groups (thread (c, g) owns column c of
// rows g, g+8, g+16, g+24): no index division, every thread takes the pivot's
// square root itself (no serial section), each step's loads are issued before
// its stores, two barriers per step.  The same operations in the same order
// as block_cholesky + block_tri_inverse (entry (i,l) receives L(i,j) L(l,j)
// for j = 0, 1, ...; Linv(l,c) its subtractions q = 0, 1, ...), so the
// results are bit-identical.  G: r x r (row stride r); L, Linv: shared.
// Returns 1 on success; 0 when a pivot fails kCholSafe (eigen path).
__device__ int block_chol_inv32(int r, const double *G, double *L, double *Linv) {
  const int c = threadIdx.x & 31, g = threadIdx.x >> 5;
  double maxd = 0.0;
  for (int j = 0; j < r; ++j) maxd = fmax(maxd, G[j * r + j]);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int i = g + 8 * k;
    if (i < r && c < r) {
      L[i * r + c] = c <= i ? G[i * r + c] : 0.0;
      Linv[i * r + c] = i == c ? 1.0 : 0.0;
    }
  }
  __syncthreads();
  if (!(maxd > 0.0)) return 0;
  for (int j = 0; j < r; ++j) {
    __syncthreads();   // the previous step's trailing update is visible
    const double dj = L[j * r + j];
    if (!(dj > kCholSafe * maxd)) return 0;   // block-uniform
    const double ljj = sqrt(dj);
    if (g == 0 && c > j && c < r) L[c * r + j] = L[c * r + j] / ljj;
    __syncthreads();
    if (g == 0 && c == j) L[j * r + j] = ljj;   // nobody reads L(j,j) in this phase
    if (c > j && c < r) {   // column c of the trailing rows i >= c
      const double lcj = L[c * r + j];
      double lij[4], cur[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int i = g + 8 * k;
        const bool on = i >= c && i < r;
        lij[k] = on ? L[i * r + j] : 0.0;
        cur[k] = on ? L[i * r + c] : 0.0;
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int i = g + 8 * k;
        if (i >= c && i < r) L[i * r + c] = cur[k] - lij[k] * lcj;
      }
    }
  }
  __syncthreads();
  // L^{-1} by rows: row i divided by L(i,i), then subtracted from the rows below
  for (int i = 0; i < r; ++i) {
    const double lii = L[i * r + i];
    if (g == 0 && c <= i) Linv[i * r + c] = Linv[i * r + c] / lii;
    __syncthreads();
    if (c <= i) {
      const double xic = Linv[i * r + c];
      double lli[4], cur[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int l = g + 8 * k;
        const bool on = l > i && l < r;
        lli[k] = on ? L[l * r + i] : 0.0;
        cur[k] = on ? Linv[l * r + c] : 0.0;
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int l = g + 8 * k;
        if (l > i && l < r) Linv[l * r + c] = cur[k] - lli[k] * xic;
      }
    }
    __syncthreads();
  }
  return 1;
}

// Cholesky + inverse of the factor, whole block: Li = L^{-1} (row stride r)
// in shared memory; the warp version for r <= 32.  Returns 1 on success.
__device__ int block_chol_inv(int r, const double *G, double *L, double *Li, int *ok_flag) {
  if (r <= 32 && blockDim.x == kPrepThreads) return block_chol_inv32(r, G, L, Li);
  if (!block_cholesky(r, G, L, ok_flag)) return 0;
  block_tri_inverse(r, L, Li);
  return 1;
}

// Leverage preparation from Gram G (r x r, global): W with l_i = ||a_i W||^2.
// Cholesky: W = L^{-T} (upper triangular).  Fallback: W = V_kept diag(mu^{-1/2}).
// nk < r (fewer rows than columns, e.g. C2's 24-row mode at r = 25): when the
// rows a_i = A(i,:) / lam (lam null: 1) are linearly independent -- the nk x nk
// Gram A A^T passes the Cholesky test -- the hat matrix A (A^T A)^+ A^T is the
// identity, so l_i = 1 and rank = nk exactly (AMB-11, the eigen cutoff keeps the
// nk nonzero eigenvalues A^T A shares with A A^T); tri = 2 tells the leverage
// pass.  Saves the r x r Jacobi of the rank-deficient Gram.
__device__ bool short_full_row_rank(int r, const double *A, const double *lam, int64_t nk, int ld, double *H,
                                    double *scratch, int *ok) {
  if (!A || nk <= 0 || nk >= r || nk > 32) return false;
  const int n = (int)nk;
  for (int i = threadIdx.x; i < n * n; i += blockDim.x) {
    const int p = i / n, q = i % n;
    double h = 0.0;
    for (int c = 0; c < r; ++c) {
      const double ap = lam ? A[p * (int64_t)ld + c] / lam[c] : A[p * (int64_t)ld + c];
      const double aq = lam ? A[q * (int64_t)ld + c] / lam[c] : A[q * (int64_t)ld + c];
      h += ap * aq;
    }
    H[i] = h;
  }
  __syncthreads();
  return block_cholesky(n, H, scratch, ok) != 0;
}

__device__ void lev_prep_body(int r, const double *Gg, ModeDev *md, const double *A = nullptr,
                              const double *lam = nullptr, int64_t nk = 0, int ld = 0) {
  extern __shared__ double sm[];
  double *G = sm, *L = sm + r * r, *Li = sm + 2 * r * r;
  __shared__ int ok;
  for (int i = threadIdx.x; i < r * r; i += blockDim.x) { G[i] = Gg[i]; md->GA[i] = Gg[i]; }
  __syncthreads();
  int good = block_chol_inv(r, G, L, Li, &ok);
  if (good) {
    // W = Li^T : W[p][c] = Li[c][p]
    for (int i = threadIdx.x; i < r * r; i += blockDim.x) {
      int p = i / r, c = i % r;
      md->W[p * r + c] = Li[c * r + p];
    }
    if (threadIdx.x == 0) { md->tri = 1; md->rank = r; }
    return;
  }
  if (short_full_row_rank(r, A, lam, nk, ld, L, Li, &ok)) {
    if (threadIdx.x == 0) { md->tri = 2; md->rank = (int)nk; }
    return;
  }
  // eigen fallback (AMB-11): W = V_kept diag(mu^{-1/2})
  double *a = L, *V = Li;
  __syncthreads();
  for (int i = threadIdx.x; i < r * r; i += blockDim.x) a[i] = G[i];
  __syncthreads();
  block_jacobi(r, a, V);
  __shared__ double mumax;
  __shared__ int rank_s;
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int j = 0; j < r; ++j) m = fmax(m, a[j * r + j]);
    mumax = m;
    int rk = 0;
    for (int j = 0; j < r; ++j) rk += (m > 0.0 && a[j * r + j] > (double)r * 2.220446049250313e-16 * m);
    rank_s = rk;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < r * r; i += blockDim.x) {
    int p = i / r, j = i % r;
    double mu = a[j * r + j];
    bool keep = mumax > 0.0 && mu > (double)r * 2.220446049250313e-16 * mumax;
    md->W[p * r + j] = keep ? V[p * r + j] / sqrt(mu) : 0.0;
  }
  if (threadIdx.x == 0) { md->tri = 0; md->rank = rank_s; }
}

__global__ void k_lev_prep(int r, const double *G, ModeDev *md, const double *A = nullptr, int64_t nk = 0,
                           int ld = 0) {
  lev_prep_body(r, G, md, A, nullptr, nk, ld);
}

// ======================================================================
// K1/K2: leverage rows -> p~ -> integer weights q (CDF pass 1)
// ======================================================================
constexpr int kLevThreads = 256;

// CDF pass 3: C[i] = offset(tile) + inclusive scan of q within tile.
__global__ void __launch_bounds__(kLevThreads) k_cdf_final(uint64_t *__restrict__ C, int64_t n,
                                                           const uint64_t *__restrict__ tile_off,
                                                           const StepCtl *ctl = nullptr) {
  CPARLS_GUARD(ctl);
  int64_t i = (int64_t)blockIdx.x * kLevThreads + threadIdx.x;
  uint64_t q = i < n ? C[i] : 0ull;
  uint64_t tot;
  uint64_t ex = block_excl_scan<unsigned long long>(q, (unsigned long long *)&tot);
  if (i < n) C[i] = tile_off[blockIdx.x] + ex + q;
}

// exclusive scan of u64 tile sums (single block): each thread scans
// kScanItems consecutive entries serially, one block scan per 2048 (integer
// adds: the result does not depend on the grouping)
__global__ void k_scan_u64_single(uint64_t *part, int64_t nb, const StepCtl *ctl = nullptr) {
  CPARLS_GUARD(ctl);
  unsigned long long carry = 0;
  for (int64_t base = 0; base < nb; base += kScanTile) {
    const int64_t b0 = base + (int64_t)threadIdx.x * kScanItems;
    unsigned long long v[kScanItems];
    unsigned long long sum = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
      v[i] = b0 + i < nb ? part[b0 + i] : 0ull;
      sum += v[i];
    }
    unsigned long long tot;
    unsigned long long ex = carry + block_excl_scan<unsigned long long>(sum, &tot);
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
      if (b0 + i < nb) part[b0 + i] = ex;
      ex += v[i];
    }
    carry += tot;
    __syncthreads();
  }
}

// Recompute q from given p~ (set_ptilde path), same rounding as k_lev_rows.
__global__ void k_q_from_pt(const double *__restrict__ pt, int64_t n, uint64_t *__restrict__ C,
                            uint64_t *__restrict__ tile_sum, double *alpha_out, unsigned long long *drawable_out,
                            const StepCtl *ctl = nullptr) {
  CPARLS_GUARD(ctl);
  int64_t i = (int64_t)blockIdx.x * kLevThreads + threadIdx.x;
  double p = i < n ? pt[i] : 0.0;
  uint64_t q = __double2ull_rn(p * kTwo62);
  if (i < n) C[i] = q;
  unsigned long long qs = warp_sum<unsigned long long>(q);
  double pm = p;
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) pm = fmax(pm, __shfl_xor_sync(0xffffffffu, pm, m));
  unsigned dr = __popc(__ballot_sync(0xffffffffu, i < n && p > 1.0842021724855044e-19));
  __shared__ unsigned long long wq[kLevThreads / 32];
  __shared__ double wp[kLevThreads / 32];
  __shared__ unsigned wd[kLevThreads / 32];
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) { wq[w] = qs; wp[w] = pm; wd[w] = dr; }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long s = 0; double m = 0.0; unsigned long long d = 0;
    for (int k = 0; k < kLevThreads / 32; ++k) { s += wq[k]; m = fmax(m, wp[k]); d += wd[k]; }
    tile_sum[blockIdx.x] = s;
    atomic_max_nonneg(alpha_out, m);
    atomicAdd(drawable_out, d);
  }
}

// U[0,1) factor init (AMB-21): entry (i,c) of mode m from Philox4x32-10 with
// counter (i, c, m, 0x1417), key (seed, 0x55AA); u = (x1<<21 | x0>>11) 2^-53.
__global__ void k_init_uniform(double *A, int64_t n, int r, int ld, int m, uint32_t seed) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * ld) return;
  int64_t i = t / ld;
  int c = (int)(t - i * ld);
  double v = 0.0;
  if (c < r) {
    u32x4 x = philox4x32_10({(uint32_t)i, (uint32_t)c, (uint32_t)m, 0x1417u}, seed, 0x55AAu);
    uint64_t w = ((uint64_t)x.y << 21) | (x.x >> 11);
    v = (double)w * 1.1102230246251565e-16;
  }
  A[t] = v;
}

// ======================================================================
// K3 DIDX
// ======================================================================
struct OtherModes {
  int d;
  int mode[kMaxModes];
  int64_t n[kMaxModes];
  const double *pt[kMaxModes];
  const uint64_t *C[kMaxModes];
  const double *A[kMaxModes];
  uint64_t mult[kMaxModes];   // prod_{l<j} n_l
  const ModeDev *md[kMaxModes];   // alpha and drawable counts of the other modes (device)
  FastDiv div[kMaxModes];     // division by n[j] (key decoding)
};

// max p~ of other mode l, read on the device
__device__ __forceinline__ double om_alpha(const OtherModes &om, int l) { return om.md[l]->alpha; }

// Canonical product with position j = x, every other position at alpha (the
// largest p any index with i_j fixed can reach; fp multiply is monotone).
__device__ __forceinline__ double prod_with(const OtherModes &om, const double *al, int j, double x) {
  double p = (j == 0) ? x : al[0];
  for (int l = 1; l < om.d; ++l) p = p * ((l == j) ? x : al[l]);
  return p;
}
__device__ __forceinline__ void load_alphas(const OtherModes &om, double *al) {
  for (int l = 0; l < om.d; ++l) al[l] = om_alpha(om, l);
}

// pass 1: per-tile counts of candidates of mode j
__global__ void k_cand_count(OtherModes om, int j, double tau, int64_t *__restrict__ part,
                             const StepCtl *ctl = nullptr) {
  CPARLS_GUARD(ctl);
  double al[kMaxModes];
  load_alphas(om, al);
  int64_t base = (int64_t)blockIdx.x * kScanTile;
  int64_t s = 0;
  const double *pt = om.pt[j];
  for (int i = 0; i < kScanItems; ++i) {
    int64_t idx = base + (int64_t)i * kScanThreads + threadIdx.x;
    if (idx < om.n[j] && prod_with(om, al, j, pt[idx]) > tau) ++s;
  }
  int64_t tot;
  block_excl_scan<int64_t>(s, &tot);
  if (threadIdx.x == 0) part[blockIdx.x] = tot;
}

// pass 3: ordered scatter of candidates: key = ~bits(p~) (descending order
// after an ascending stable sort), value = row index.
__global__ void k_cand_scatter(OtherModes om, int j, double tau, const int64_t *__restrict__ part,
                               uint64_t *__restrict__ ckey, uint32_t *__restrict__ cidx,
                               const StepCtl *ctl = nullptr) {
  CPARLS_GUARD(ctl);
  double al[kMaxModes];
  load_alphas(om, al);
  int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  const double *pt = om.pt[j];
  bool f[kScanItems];
  int64_t s = 0;
  for (int i = 0; i < kScanItems; ++i) {
    int64_t idx = base + i;
    f[i] = idx < om.n[j] && prod_with(om, al, j, pt[idx]) > tau;
    s += f[i];
  }
  int64_t tot;
  int64_t pos = block_excl_scan<int64_t>(s, &tot) + part[blockIdx.x];
  for (int i = 0; i < kScanItems; ++i) {
    if (f[i]) {
      int64_t idx = base + i;
      ckey[pos] = ~(uint64_t)__double_as_longlong(pt[idx]);
      cidx[pos] = (uint32_t)idx;
      ++pos;
    }
  }
}

__device__ __forceinline__ double cand_val(uint64_t k) { return __longlong_as_double((long long)~k); }

// Level expansion count: entry e (partial product pp_e) x sorted candidates of
// level l: count of the prefix with fl(pp*v)*alpha_{l+1}*... > tau.
// Counts live on the device when nlist_dev / ncand_dev are given (asynchronous
// step: grid-stride over an upper-bound grid).
__global__ void k_didx_count(const double *__restrict__ pp, int64_t nlist, const uint64_t *__restrict__ ckey,
                             int64_t ncand, OtherModes om, int l, double tau, int64_t *__restrict__ cnt,
                             const int64_t *nlist_dev = nullptr, const int64_t *ncand_dev = nullptr,
                             const StepCtl *ctl = nullptr) {
  CPARLS_GUARD(ctl);
  nlist = dcount(nlist, nlist_dev);
  ncand = dcount(ncand, ncand_dev);
  double al[kMaxModes];
  load_alphas(om, al);
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nlist; e += (int64_t)gridDim.x * blockDim.x) {
    double base = pp[e];
    int64_t lo = 0, len = ncand;  // first t where predicate fails
    while (len > 0) {
      int64_t half = len >> 1;
      double b = base * cand_val(ckey[lo + half]);
      for (int k = l + 1; k < om.d; ++k) b = b * al[k];
      if (b > tau) { lo += half + 1; len -= half + 1; }
      else len = half;
    }
    cnt[e] = lo;
  }
}

// Level expansion emit: one warp per entry, lanes over its candidate prefix.
__global__ void k_didx_emit(const uint64_t *__restrict__ pkey, const double *__restrict__ pp, int64_t nlist,
                            const int64_t *__restrict__ cnt, const int64_t *__restrict__ off,
                            const uint64_t *__restrict__ ckey, const uint32_t *__restrict__ cidx, uint64_t mult,
                            uint64_t *__restrict__ nkey, double *__restrict__ npp, const int64_t *nlist_dev = nullptr,
                            const StepCtl *ctl = nullptr) {
  CPARLS_GUARD(ctl);
  nlist = dcount(nlist, nlist_dev);
  const int lane = threadIdx.x & 31;
  for (int64_t e = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; e < nlist;
       e += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    int64_t c = cnt[e], o = off[e];
    uint64_t k0 = pkey[e];
    double p0 = pp[e];
    for (int64_t t = lane; t < c; t += 32) {
      nkey[o + t] = k0 + (uint64_t)cidx[t] * mult;
      npp[o + t] = p0 * cand_val(ckey[t]);
    }
  }
}

// Level-0 list from the sorted candidates of mode m_1.
__global__ void k_didx_level0(const uint64_t *__restrict__ ckey, const uint32_t *__restrict__ cidx, int64_t n,
                              uint64_t *__restrict__ key, double *__restrict__ pp, const int64_t *n_dev = nullptr,
                              const StepCtl *ctl = nullptr) {
  CPARLS_GUARD(ctl);
  n = dcount(n, n_dev);
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    key[t] = cidx[t];
    pp[t] = cand_val(ckey[t]);
  }
}

// compensated sum of n doubles -> block partial dd
__global__ void k_sum_dd(const double *__restrict__ x, int64_t n, dd *__restrict__ part,
                         const int64_t *n_dev = nullptr, const StepCtl *ctl = nullptr) {
  CPARLS_GUARD(ctl);
  n = dcount(n, n_dev);
  dd s = {0.0, 0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    s = dd_add_d(s, x[i]);
  s = warp_sum_dd(s);
  __shared__ dd ws[32];
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) ws[w] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    dd t = {0.0, 0.0};
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t = dd_add(t, ws[i]);
    part[blockIdx.x] = t;
  }
}
__global__ void k_sum_dd_final(const dd *__restrict__ part, int nb, double *out, const StepCtl *ctl = nullptr) {
  CPARLS_GUARD(ctl);
  if (threadIdx.x == 0) {
    dd t = {0.0, 0.0};
    for (int i = 0; i < nb; ++i) t = dd_add(t, part[i]);
    *out = t.hi + t.lo;
  }
}

// Deterministic block of the sample set: w^2 = 1.
__global__ void k_det_emit(const uint64_t *__restrict__ key, const double *__restrict__ p, int64_t n,
                           uint64_t *__restrict__ skey, double *__restrict__ sw2, double *__restrict__ sp,
                           int32_t *__restrict__ scnt, uint8_t *__restrict__ sdet, const int64_t *n_dev = nullptr,
                           const StepCtl *ctl = nullptr) {
  CPARLS_GUARD(ctl);
  n = dcount(n, n_dev);
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  skey[t] = key[t]; sw2[t] = 1.0; sp[t] = p[t]; scnt[t] = 1; sdet[t] = 1;
}

// gather by index (u32) for the truncation path
__global__ void k_gather_kp(const uint64_t *__restrict__ key, const double *__restrict__ p,
                            const uint32_t *__restrict__ idx, int64_t n, uint64_t *__restrict__ okey,
                            double *__restrict__ op) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  okey[t] = key[idx[t]];
  op[t] = p[idx[t]];
}
__global__ void k_iota_u32(uint32_t *v, int64_t n) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) v[t] = (uint32_t)t;
}
__global__ void k_pbits_desc(const double *__restrict__ p, int64_t n, uint64_t *__restrict__ k) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) k[t] = ~(uint64_t)__double_as_longlong(p[t]);
}

// ======================================================================
// K4 SIDX (Alg. 2): attempts [a0, a0+cnt)
// ======================================================================
constexpr int kSidxThreads = 256;

__global__ void __launch_bounds__(kSidxThreads) k_sidx_gen(OtherModes om, uint64_t a0, int64_t cnt, double tau,
                                                           uint32_t seed_lo, uint32_t seed_hi, uint32_t step,
                                                           uint64_t *__restrict__ akey, double *__restrict__ ap,
                                                           int64_t *__restrict__ part) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int acc = 0;
  if (t < cnt) {
    uint64_t a = a0 + (uint64_t)t;
    uint32_t words[2 * kMaxModes];
    for (int lane = 0; lane < (om.d + 1) / 2; ++lane) {
      u32x4 x = philox4x32_10({(uint32_t)a, (uint32_t)(a >> 32), step, (uint32_t)lane}, seed_lo, seed_hi);
      words[4 * lane + 0] = x.x; words[4 * lane + 1] = x.y;
      words[4 * lane + 2] = x.z; words[4 * lane + 3] = x.w;
    }
    uint64_t key = 0;
    double p = 1.0;
    for (int j = 0; j < om.d; ++j) {
      uint32_t lo = words[4 * (j / 2) + 2 * (j % 2)], hi = words[4 * (j / 2) + 2 * (j % 2) + 1];
      uint64_t R = ((uint64_t)hi << 32) | lo;
      const uint64_t *C = om.C[j];
      uint64_t W = __ldg(C + om.n[j] - 1);
      uint64_t tt = __umul64hi(R, W);                       // AMB-9
      int64_t i = upper_bound_u64(C, om.n[j], tt);          // i_k ~ Multi(p~_k)
      double v = __ldg(om.pt[j] + i);
      p = (j == 0) ? v : p * v;                              // canonical product (AMB-5)
      key += (uint64_t)i * om.mult[j];
    }
    acc = (p <= tau);
    akey[t] = acc ? key : kEmptyKey;
    ap[t] = p;
  }
  int64_t tot;
  block_excl_scan<int64_t>((int64_t)acc, &tot);
  if (threadIdx.x == 0) part[blockIdx.x] = tot;
}

// Ordered compaction of accepted attempts; keeps positions < need (AMB-8).
__global__ void __launch_bounds__(kSidxThreads) k_sidx_scatter(const uint64_t *__restrict__ akey,
                                                               const double *__restrict__ ap, int64_t cnt,
                                                               const int64_t *__restrict__ part, int64_t have,
                                                               int64_t need, uint64_t a0, uint64_t *__restrict__ rkey,
                                                               double *__restrict__ rp,
                                                               unsigned long long *__restrict__ last_attempt) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int acc = (t < cnt) && akey[t] != kEmptyKey;
  int64_t tot;
  int64_t pos = have + part[blockIdx.x] + block_excl_scan<int64_t>((int64_t)acc, &tot);
  if (acc && pos < need) {
    rkey[pos] = akey[t];
    rp[pos] = ap[t];
    if (pos == need - 1) *last_attempt = a0 + (uint64_t)t;
  }
}

// ======================================================================
// K5 CIDX: combine repeats with a hash table
// ======================================================================
__device__ __forceinline__ uint64_t mix64(uint64_t k) {
  k ^= k >> 33; k *= 0xff51afd7ed558ccdull; k ^= k >> 33; k *= 0xc4ceb9fe1a85ec53ull; k ^= k >> 33;
  return k;
}

// Deterministic combine (AMB-35): the unique random rows are emitted in the
// order of their first draw (attempt order, itself deterministic) instead of
// hash-slot order via an atomic counter.  insert also keeps the first draw
// index per slot; flags marks each key's first draw (and its slot); an
// exclusive scan of the flags gives the output positions.
__global__ void k_cidx_insert_first(const uint64_t *__restrict__ rkey, const double *__restrict__ rp, int64_t n,
                                    unsigned long long *__restrict__ hkey, uint32_t *__restrict__ hcnt,
                                    double *__restrict__ hp, uint32_t *__restrict__ hfirst, uint64_t hmask,
                                    const int64_t *n_dev = nullptr, const StepCtl *ctl = nullptr) {
  CPARLS_GUARD(ctl);
  n = dcount(n, n_dev);
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  uint64_t k = rkey[t];
  uint64_t h = mix64(k) & hmask;
  while (true) {
    unsigned long long prev = atomicCAS(&hkey[h], kEmptyKey, (unsigned long long)k);
    if (prev == kEmptyKey || prev == k) {
      atomicAdd(&hcnt[h], 1u);
      atomicMin(&hfirst[h], (uint32_t)t);
      if (prev == kEmptyKey) hp[h] = rp[t];   // p depends only on the key
      return;
    }
    h = (h + 1) & hmask;
  }
}

__global__ void k_cidx_first_flags(const uint64_t *__restrict__ rkey, int64_t n,
                                   const unsigned long long *__restrict__ hkey,
                                   const uint32_t *__restrict__ hfirst, uint64_t hmask,
                                   int64_t *__restrict__ flag, uint32_t *__restrict__ slot,
                                   const int64_t *n_dev = nullptr, const StepCtl *ctl = nullptr) {
  CPARLS_GUARD(ctl);
  n = dcount(n, n_dev);
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const uint64_t k = rkey[t];
  uint64_t h = mix64(k) & hmask;
  while (hkey[h] != k) h = (h + 1) & hmask;
  slot[t] = (uint32_t)h;
  flag[t] = hfirst[h] == (uint32_t)t ? 1 : 0;
}

// w^2 = c (1 - p_det) / (s_rnd p)  (P:537 with s -> s_rnd, AMB-3); resets the slot
__global__ void k_cidx_emit_first(const int64_t *__restrict__ flag, const int64_t *__restrict__ pos,
                                  const uint32_t *__restrict__ slot, int64_t n,
                                  unsigned long long *__restrict__ hkey, uint32_t *__restrict__ hcnt,
                                  const double *__restrict__ hp, uint32_t *__restrict__ hfirst,
                                  const double *__restrict__ pdet_ptr, int64_t s_rnd, int64_t base,
                                  uint64_t *__restrict__ skey, double *__restrict__ sw2, double *__restrict__ sp,
                                  int32_t *__restrict__ scnt, uint8_t *__restrict__ sdet,
                                  const StepCtl *ctl = nullptr) {
  CPARLS_GUARD(ctl);
  if (ctl) { n = ctl->have; s_rnd = ctl->s_rnd; base = ctl->sdet; }   // asynchronous step: device sizes
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n || !flag[t]) return;
  const uint32_t h = slot[t];
  const uint32_t c = hcnt[h];
  const double p = hp[h];
  const int64_t o = base + pos[t];
  skey[o] = hkey[h];
  scnt[o] = (int32_t)c;
  sp[o] = p;
  sw2[o] = ((double)c * (1.0 - *pdet_ptr)) / ((double)s_rnd * p);
  sdet[o] = 0;
  hkey[h] = kEmptyKey;   // reset for the next sample
  hcnt[h] = 0;
  hfirst[h] = 0xFFFFFFFFu;
}

// ======================================================================
// K7 TnsrSamp lookup: equal_range of each sampled key in the
// mode-k sorted keys, narrowed by the top-level directory.
// ======================================================================
// Sample keys are canonical (eq:bijection, AMB-1: other modes ascending, first
// fastest); a mode copy may store its keys with another order of the other
// modes (ModeIndex::order), so the key is re-encoded before the search.
struct KeyRemap {
  int d;
  int identity;
  int64_t n[kMaxModes];       // canonical order dims
  uint64_t cmult[kMaxModes];  // multiplier of canonical digit j in the copy's key
  FastDiv div[kMaxModes];     // division by n[j]
};

__global__ void k_lookup(const uint64_t *__restrict__ skey, int64_t sbar, const uint64_t *__restrict__ keys,
                         const int64_t *__restrict__ dir, int shift, int64_t nbkt, KeyRemap rm,
                         int64_t *__restrict__ lo_out, int64_t *__restrict__ len_out,
                         const int64_t *sbar_dev = nullptr, const StepCtl *ctl = nullptr) {
  CPARLS_GUARD(ctl);
  sbar = dcount(sbar, sbar_dev);
  int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= sbar) return;
  uint64_t k = skey[j];
  if (!rm.identity) {
    uint64_t t = k, kk = 0;
    for (int m = 0; m < rm.d; ++m) {
      uint64_t rem;
      const uint64_t q = fastdivmod(t, rm.div[m], rem);
      kk += rem * rm.cmult[m];
      t = q;
    }
    k = kk;
  }
  uint64_t b = k >> shift;
  int64_t lo = 0, hi = 0;
  if ((int64_t)b < nbkt) {
    lo = __ldg(dir + b);
    hi = __ldg(dir + b + 1);
  }
  // lower_bound
  int64_t L = lo, len = hi - lo;
  while (len > 0) {
    int64_t half = len >> 1;
    if (__ldg(keys + L + half) < k) { L += half + 1; len -= half + 1; }
    else len = half;
  }
  int64_t U = L;
  len = hi - L;
  while (len > 0) {
    int64_t half = len >> 1;
    if (__ldg(keys + U + half) <= k) { U += half + 1; len -= half + 1; }
    else len = half;
  }
  lo_out[j] = L;
  len_out[j] = U - L;
}

// ======================================================================
// K9 solve + normalize
// ======================================================================
// Single block: Cholesky of the sampled Gram with pivot test; fallback to the
// eigen pseudo-inverse (AMB-12).  Ginv = G^{-1} (or G^+).
__global__ void k_solve_prep(int r, SolveDev *sd, const StepCtl *ctl = nullptr) {
  CPARLS_GUARD(ctl);
  extern __shared__ double sm[];
  double *G = sm, *L = sm + r * r, *Li = sm + 2 * r * r;
  __shared__ int ok;
  for (int i = threadIdx.x; i < r * r; i += blockDim.x) G[i] = sd->G[i];
  __syncthreads();
  int good = block_chol_inv(r, G, L, Li, &ok);
  if (good) {
    __syncthreads();
    // Ginv = Li^T Li
    for (int i = threadIdx.x; i < r * r; i += blockDim.x) {
      int p = i / r, q = i % r;
      double s = 0.0;
      for (int k = max(p, q); k < r; ++k) s += Li[k * r + p] * Li[k * r + q];
      sd->Ginv[i] = s;
    }
    if (threadIdx.x == 0) { sd->rank_used = r; sd->chol_fallback = 0; }
    return;
  }
  double *a = L, *V = Li;
  for (int i = threadIdx.x; i < r * r; i += blockDim.x) a[i] = G[i];
  __syncthreads();
  block_jacobi(r, a, V);
  __shared__ double inv[kMaxRank];
  __shared__ double mumax;
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int j = 0; j < r; ++j) m = fmax(m, a[j * r + j]);
    mumax = m;
    int rk = 0;
    for (int j = 0; j < r; ++j) {
      double mu = a[j * r + j];
      bool keep = m > 0.0 && mu > (double)r * 2.220446049250313e-16 * m;
      rk += keep;
      inv[j] = keep ? 1.0 / mu : 0.0;
    }
    sd->rank_used = rk;
    sd->chol_fallback = 1;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < r * r; i += blockDim.x) {
    int p = i / r, q = i % r;
    double sum = 0.0;
    for (int j = 0; j < r; ++j) sum += V[p * r + j] * inv[j] * V[q * r + j];
    sd->Ginv[i] = sum;
  }
}

// lambda_c = ||B(:,c)||, G_A = B^T B / (lambda lambda^T), then the
// leverage preparation of the normalized factor.
__global__ void k_norm_prep(int r, SolveDev *sd, ModeDev *md, const StepCtl *ctl = nullptr,
                            const double *B = nullptr, int64_t nk = 0, int ld = 0) {
  CPARLS_GUARD(ctl);
  extern __shared__ double sm[];
  double *GA = sm + 3 * r * r;   // beyond lev_prep's scratch
  for (int c = threadIdx.x; c < r; c += blockDim.x) sd->lambda[c] = sqrt(fmax(sd->BtB[c * r + c], 0.0));
  __syncthreads();
  for (int i = threadIdx.x; i < r * r; i += blockDim.x) {
    int p = i / r, q = i % r;
    double lp = sd->lambda[p], lq = sd->lambda[q];
    GA[i] = (lp > 0.0 && lq > 0.0) ? (sd->BtB[i] / lp) / lq : 0.0;
  }
  __syncthreads();
  lev_prep_body(r, GA, md, B, sd->lambda, nk, ld);
}

// ======================================================================
// K0 index build helpers (one-time, in cparls_create)
// ======================================================================
template <typename IT>
__global__ void k_make_outkey(const IT *__restrict__ coords, int64_t nnz, int D, int k, uint32_t *__restrict__ okey,
                              uint32_t *__restrict__ ids) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nnz) return;
  okey[e] = (uint32_t)coords[e * D + k];
  ids[e] = (uint32_t)e;
}

struct KeySpec {
  int D, k;
  int64_t dims[kMaxModes];
  int order[kMaxModes];   // the copy's other modes, fastest-varying first
};

template <typename IT>
__global__ void k_make_keys(const IT *__restrict__ coords, int64_t nnz, KeySpec ks, const uint32_t *__restrict__ ids,
                            uint64_t *__restrict__ keys) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nnz) return;
  int64_t e = ids[t];
  uint64_t key = 0, mult = 1;
  for (int j = 0; j < ks.D - 1; ++j) {
    const int m = ks.order[j];
    key += (uint64_t)coords[e * ks.D + m] * mult;
    mult *= (uint64_t)ks.dims[m];
  }
  keys[t] = key;
}

// rows x r block of a row-major (pitch ld) matrix into a dense rows x r buffer
__global__ void k_pack_rows(const double *__restrict__ src, int ld, int r, int64_t rows, double *__restrict__ dst) {
  const int64_t n = rows * r;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / r;
    dst[i] = src[row * ld + (i - row * r)];
  }
}

// Single-sort build (round 2): one composite key per nonzero, the copy's key
// times n_k plus the mode-k coordinate, so one stable radix sort by it yields
// (key, then out, then input order) -- the order of the two stable sorts (by
// out, then by key) -- with the value as the sort's payload (no id gathers).
template <typename IT, typename VT>
__global__ void k_make_comp(const IT *__restrict__ coords, const VT *__restrict__ vals, int64_t nnz, KeySpec ks,
                            uint64_t *__restrict__ comp, VT *__restrict__ v) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
    uint64_t key = 0, mult = 1;
    for (int j = 0; j < ks.D - 1; ++j) {
      const int m = ks.order[j];
      key += (uint64_t)coords[e * ks.D + m] * mult;
      mult *= (uint64_t)ks.dims[m];
    }
    comp[e] = key * (uint64_t)ks.dims[ks.k] + (uint64_t)coords[e * ks.D + ks.k];
    v[e] = vals[e];
  }
}

// composite -> (key in place, out)
__global__ void k_split_comp(uint64_t *__restrict__ comp, int64_t nnz, FastDiv nk, int32_t *__restrict__ out) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
    uint64_t rem;
    const uint64_t q = fastdivmod(comp[e], nk, rem);
    comp[e] = q;
    out[e] = (int32_t)rem;
  }
}

// Row degrees of the slowest key mode of a sorted copy from its run
// boundaries (no atomics: a Zipf head row would serialize them): beg[d] /
// end[d] = first / one-past-last position whose key has slowest digit d.
__global__ void k_slow_bounds(const uint64_t *__restrict__ keys, int64_t nnz, FastDiv stride, int64_t *__restrict__ beg,
                              int64_t *__restrict__ end) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t d = fastdiv(keys[e], stride);
    if (e == 0 || fastdiv(keys[e - 1], stride) != d) beg[d] = e;
    if (e == nnz - 1 || fastdiv(keys[e + 1], stride) != d) end[d] = e + 1;
  }
}

__global__ void k_bounds_deg(const int64_t *__restrict__ beg, const int64_t *__restrict__ end, int64_t n,
                             uint32_t *__restrict__ deg) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    deg[i] = (uint32_t)(end[i] - beg[i]);
}

template <typename IT, typename VT>
__global__ void k_gather_nz(const IT *__restrict__ coords, const VT *__restrict__ vals, int64_t nnz, int D, int k,
                            const uint32_t *__restrict__ ids, int32_t *__restrict__ out, VT *__restrict__ v) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nnz) return;
  int64_t e = ids[t];
  out[t] = (int32_t)coords[e * D + k];
  v[t] = vals[e];
}

template <typename IT>
__global__ void k_check_coords(const IT *__restrict__ coords, int64_t nnz, KeySpec ks, unsigned long long *bad) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nnz) return;
  for (int m = 0; m < ks.D; ++m) {
    long long c = (long long)coords[e * ks.D + m];
    if (c < 0 || c >= ks.dims[m]) { atomicAdd(bad, 1ull); return; }
  }
}

__global__ void k_dir_fill(const uint64_t *__restrict__ keys, int64_t nnz, int shift, int64_t *__restrict__ dir,
                           int64_t nbkt) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nnz) return;
  int64_t b = (int64_t)(keys[i] >> shift);
  int64_t bp = (i == 0) ? -1 : (int64_t)(keys[i - 1] >> shift);
  for (int64_t bb = bp + 1; bb <= b && bb < nbkt; ++bb) dir[bb] = i;
  if (i == nnz - 1)
    for (int64_t bb = b + 1; bb <= nbkt; ++bb) dir[bb] = nnz;
}

template <typename VT>
__global__ void k_sumsq(const VT *__restrict__ v, int64_t n, dd *__restrict__ part, double *maxabs) {
  dd s = {0.0, 0.0};
  double mx = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double x = (double)v[i];
    s = dd_add_d(s, x * x);
    mx = fmax(mx, fabs(x));
  }
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, m));
  if ((threadIdx.x & 31) == 0) atomic_max_nonneg(maxabs, mx);
  s = warp_sum_dd(s);
  __shared__ dd ws[32];
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) ws[w] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    dd t = {0.0, 0.0};
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t = dd_add(t, ws[i]);
    part[blockIdx.x] = t;
  }
}

// gather matched (out, val) of all samples in current sample order
template <typename VT>
__global__ void k_gather_fibers(const int64_t *__restrict__ off, const int64_t *__restrict__ lo,
                                const int64_t *__restrict__ len, int64_t sbar, const int32_t *__restrict__ outidx,
                                const VT *__restrict__ vals, int64_t *__restrict__ o, double *__restrict__ v) {
  int64_t j = blockIdx.x;
  if (j >= sbar) return;
  for (int64_t t = threadIdx.x; t < len[j]; t += blockDim.x) {
    o[off[j] + t] = outidx[lo[j] + t];
    v[off[j] + t] = (double)vals[lo[j] + t];
  }
}

// ---- sharded build: row degrees, destination ranks, packing ----
template <typename IT>
__global__ void k_coord_degree(const IT *__restrict__ coords, int64_t nnz, int D, int k,
                               unsigned long long *__restrict__ deg) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(deg + (int64_t)coords[e * D + k], 1ull);
}

// Destination rank of a nonzero in the sharded build of mode k:
// the owner of its mode-k row, or -- for a heavy row -- a rank chosen by a hash
// of its other coordinates (the row's nonzeros spread evenly over the ranks).
__host__ __device__ __forceinline__ uint64_t heavy_hash(uint64_t k) {
  k ^= k >> 33; k *= 0xff51afd7ed558ccdull; k ^= k >> 33; k *= 0xc4ceb9fe1a85ec53ull; k ^= k >> 33;
  return k;
}
// rank of one nonzero (its D coordinates c): the owner of row c[k] (last p
// with bound[p] <= c[k]), or for a heavy row the hash of its other coordinates
template <typename IT>
__host__ __device__ __forceinline__ int route_rank(const IT *c, int D, int k, const int64_t *bound, int P,
                                                   const uint8_t *heavy) {
  const int64_t row = (int64_t)c[k];
  if (heavy && heavy[row]) {
    uint64_t key = 0;
    for (int m = 0; m < D; ++m)
      if (m != k) key = key * 0x9E3779B97F4A7C15ull + (uint64_t)c[m];
    return (int)(((unsigned __int128)heavy_hash(key) * (unsigned)P) >> 64);
  }
  int lo = 0, len = P;
  while (len > 0) {
    const int half = len >> 1;
    if (bound[lo + half + 1] <= row) { lo += half + 1; len -= half + 1; }
    else len = half;
  }
  return lo;
}

template <typename IT>
__global__ void k_dest_rank(const IT *__restrict__ coords, int64_t nnz, int D, int k,
                            const int64_t *__restrict__ bound, int P, uint32_t *__restrict__ dest,
                            uint32_t *__restrict__ idx, unsigned long long *__restrict__ cnt,
                            const uint8_t *__restrict__ heavy) {
  __shared__ unsigned long long h[256];
  for (int i = threadIdx.x; i < P; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < nnz) {
    const int lo = route_rank<IT>(coords + e * D, D, k, bound, P, heavy);
    dest[e] = (uint32_t)lo;
    idx[e] = (uint32_t)e;
    atomicAdd(&h[lo], 1ull);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < P; i += blockDim.x)
    if (h[i]) atomicAdd(cnt + i, h[i]);
}

template <typename IT, typename VT>
__global__ void k_pack_nz(const IT *__restrict__ coords, const VT *__restrict__ vals, int64_t nnz, int D,
                          const uint32_t *__restrict__ perm, IT *__restrict__ sc, VT *__restrict__ sv) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nnz) return;
  const int64_t e = perm[t];
  for (int m = 0; m < D; ++m) sc[t * D + m] = coords[e * D + m];
  sv[t] = vals[e];
}



// canonical (ascending key) order of the combined sample: gather every sample
// array through the sort permutation (the keys arrive sorted)
__global__ void k_sample_permute(const uint32_t *__restrict__ perm, int64_t n, const double *__restrict__ w2,
                                 const double *__restrict__ p, const int32_t *__restrict__ cnt,
                                 const uint8_t *__restrict__ isdet, double *__restrict__ w2o, double *__restrict__ po,
                                 int32_t *__restrict__ cnto, uint8_t *__restrict__ isdeto) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int64_t j = perm[t];
  w2o[t] = w2[j];
  po[t] = p[j];
  cnto[t] = cnt[j];
  isdeto[t] = isdet[j];
}

// ---- fixed-point sampled RHS (rhs.cuh): per-column scales --------------------
// A matched entry e of fiber j adds w_j^2 x_e z_j to row out_e, and a fiber has
// one entry per row (x dupmax for duplicate coordinates), so
// |M_ic| <= max|x| dupmax sum_j w_j^2 |z_jc| =: U_c.  The RHS accumulates
// round(w_j^2 x_e z_jc 2^e_c) in int64 with 2^e_c = 2^(60 - ceil log2 U_c): exact
// integer sums (order-free, so the RHS is bit-reproducible) at a resolution of
// 2^-60 U_c, and 64-bit integer reductions run ~15% faster than fp64 ones
// (libcparls_peaks.so: 635 vs ~550 G lane-ops/s on this pattern).
// The column sums sum_j w_j^2 |z_jc| come per block from k_krp_rows (k_gram_scales).

// K6 epilogue, one launch: the sampled Gram from k_gram_rows_t's block
// partials (warp per upper entry, double-double, as k_pairs_reduce) and the
// per-column fixed-point scales from k_krp_rows' column-sum partials (warp per
// column; the last block to finish derives the scales from all columns).
// scale[c] = 2^e_c, scale[kMaxRank + c] = 2^-e_c (exact powers of two),
// scale[2 kMaxRank] = 1 for fixed point, 0 when this step falls back to fp64
// reductions (k_rhs and k_solve_rows_t read the flag).
__global__ void k_gram_scales(const double *__restrict__ part, const double *__restrict__ cpart, int64_t nb,
                              int64_t nbc, int r,
                              double *__restrict__ G, double *__restrict__ colsum, const double *maxabs,
                              double dupmax, double *__restrict__ scale, unsigned int *done_count,
                              const StepCtl *ctl = nullptr) {
  CPARLS_GUARD(ctl);
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t rr = (int64_t)r * r;
  if (w < rr) {
    const int p = (int)(w / r), q = (int)(w % r);
    if (p <= q) {
      dd sum = {0.0, 0.0};
      for (int64_t b = lane; b < nb; b += 32) sum = dd_add_d(sum, part[b * rr + w]);
      sum = warp_sum_dd(sum);
      if (lane == 0) {
        const double v = sum.hi + sum.lo;
        G[p * r + q] = v;
        G[q * r + p] = v;
      }
    }
  } else if (w < rr + r) {
    const int c = (int)(w - rr);
    double u = 0.0;
    for (int64_t b = lane; b < nbc; b += 32) u += cpart[b * r + c];
    u = warp_sum<double>(u);
    if (lane == 0) colsum[c] = u;
  }
  // last block: the scales from every column's sum
  __shared__ int last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(done_count, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  __shared__ int ok_all;
  if (threadIdx.x == 0) ok_all = 1;
  __syncthreads();
  const int c = threadIdx.x;
  int e = 0;
  if (c < r) {
    const double u = __ldcg(colsum + c) * *maxabs * dupmax;
    if (!(u < INFINITY)) atomicAnd(&ok_all, 0);   // inf / NaN bound
    else if (u > 0.0) {
      int ex;
      frexp(u, &ex);              // u < 2^ex
      e = 60 - ex;
      if (e < -960 || e > 960) atomicAnd(&ok_all, 0);   // 2^e_c or the terms' quanta out of range
    }
  }
  __syncthreads();
  const bool ok = ok_all != 0;
  if (c < r) {
    scale[c] = ok ? ldexp(1.0, e) : 1.0;
    scale[kMaxRank + c] = ok ? ldexp(1.0, -e) : 1.0;
  }
  if (c == 0) {
    scale[2 * kMaxRank] = ok ? 1.0 : 0.0;
    *done_count = 0u;   // ready for the next launch (stream-ordered)
  }
}

inline unsigned gram_scales_grid(int r) { return (unsigned)ceil_div(((int64_t)r * r + r) * 32, 256); }

// longest run of equal (key, out) in a sorted copy (duplicate coordinates)
__global__ void k_dup_runs(const uint64_t *__restrict__ key, const int32_t *__restrict__ out, int64_t nnz,
                           unsigned long long *maxrun) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
    if (e > 0 && key[e] == key[e - 1] && out[e] == out[e - 1]) continue;
    int64_t f = e + 1;
    while (f < nnz && key[f] == key[e] && out[f] == out[e]) ++f;
    if (f - e > 1) atomicMax(maxrun, (unsigned long long)(f - e));
  }
}

}  // namespace cparls

#include "rows.cuh"
#include "rhs.cuh"
#include "fit.cuh"
#include "fitest.cuh"
#include "als.cuh"
#include "rrf.cuh"
