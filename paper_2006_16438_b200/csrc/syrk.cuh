// syrk.cuh -- register-blocked Gram accumulation G += sum_rows w_row x_row x_row^T
// over row tiles staged in shared memory, used by the factor Gram (leverage),
// the sampled Gram Z~^T Z~ and B^T B (column norms).
//
// Mapping (256 threads): 8 row groups x 32 lanes.  The upper triangle of the
// r x r Gram is cut into 4x4 blocks (RB = ceil(r/4) per side, RB(RB+1)/2
// blocks); lane l owns blocks l, l+32, ...  Row group g walks rows g, g+8, ...
// of the tile.  Per row a lane issues 8 shared loads for 16 FMAs (vs 2 loads
// per FMA for one-pair-per-thread), so the pass stays off the smem roofline.
#pragma once
#include "common.cuh"

namespace cparls {

constexpr int kSyrkThreads = 256;

template <int RMAX>
struct Syrk {
  static constexpr int RB = (RMAX + 3) / 4;
  static constexpr int NBLK = RB * (RB + 1) / 2;
  static constexpr int PER = (NBLK + 31) / 32;
  double acc[PER][16];
  int bp[PER], bq[PER];

  __device__ __forceinline__ void init(int r) {
    const int lane = threadIdx.x & 31;
    const int rb = (r + 3) / 4;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      int b = lane + 32 * k;
      // map linear block index -> (p-block, q-block), p <= q
      int p = 0, rem = b;
      while (p < rb && rem >= rb - p) { rem -= rb - p; ++p; }
      bp[k] = (p < rb) ? p : -1;
      bq[k] = p + rem;
#pragma unroll
      for (int i = 0; i < 16; ++i) acc[k][i] = 0.0;
    }
  }

  // rows [0, rows) of tile (stride S doubles; columns >= r must read as 0,
  // so S >= 4*rb is required and the padding must be zeroed);
  // w == nullptr means unit weights.
  __device__ __forceinline__ void accumulate(const double *tile, int rows, int S, const double *w) {
    const int g = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      if (bp[k] < 0) continue;
      const int p0 = 4 * bp[k], q0 = 4 * bq[k];
      for (int row = g; row < rows; row += kSyrkThreads / 32) {
        const double *x = tile + row * S;
        double wr = w ? w[row] : 1.0;
        double xp[4], xq[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) { xp[i] = x[p0 + i] * wr; xq[i] = x[q0 + i]; }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[k][4 * i + j] += xp[i] * xq[j];
      }
    }
  }

  // Unit weights, even S (16-byte aligned rows): the 4+4 operands of a lane's
  // block as four 16-byte loads per row.
  __device__ __forceinline__ void accumulate_v(const double *tile, int rows, int S) {
    const int g = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      if (bp[k] < 0) continue;
      const int p0 = 4 * bp[k], q0 = 4 * bq[k];
      for (int row = g; row < rows; row += kSyrkThreads / 32) {
        const double *x = tile + row * S;
        const double2 a01 = *reinterpret_cast<const double2 *>(x + p0);
        const double2 a23 = *reinterpret_cast<const double2 *>(x + p0 + 2);
        const double2 b01 = *reinterpret_cast<const double2 *>(x + q0);
        const double2 b23 = *reinterpret_cast<const double2 *>(x + q0 + 2);
        const double xp[4] = {a01.x, a01.y, a23.x, a23.y}, xq[4] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[k][4 * i + j] += xp[i] * xq[j];
      }
    }
  }

  // Warp-private variant: this warp's lanes walk every row of a tile the warp
  // owns (rows [0, rows), stride S); finish() still sums the 8 warps.
  __device__ __forceinline__ void accumulate_warp(const double *tile, int rows, int S) {
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      if (bp[k] < 0) continue;
      const int p0 = 4 * bp[k], q0 = 4 * bq[k];
      for (int row = 0; row < rows; ++row) {
        const double *x = tile + row * S;
        double xp[4], xq[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) { xp[i] = x[p0 + i]; xq[i] = x[q0 + i]; }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[k][4 * i + j] += xp[i] * xq[j];
      }
    }
  }

  // Reduce the 8 row groups (group g adds into group 0 through a small shared
  // buffer of PER*32*16 doubles) and write the block's upper-triangle partial
  // (full r*r layout; entries p > q are not written) to out.
  __device__ __forceinline__ void finish(int r, double *scratch, double *out) {
    const int g = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int src = 1; src < kSyrkThreads / 32; ++src) {
      __syncthreads();
      if (g == src) {
#pragma unroll
        for (int k = 0; k < PER; ++k)
#pragma unroll
          for (int i = 0; i < 16; ++i) scratch[(k * 32 + lane) * 16 + i] = acc[k][i];
      }
      __syncthreads();
      if (g == 0) {
#pragma unroll
        for (int k = 0; k < PER; ++k)
#pragma unroll
          for (int i = 0; i < 16; ++i) acc[k][i] += scratch[(k * 32 + lane) * 16 + i];
      }
    }
    if (g == 0) {
#pragma unroll
      for (int k = 0; k < PER; ++k) {
        if (bp[k] < 0) continue;
        const int p0 = 4 * bp[k], q0 = 4 * bq[k];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            int p = p0 + i, q = q0 + j;
            if (p < r && q < r && p <= q) out[p * r + q] = acc[k][4 * i + j];
          }
      }
    }
  }
};

// Sum nb block partials (full r*r layout, upper triangle valid) into a full
// symmetric r x r matrix.  One warp per upper entry, double-double sums.
__global__ void k_pairs_reduce(const double *__restrict__ part, int64_t nb, int r, double *__restrict__ G,
                               const StepCtl *ctl = nullptr) {
  CPARLS_GUARD(ctl);
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= (int64_t)r * r) return;
  const int p = (int)(w / r), q = (int)(w % r);
  if (p > q) return;
  dd s = {0.0, 0.0};
  for (int64_t b = lane; b < nb; b += 32) s = dd_add_d(s, part[b * r * r + w]);
  s = warp_sum_dd(s);
  if (lane == 0) {
    double v = s.hi + s.lo;
    G[p * r + q] = v;
    G[q * r + p] = v;
  }
}

inline unsigned pairs_reduce_grid(int r) { return (unsigned)ceil_div((int64_t)r * r * 32, 256); }

}  // namespace cparls
