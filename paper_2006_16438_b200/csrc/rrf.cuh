// rrf.cuh -- N4: randomized range finder initialization
// (sec:enron; reading AMB-34): A_k = X_(k)(:, S) Omega, S = s_init
// nonempty mode-k fibers drawn uniformly (ranked by canonical key), Omega
// standard normal.  The fibers are the runs of equal keys of the mode-k sorted
// copy; the draws scatter x_e Omega(j, :) into the zeroed M with fp64 reds
// (s_init fibers, a tiny fraction of the copy).
#pragma once
#include "common.cuh"

namespace cparls {

constexpr uint32_t kRrfTag = 0x52524600u;

__device__ __forceinline__ u32x4 rrf_words(uint64_t seed, uint64_t j, int k, uint32_t lane) {
  return philox4x32_10({(uint32_t)j, (uint32_t)(j >> 32), kRrfTag + (uint32_t)k, lane}, (uint32_t)seed,
                       (uint32_t)(seed >> 32));
}

__device__ __forceinline__ double rrf_omega(uint64_t seed, int k, uint64_t j, int c) {
  const u32x4 o = rrf_words(seed, j, k, (uint32_t)(c / 2));
  const uint64_t a = (uint64_t)o.x | ((uint64_t)o.y << 32), b = (uint64_t)o.z | ((uint64_t)o.w << 32);
  const double u1 = (double)((a >> 11) + 1) * 0x1p-53, u2 = (double)(b >> 11) * 0x1p-53;
  const double rho = sqrt(-2.0 * log(u1));
  const double th = 2.0 * 3.14159265358979323846 * u2;
  return (c % 2 == 0) ? rho * cos(th) : rho * sin(th);
}

// fiber starts of a sorted key array: flag[e] = (e == 0 || key[e] != key[e-1])
__global__ void k_fiber_flags(const uint64_t *__restrict__ keys, int64_t nnz, int64_t *__restrict__ flag) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x)
    flag[e] = (e == 0 || keys[e] != keys[e - 1]) ? 1 : 0;
}

// compacted fibers: start, length, canonical key (the copy key re-encoded)
struct KeyToCanon {
  int d;
  int64_t n[kMaxModes];      // copy order dims (fastest first)
  uint64_t cmult[kMaxModes]; // multiplier of copy digit j in the canonical key
};
__global__ void k_fiber_list(const uint64_t *__restrict__ keys, int64_t nnz, const int64_t *__restrict__ flag,
                             const int64_t *__restrict__ pos, KeyToCanon kc, int64_t *__restrict__ fstart,
                             uint64_t *__restrict__ fkey) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
    if (!flag[e]) continue;
    uint64_t t = keys[e], ck = 0;
    for (int j = 0; j < kc.d; ++j) {
      const uint64_t q = t / (uint64_t)kc.n[j];
      ck += (t - q * (uint64_t)kc.n[j]) * kc.cmult[j];
      t = q;
    }
    fstart[pos[e]] = e;
    fkey[pos[e]] = ck;
  }
}

// one warp per draw j: fiber u = mulhi(R, nfib) (rank in canonical order,
// perm maps rank -> compacted fiber), lanes = columns
__global__ void k_rrf_scatter(int64_t s_init, uint64_t seed, int k, int64_t nfib, const uint32_t *__restrict__ perm,
                              const int64_t *__restrict__ fstart, int64_t nnz, const int32_t *__restrict__ outidx,
                              const void *__restrict__ vals, int vf32, int r, int ld, double *__restrict__ M) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t j = w0; j < s_init; j += nw) {
    const u32x4 o = rrf_words(seed, (uint64_t)j, k, 0xFFFFu);
    const int64_t u = (int64_t)__umul64hi((uint64_t)o.x | ((uint64_t)o.y << 32), (uint64_t)nfib);
    const int64_t f = perm ? (int64_t)perm[u] : u;
    const int64_t e0 = fstart[f], e1 = (f + 1 < nfib) ? fstart[f + 1] : nnz;
    const double om0 = lane < r ? rrf_omega(seed, k, (uint64_t)j, lane) : 0.0;
    const double om1 = lane + 32 < r ? rrf_omega(seed, k, (uint64_t)j, lane + 32) : 0.0;
    for (int64_t e = e0; e < e1; ++e) {
      const int64_t i = outidx[e];
      const double x = vf32 ? (double)reinterpret_cast<const float *>(vals)[e]
                            : reinterpret_cast<const double *>(vals)[e];
      if (lane < r) atomicAdd(M + i * ld + lane, x * om0);
      if (lane + 32 < r) atomicAdd(M + i * ld + lane + 32, x * om1);
    }
  }
}

}  // namespace cparls
