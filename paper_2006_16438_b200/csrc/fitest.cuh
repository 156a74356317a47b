// fitest.cuh -- estimated fit by stratified sampling (sec:estimating-fit,
// P:964-989; readings AMB-32/33 in DESIGN.md).
//
// The sample is drawn once, inside cparls_create ("We sample the
// elements of the tensor once at the beginning"): ceil(alpha s_fit) nonzeros
// uniformly with replacement from the input COO order, and the first
// floor((1-alpha) s_fit) uniform cells that are not nonzeros (rejection,
// attempt order).  Membership of a proposed cell is decided on the mode-0
// sorted copy: its key range (directory + binary search), then a binary
// search of i_0 among the fiber's row-sorted entries.  The estimate
// F^ = sum_i phi_i (m_i - x_i)^2 is one gather pass over the frozen sample.
#pragma once
#include "common.cuh"

namespace cparls {

constexpr uint32_t kFitSampleTag = 0x46495400u;

__device__ __forceinline__ uint64_t fs_word(uint64_t seed, uint64_t ctr, uint32_t lane, int half) {
  const u32x4 o = philox4x32_10({(uint32_t)ctr, (uint32_t)(ctr >> 32), kFitSampleTag, lane}, (uint32_t)seed,
                                (uint32_t)(seed >> 32));
  return half == 0 ? ((uint64_t)o.x | ((uint64_t)o.y << 32)) : ((uint64_t)o.z | ((uint64_t)o.w << 32));
}

struct FitSampleDev {
  int D;
  int64_t dims[kMaxModes];
  int32_t *idx[kMaxModes];   // per mode, n_total entries
  double *x;
};

// nonzero stratum: draw i -> COO entry e = mulhi(R, nnz)
template <typename IT, typename VT>
__global__ void k_fs_nz(const IT *__restrict__ coords, const VT *__restrict__ vals, int64_t nnz, int64_t n_nz,
                        uint64_t seed, FitSampleDev fs) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_nz) return;
  const int64_t e = (int64_t)__umul64hi(fs_word(seed, (uint64_t)i, 0u, 0), (uint64_t)nnz);
  for (int m = 0; m < fs.D; ++m) fs.idx[m][i] = (int32_t)coords[e * fs.D + m];
  fs.x[i] = (double)vals[e];
}

// Mode-0 copy view for the membership test: keys ordered by `order`
// (fastest first), sorted by (key, out).
struct MemberIndex {
  const uint64_t *key;
  const int32_t *out;
  const int64_t *dir;
  int shift;
  int64_t nbkt;
  int d;
  int order[kMaxModes];
  uint64_t mult[kMaxModes];
};

__device__ __forceinline__ bool is_nonzero(const MemberIndex &mi, const int64_t *ii) {
  uint64_t k = 0;
  for (int j = 0; j < mi.d; ++j) k += (uint64_t)ii[mi.order[j]] * mi.mult[j];
  const uint64_t b = k >> mi.shift;
  if ((int64_t)b >= mi.nbkt) return false;
  int64_t L = __ldg(mi.dir + b), len = __ldg(mi.dir + b + 1) - L;
  while (len > 0) {   // lower_bound of k
    const int64_t h = len >> 1;
    if (__ldg(mi.key + L + h) < k) { L += h + 1; len -= h + 1; }
    else len = h;
  }
  int64_t U = L;
  len = __ldg(mi.dir + b + 1) - L;
  while (len > 0) {   // upper_bound of k
    const int64_t h = len >> 1;
    if (__ldg(mi.key + U + h) <= k) { U += h + 1; len -= h + 1; }
    else len = h;
  }
  const int32_t o = (int32_t)ii[0];
  while (U - L > 0) {   // binary search of i_0 among the fiber's sorted rows
    const int64_t mid = L + ((U - L) >> 1);
    const int32_t v = __ldg(mi.out + mid);
    if (v == o) return true;
    if (v < o) L = mid + 1;
    else U = mid;
  }
  return false;
}

// zero stratum, attempts [a0, a0 + win): accepted flag (0/1) per attempt, and
// the proposed cell
__global__ void k_fs_zero_gen(MemberIndex mi, int D, FitSampleDev fs,
                              uint64_t seed, uint64_t a0, int64_t win, int64_t *__restrict__ flag,
                              int32_t *__restrict__ cell /* win x D */) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= win) return;
  const uint64_t a = a0 + (uint64_t)t;
  int64_t ii[kMaxModes];
  for (int m = 0; m < D; ++m) {
    const uint64_t R = fs_word(seed, a, 1u + (uint32_t)(m / 2), m % 2);
    ii[m] = (int64_t)__umul64hi(R, (uint64_t)fs.dims[m]);
    cell[t * D + m] = (int32_t)ii[m];
  }
  flag[t] = is_nonzero(mi, ii) ? 0 : 1;
}

// accepted attempts in order: exclusive rank pos[t]; keep ranks < need
__global__ void k_fs_zero_scatter(const int64_t *__restrict__ flag, const int64_t *__restrict__ pos, int64_t win,
                                  const int32_t *__restrict__ cell, int D, int64_t base, int64_t need,
                                  FitSampleDev fs, unsigned long long *last_attempt, uint64_t a0) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= win || !flag[t]) return;
  const int64_t q = pos[t];
  if (q >= need) return;
  for (int m = 0; m < D; ++m) fs.idx[m][base + q] = cell[t * D + m];
  fs.x[base + q] = 0.0;
  if (q == need - 1) *last_attempt = (unsigned long long)(a0 + (uint64_t)t);
}

// F^ partials: sub-warp of SW lanes per sample, 4 columns per lane.
template <int SW>
__global__ void __launch_bounds__(256) k_fit_est(FitSampleDev fs, int64_t n_nz, int64_t n_tot, double phi_nz,
                                                 double phi_z, FitDecode fa, const double *__restrict__ lam, int r,
                                                 int ld,
                                                 dd *__restrict__ part) {
  // fa.A[m] = factor of mode m (all D modes, canonical order), fa.d = D
  const int lane = threadIdx.x & 31, sl = lane & (SW - 1);
  const int c0 = 4 * sl;
  const bool colok = c0 < ld;
  double lam4[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) lam4[q] = (c0 + q < r) ? lam[c0 + q] : 0.0;
  dd acc = {0.0, 0.0};
  const int64_t per = 32 / SW;
  const int64_t gsub = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / SW;
  const int64_t nsub = (int64_t)gridDim.x * blockDim.x / SW;
  for (int64_t i0 = gsub - (gsub % per); i0 < n_tot; i0 += nsub) {
    const int64_t i = i0 + (gsub % per);
    const bool valid = i < n_tot;
    double h[4] = {lam4[0], lam4[1], lam4[2], lam4[3]};
    if (valid && colok) {
      for (int m = 0; m < fa.d; ++m) {
        double p0x, p0y, p1x, p1y;   // one 256-bit load (rows are 32-byte aligned)
        asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
            : "=d"(p0x), "=d"(p0y), "=d"(p1x), "=d"(p1y)
            : "l"(fa.A[m] + (int64_t)fs.idx[m][i] * ld + c0));
        h[0] *= p0x; h[1] *= p0y; h[2] *= p1x; h[3] *= p1y;
      }
    } else {
      h[0] = h[1] = h[2] = h[3] = 0.0;
    }
    double mpart = (h[0] + h[1]) + (h[2] + h[3]);
#pragma unroll
    for (int o = SW / 2; o >= 1; o >>= 1) mpart += __shfl_xor_sync(0xffffffffu, mpart, o, SW);
    if (valid && sl == 0) {
      const double dlt = mpart - fs.x[i];
      acc = dd_add_d(acc, (i < n_nz ? phi_nz : phi_z) * (dlt * dlt));
    }
  }
  acc = warp_sum_dd(acc);
  __shared__ dd ws[8];
  if (lane == 0) ws[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    dd t = {0.0, 0.0};
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t = dd_add(t, ws[w]);
    part[blockIdx.x] = t;
  }
}

// m_i at every sample position (diagnostics: cparls_fit_sample_model), the
// same arithmetic as k_fit_est
template <int SW>
__global__ void __launch_bounds__(256) k_fit_est_model(FitSampleDev fs, int64_t n_tot, FitDecode fa,
                                                       const double *__restrict__ lam, int r, int ld,
                                                       double *__restrict__ mout) {
  const int lane = threadIdx.x & 31, sl = lane & (SW - 1);
  const int c0 = 4 * sl;
  const bool colok = c0 < ld;
  double lam4[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) lam4[q] = (c0 + q < r) ? lam[c0 + q] : 0.0;
  const int64_t per = 32 / SW;
  const int64_t gsub = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / SW;
  const int64_t nsub = (int64_t)gridDim.x * blockDim.x / SW;
  for (int64_t i0 = gsub - (gsub % per); i0 < n_tot; i0 += nsub) {
    const int64_t i = i0 + (gsub % per);
    const bool valid = i < n_tot;
    double h[4] = {lam4[0], lam4[1], lam4[2], lam4[3]};
    if (valid && colok) {
      for (int m = 0; m < fa.d; ++m) {
        double p0x, p0y, p1x, p1y;   // one 256-bit load (rows are 32-byte aligned)
        asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
            : "=d"(p0x), "=d"(p0y), "=d"(p1x), "=d"(p1y)
            : "l"(fa.A[m] + (int64_t)fs.idx[m][i] * ld + c0));
        h[0] *= p0x; h[1] *= p0y; h[2] *= p1x; h[3] *= p1y;
      }
    } else {
      h[0] = h[1] = h[2] = h[3] = 0.0;
    }
    double mpart = (h[0] + h[1]) + (h[2] + h[3]);
#pragma unroll
    for (int o = SW / 2; o >= 1; o >>= 1) mpart += __shfl_xor_sync(0xffffffffu, mpart, o, SW);
    if (valid && sl == 0) mout[i] = mpart;
  }
}

// F^ = sum of partials; out[0] = 1 - sqrt(max(F^,0))/||X||, out[1] = F^
__global__ void k_fit_est_final(const dd *__restrict__ part, int nb, double normX2, double *out) {
  __shared__ dd red[256];
  dd s = {0.0, 0.0};
  for (int i = threadIdx.x; i < nb; i += blockDim.x) s = dd_add(s, part[i]);
  red[threadIdx.x] = s;
  __syncthreads();
  for (int k = blockDim.x / 2; k > 0; k >>= 1) {
    if (threadIdx.x < k) red[threadIdx.x] = dd_add(red[threadIdx.x], red[threadIdx.x + k]);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double F = red[0].hi + red[0].lo;
    out[0] = 1.0 - sqrt(F > 0.0 ? F : 0.0) / sqrt(normX2);
    out[1] = F;
  }
}

}  // namespace cparls
