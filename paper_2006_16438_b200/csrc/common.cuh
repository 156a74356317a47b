// common.cuh -- device helpers shared by the cparls kernels (sm_100a).
// Part of the product path; shares nothing with oracle/.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

namespace cparls {

constexpr int kMaxModes = 8;
constexpr int kMaxRank = 64;
constexpr unsigned long long kEmptyKey = 0xFFFFFFFFFFFFFFFFull;
constexpr double kTwo62 = 4611686018427387904.0;  // 2^62

// Division by an invariant divisor 1 <= d < 2^63 for any 64-bit dividend
// (Granlund & Montgomery 1994, the round-up method): with l = ceil(log2 d),
// m = floor(2^64 (2^l - d) / d) + 1, t = mulhi(m, x):
// x / d = (t + ((x - t) >> min(l, 1))) >> max(l - 1, 0).  Replaces the ~70-
// instruction 64-bit division when decoding sample keys into indices.
struct FastDiv {
  uint64_t m = 1;
  uint64_t d = 1;
  uint32_t s1 = 0, s2 = 0;
};

inline FastDiv make_fastdiv(uint64_t d) {
  FastDiv f;
  int l = 0;
  while (l < 63 && (uint64_t(1) << l) < d) ++l;
  const unsigned __int128 num = ((unsigned __int128)((uint64_t(1) << l) - d)) << 64;
  f.m = (uint64_t)(num / d) + 1;
  f.d = d;
  f.s1 = l < 1 ? l : 1;
  f.s2 = l > 1 ? l - 1 : 0;
  return f;
}

__host__ __device__ __forceinline__ uint64_t fastdiv(uint64_t x, const FastDiv &f) {
#ifdef __CUDA_ARCH__
  const uint64_t t = __umul64hi(f.m, x);
#else
  const uint64_t t = (uint64_t)(((unsigned __int128)f.m * x) >> 64);
#endif
  return (t + ((x - t) >> f.s1)) >> f.s2;
}

// x / d with the remainder
__host__ __device__ __forceinline__ uint64_t fastdivmod(uint64_t x, const FastDiv &f, uint64_t &rem) {
  const uint64_t q = fastdiv(x, f);
  rem = x - q * f.d;
  return q;
}

struct CudaError : std::runtime_error {
  cudaError_t code;
  CudaError(cudaError_t c, const std::string &m) : std::runtime_error(m), code(c) {}
};
struct ApiError : std::runtime_error {
  int status;
  ApiError(int s, const std::string &m) : std::runtime_error(m), status(s) {}
};

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess)                                                                 \
      throw ::cparls::CudaError(e_, std::string(#x) + ": " + cudaGetErrorString(e_) + " @" + \
                                          __FILE__ + ":" + std::to_string(__LINE__));      \
  } while (0)

#define CK_LAUNCH() CK(cudaGetLastError())

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// ---------------------------------------------------------------- Philox4x32-10
struct u32x4 { uint32_t x, y, z, w; };

__device__ __forceinline__ u32x4 philox4x32_10(u32x4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int round = 0; round < 10; ++round) {
    if (round > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    u32x4 n;
    n.x = hi1 ^ c.y ^ k0; n.y = lo1; n.z = hi0 ^ c.w ^ k1; n.w = lo0;
    c = n;
  }
  return c;
}

// ---------------------------------------------------------------- double-double
struct dd { double hi, lo; };
__device__ __forceinline__ dd dd_two_sum(double a, double b) {
  double s = __dadd_rn(a, b);
  double bb = __dsub_rn(s, a);
  double err = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
  return {s, err};
}
__device__ __forceinline__ dd dd_add(dd a, dd b) {
  dd s = dd_two_sum(a.hi, b.hi);
  double lo = __dadd_rn(__dadd_rn(s.lo, a.lo), b.lo);
  return dd_two_sum(s.hi, lo);
}
__device__ __forceinline__ dd dd_add_d(dd a, double b) {
  dd s = dd_two_sum(a.hi, b);
  return dd_two_sum(s.hi, __dadd_rn(s.lo, a.lo));
}
__device__ __forceinline__ dd dd_shfl_xor(dd v, int m) {
  return {__shfl_xor_sync(0xffffffffu, v.hi, m), __shfl_xor_sync(0xffffffffu, v.lo, m)};
}
__device__ __forceinline__ dd warp_sum_dd(dd v) {
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) v = dd_add(v, dd_shfl_xor(v, m));
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
  return v;
}

// atomic max for non-negative doubles (bit pattern order == value order)
__device__ __forceinline__ void atomic_max_nonneg(double *addr, double v) {
  atomicMax(reinterpret_cast<unsigned long long *>(addr), (unsigned long long)__double_as_longlong(v));
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ---------------------------------------------------------------- L2 policies
// Streaming data (read once) is loaded evict_first and bypasses L1, so it does
// not push reused factor rows out of L2; gathered factor rows use evict_last.
__device__ __forceinline__ uint64_t l2_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t ld_stream(const uint64_t *a, uint64_t pol) {
  uint64_t v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ int32_t ld_stream(const int32_t *a, uint64_t pol) {
  int32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ float ld_stream(const float *a, uint64_t pol) {
  float v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ double ld_stream(const double *a, uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ double2 ld_keep2(const double2 *a, uint64_t pol) {
  double2 v;
  asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ void cp_async16_keep(void *smem, const void *gmem, uint64_t pol) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "l"(pol)
               : "memory");
}

// ---------------------------------------------------------------- asynchronous mode step
// Device control block of the host-synchronisation-free mode step
// (cparls.cu: sample_async / solve_async).  Every size the host used to read
// back (candidate counts, DIDX list length, s_det, p_det, SIDX progress, s_bar,
// m_k) lives here; kernels launched with upper-bound grids read them.  When a
// step needs the host-driven path (a capacity is exceeded, or a rare branch:
// the AMB-6 truncation, tau < 2^-63) a kernel raises `abort`; every guarded
// kernel after it returns at entry, so the state stays exactly as before that
// step, and the host redoes the step with the host-driven sampler at its next
// synchronisation.
struct StepCtl {
  int abort;                    // != 0: guarded kernels return at entry
  int skip;                     // AMB-7: the random phase of this step is skipped
  int64_t abort_step;         // global step (t*D + k) that raised abort (first)
  int64_t ncand[kMaxModes];   // DIDX candidates per other mode
  unsigned long long cand_acc[kMaxModes];   // k_cand_append counters (k_cand_sort moves them to ncand, resets)
  int64_t nlist;              // DIDX list length (current level)
  int64_t sdet, s_rnd, have, nuniq, sbar, attempts;
  double pdet;
  // SIDX decoupled look-back (k_sidx_run)
  unsigned long long sidx_next_tile;
  unsigned sidx_epoch;
  int sidx_done;
  int64_t scan_total;         // scratch total of the device-count scans
  int64_t nseg;               // RHS (window, fiber) segments of the step
  // statistics accumulated on the device, folded into cparls_stats at a sync
  int64_t st_steps, st_sum_mk, st_sum_sbar, st_sum_attempts, st_sum_sdet, st_sum_touched;
  int64_t st_last_mk, st_last_sbar, st_last_attempts;
  int64_t st_touched[kMaxModes];
};

#define CPARLS_GUARD(ctl)                  \
  do {                                     \
    if ((ctl) != nullptr && (ctl)->abort) \
      return;                              \
  } while (0)

// raise abort for global step `step` (the first raise records its step)
__device__ __forceinline__ void step_abort(StepCtl *ctl, int64_t step) {
  if (atomicCAS(&ctl->abort, 0, 1) == 0) ctl->abort_step = step;
}

// count that may live on the device: *n_dev if given, else n
__device__ __forceinline__ int64_t dcount(int64_t n, const int64_t *n_dev) {
  return n_dev ? *n_dev : n;
}

// first index i in [0,n) with C[i] > t (upper_bound); C non-decreasing
__device__ __forceinline__ int64_t upper_bound_u64(const uint64_t *__restrict__ C, int64_t n, uint64_t t) {
  int64_t lo = 0, len = n;
  while (len > 0) {
    int64_t half = len >> 1;
    if (__ldg(C + lo + half) <= t) { lo += half + 1; len -= half + 1; }
    else len = half;
  }
  return lo;
}

}  // namespace cparls
