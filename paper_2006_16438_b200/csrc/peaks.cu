// peaks.cu -- measurement-only microbenchmarks (libcparls_peaks.so), used by
// bench.py to put the hot kernels next to the hardware ceiling of their own
// access pattern.  Not part of the method and not called by libcparls.
//
// cparls_peak_red_f64: sustained rate of r-lane fp64 reductions (one
//   red.global.add.f64 per lane, lanes = columns of one row-major row) into
//   uniformly random rows of an n x ld matrix -- the access pattern of k_rhs.
// cparls_peak_gather: sustained rate of r-wide fp64 row gathers (16-byte loads,
//   ld/4 lanes per row) from uniformly random rows -- the pattern of k_fit_sub.
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

__device__ __forceinline__ uint32_t mix32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

__global__ void k_peak_red(double *M, int64_t rows, int r, int ld, int64_t ops_per_warp, uint32_t salt) {
  const int lane = threadIdx.x & 31;
  const uint32_t wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  for (int64_t i = 0; i < ops_per_warp; ++i) {
    const uint32_t h = mix32(wid * 0x9E3779B9u + (uint32_t)i * 0x85EBCA6Bu + salt);
    const int64_t row = (int64_t)(((uint64_t)h * (uint64_t)rows) >> 32);
    if (lane < r) atomicAdd(M + row * ld + lane, 1e-3);
  }
}

// same pattern with 64-bit integer and 32-bit float reductions (what a
// fixed-point or single-precision accumulation would cost)
template <typename T>
__global__ void k_peak_red_t(T *M, int64_t rows, int r, int ld, int64_t ops_per_warp, uint32_t salt) {
  const int lane = threadIdx.x & 31;
  const uint32_t wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  for (int64_t i = 0; i < ops_per_warp; ++i) {
    const uint32_t h = mix32(wid * 0x9E3779B9u + (uint32_t)i * 0x85EBCA6Bu + salt);
    const int64_t row = (int64_t)(((uint64_t)h * (uint64_t)rows) >> 32);
    if (lane < r) atomicAdd(M + row * ld + lane, (T)3);
  }
}

// reductions into the rows of a given index stream (e.g. the tensor's own
// mode coordinates): warp w walks idx[w*per_warp ...), lane c adds to column c
template <typename T>
__global__ void k_peak_red_idx(T *M, const int32_t *__restrict__ idx, int64_t n, int r, int ld,
                               int64_t per_warp) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t b = wid * per_warp, e = min(n, b + per_warp);
  for (int64_t i = b; i < e; ++i) {
    const int64_t row = __ldg(idx + i);
    if (lane < r) atomicAdd(M + row * ld + lane, (T)3);
  }
}

template <int SW>
__global__ void k_peak_gather(const double *__restrict__ A, int64_t rows, int ld, int64_t rows_per_warp,
                              double *out) {
  const int lane = threadIdx.x & 31;
  const int sl = lane & (SW - 1);
  const uint32_t wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  double acc = 0.0;
  for (int64_t i = 0; i < rows_per_warp; i += 32 / SW * 4) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t h = mix32(wid * 0x9E3779B9u + (uint32_t)(i + u * (32 / SW) + lane / SW) * 0x85EBCA6Bu);
      const int64_t row = (int64_t)(((uint64_t)h * (uint64_t)rows) >> 32);
      if (4 * sl < ld) {
        const double2 *p = reinterpret_cast<const double2 *>(A + row * ld + 4 * sl);
        const double2 a = __ldg(p), b = __ldg(p + 1);
        acc += a.x + a.y + b.x + b.y;
      }
    }
  }
  if (acc == 1234.5) out[0] = acc;   // keep the loads
}

}  // namespace

extern "C" {

// Returns lane-ops per second (rows * r reductions / time).  M: device buffer of
// rows * ld doubles (contents are overwritten).  Times `reps` launches with
// CUDA events on the default stream after one warm-up launch.
double cparls_peak_red_f64(double *M, int64_t rows, int r, int ld, int64_t ops_per_warp, int blocks, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k_peak_red<<<blocks, 256>>>(M, rows, r, ld, ops_per_warp, 1u);
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) k_peak_red<<<blocks, 256>>>(M, rows, r, ld, ops_per_warp, 7u + i);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  if (cudaGetLastError() != cudaSuccess || ms <= 0.f) return -1.0;
  const double ops = (double)reps * blocks * (256 / 32) * (double)ops_per_warp * r;
  return ops / (ms * 1e-3);
}

// kind 0: unsigned long long, 1: float.  Returns lane-ops per second.
double cparls_peak_red_kind(void *M, int64_t rows, int r, int ld, int64_t ops_per_warp, int blocks, int reps,
                            int kind) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto launch = [&](uint32_t salt) {
    if (kind == 0)
      k_peak_red_t<unsigned long long><<<blocks, 256>>>((unsigned long long *)M, rows, r, ld, ops_per_warp, salt);
    else
      k_peak_red_t<float><<<blocks, 256>>>((float *)M, rows, r, ld, ops_per_warp, salt);
  };
  launch(1u);
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) launch(7u + i);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  if (cudaGetLastError() != cudaSuccess || ms <= 0.f) return -1.0;
  return (double)reps * blocks * 8 * (double)ops_per_warp * r / (ms * 1e-3);
}

// kind 0: unsigned long long, 2: double.  idx: n device row ids (< rows of M).
// Returns lane-ops per second (n * r / time).
double cparls_peak_red_idx(void *M, const int32_t *idx, int64_t n, int r, int ld, int blocks, int reps, int kind) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int64_t warps = (int64_t)blocks * 8;
  const int64_t per_warp = (n + warps - 1) / warps;
  auto launch = [&]() {
    if (kind == 0)
      k_peak_red_idx<unsigned long long><<<blocks, 256>>>((unsigned long long *)M, idx, n, r, ld, per_warp);
    else
      k_peak_red_idx<double><<<blocks, 256>>>((double *)M, idx, n, r, ld, per_warp);
  };
  launch();
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) launch();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  if (cudaGetLastError() != cudaSuccess || ms <= 0.f) return -1.0;
  return (double)reps * (double)n * r / (ms * 1e-3);
}

// Returns bytes per second of row data gathered (rows gathered * ld * 8 / time).
double cparls_peak_gather(const double *A, int64_t rows, int ld, int64_t rows_per_warp, int blocks, int reps,
                          double *scratch) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto launch = [&]() {
    if (ld <= 8) k_peak_gather<2><<<blocks, 256>>>(A, rows, ld, rows_per_warp, scratch);
    else if (ld <= 32) k_peak_gather<8><<<blocks, 256>>>(A, rows, ld, rows_per_warp, scratch);
    else k_peak_gather<16><<<blocks, 256>>>(A, rows, ld, rows_per_warp, scratch);
  };
  launch();
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) launch();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  if (cudaGetLastError() != cudaSuccess || ms <= 0.f) return -1.0;
  const double nrows = (double)reps * blocks * (256 / 32) * (double)rows_per_warp;
  return nrows * ld * 8.0 / (ms * 1e-3);
}

}  // extern "C"
