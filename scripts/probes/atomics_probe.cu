// atomics_probe.cu -- measurement-only: what an r-wide row accumulation costs
// on B200 in each memory level, to choose the sampled-RHS (k_rhs) design.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o atomics_probe atomics_probe.cu
// Prints one line per pattern: lane-ops/s (or bytes/s for gathers).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t mix32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}
__device__ __forceinline__ int64_t rnd_row(uint32_t wid, int64_t i, uint32_t salt, int64_t rows) {
  const uint32_t h = mix32(wid * 0x9E3779B9u + (uint32_t)i * 0x85EBCA6Bu + salt);
  return (int64_t)(((uint64_t)h * (uint64_t)rows) >> 32);
}

// 25-lane u64 red per row (k_rhs today)
__global__ void k_red_u64(unsigned long long *M, int64_t rows, int r, int ld, int64_t per_warp, uint32_t salt) {
  const int lane = threadIdx.x & 31;
  const uint32_t wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  for (int64_t i = 0; i < per_warp; ++i) {
    const int64_t row = rnd_row(wid, i, salt, rows);
    if (lane < r) atomicAdd(M + row * ld + lane, 3ull);
  }
}
__global__ void k_red_u32(unsigned *M, int64_t rows, int r, int ld, int64_t per_warp, uint32_t salt) {
  const int lane = threadIdx.x & 31;
  const uint32_t wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  for (int64_t i = 0; i < per_warp; ++i) {
    const int64_t row = rnd_row(wid, i, salt, rows);
    if (lane < r) atomicAdd(M + row * ld + lane, 3u);
  }
}
// f32x4 vector reductions: ceil(r/4) lanes per row, 16 B each
__global__ void k_red_f32x4(float *M, int64_t rows, int r, int ld, int64_t per_warp, uint32_t salt) {
  const int lane = threadIdx.x & 31;
  const uint32_t wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nl = (r + 3) / 4;
  for (int64_t i = 0; i < per_warp; ++i) {
    const int64_t row = rnd_row(wid, i, salt, rows);
    if (lane < nl) {
      float *p = M + row * ld + 4 * lane;
      asm volatile("red.global.add.v4.f32 [%0], {%1,%1,%1,%1};" ::"l"(p), "f"(1.0f) : "memory");
    }
  }
}
// 4 rows per warp instruction (8 lanes x v4 each): 4x fewer instructions
__global__ void k_red_f32x4_4rows(float *M, int64_t rows, int r, int ld, int64_t per_warp, uint32_t salt) {
  const int lane = threadIdx.x & 31;
  const uint32_t wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int sub = lane >> 3, sl = lane & 7;
  const int nl = (r + 3) / 4;
  for (int64_t i = 0; i < per_warp; i += 4) {
    const int64_t row = rnd_row(wid, i + sub, salt, rows);
    if (sl < nl) {
      float *p = M + row * ld + 4 * sl;
      asm volatile("red.global.add.v4.f32 [%0], {%1,%1,%1,%1};" ::"l"(p), "f"(1.0f) : "memory");
    }
  }
}
// L2 gather of 256-B rows (ld doubles) from a small (L2-resident) matrix, 8 lanes x 32 B per row
__global__ void k_gather(const double *__restrict__ Z, int64_t rows, int ld, int64_t per_warp, double *out,
                         uint32_t salt) {
  const int lane = threadIdx.x & 31;
  const uint32_t wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int sub = lane >> 3, sl = lane & 7;
  double acc = 0.0;
  for (int64_t i = 0; i < per_warp; i += 16) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t row = rnd_row(wid, i + 4 * u + sub, salt, rows);
      if (4 * sl < ld) {
        const double2 *p = reinterpret_cast<const double2 *>(Z + row * ld + 4 * sl);
        const double2 a = __ldg(p), b = __ldg(p + 1);
        acc += a.x + a.y + b.x + b.y;
      }
    }
  }
  if (acc == 1234.5) out[0] = acc;
}
// shared memory: 25-lane u64 atomics into random rows of a smem tile
__global__ void k_smem_atom(int srows, int r, int ld, int64_t per_warp, unsigned long long *out, uint32_t salt) {
  extern __shared__ unsigned long long sm[];
  for (int i = threadIdx.x; i < srows * ld; i += blockDim.x) sm[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint32_t wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  for (int64_t i = 0; i < per_warp; ++i) {
    const int row = (int)rnd_row(wid, i, salt, srows);
    if (lane < r) atomicAdd(sm + row * ld + lane, 3ull);
  }
  __syncthreads();
  if (threadIdx.x == 0 && sm[0] == 12345) out[0] = sm[1];
}
// shared memory: plain read-modify-write (warp-private tiles: no races)
__global__ void k_smem_rmw(int srows, int r, int ld, int64_t per_warp, unsigned long long *out, uint32_t salt) {
  extern __shared__ unsigned long long sm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned long long *t = sm + (size_t)w * srows * ld;
  for (int i = lane; i < srows * ld; i += 32) t[i] = 0;
  __syncwarp();
  const uint32_t wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  for (int64_t i = 0; i < per_warp; ++i) {
    const int row = (int)rnd_row(wid, i, salt, srows);
    if (lane < r) t[row * ld + lane] += 3ull;
    __syncwarp();
  }
  if (lane == 0 && t[0] == 12345) out[0] = t[1];
}

// plain stores of 25 u64 per random row (the SM->L2 write path without the atomic unit)
__global__ void k_store_u64(unsigned long long *M, int64_t rows, int r, int ld, int64_t per_warp, uint32_t salt) {
  const int lane = threadIdx.x & 31;
  const uint32_t wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  for (int64_t i = 0; i < per_warp; ++i) {
    const int64_t row = rnd_row(wid, i, salt, rows);
    if (lane < r) M[row * ld + lane] = (unsigned long long)i;
  }
}
// smem read-modify-write with 4 independent rows in flight per warp (ILP)
__global__ void k_smem_rmw4(int srows, int r, int ld, int64_t per_warp, unsigned long long *out, uint32_t salt) {
  extern __shared__ unsigned long long sm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned long long *t = sm + (size_t)w * srows * ld;
  for (int i = lane; i < srows * ld; i += 32) t[i] = 0;
  __syncwarp();
  const uint32_t wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int q = srows / 4;
  for (int64_t i = 0; i < per_warp; i += 4) {
    int row[4];
    unsigned long long v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) row[u] = u * q + (int)rnd_row(wid, i + u, salt, q);
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = lane < r ? t[row[u] * ld + lane] : 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) if (lane < r) t[row[u] * ld + lane] = v[u] + 3ull;
  }
  if (lane == 0 && t[0] == 12345) out[0] = t[1];
}

__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}
// the k_rhs pattern restricted to CTAs on SMs < nsm (the others exit): does the
// SM->L2 write path saturate with part of the chip?  Work counter = fixed total.
__global__ void k_red_u64_sm(unsigned long long *M, int64_t rows, int r, int ld, int64_t total, unsigned nsm,
                             unsigned long long *work, uint32_t salt) {
  if (smid() >= nsm) return;
  const int lane = threadIdx.x & 31;
  while (true) {
    unsigned long long t0 = 0;
    if (lane == 0) t0 = atomicAdd(work, 64ull);
    t0 = __shfl_sync(0xffffffffu, t0, 0);
    if ((int64_t)t0 >= total) break;
    for (int i = 0; i < 64; ++i) {
      const int64_t row = rnd_row((uint32_t)t0, i, salt, rows);
      if (lane < r) atomicAdd(M + row * ld + lane, 3ull);
    }
  }
}
// random 256-B row gathers (the fit's pattern) restricted to SMs < nsm
__global__ void k_gather_sm(const double *__restrict__ Z, int64_t rows, int ld, int64_t total, unsigned nsm,
                            unsigned long long *work, double *out, uint32_t salt) {
  if (smid() >= nsm) return;
  const int lane = threadIdx.x & 31;
  const int sub = lane >> 3, sl = lane & 7;
  double acc = 0.0;
  while (true) {
    unsigned long long t0 = 0;
    if (lane == 0) t0 = atomicAdd(work, 256ull);
    t0 = __shfl_sync(0xffffffffu, t0, 0);
    if ((int64_t)t0 >= total) break;
    for (int i = 0; i < 256; i += 16) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t row = rnd_row((uint32_t)t0, i + 4 * u + sub, salt, rows);
        const double2 *p = reinterpret_cast<const double2 *>(Z + row * ld + 4 * sl);
        const double2 a = __ldg(p), b = __ldg(p + 1);
        acc += a.x + a.y + b.x + b.y;
      }
    }
  }
  if (acc == 1234.5) out[0] = acc;
}

template <typename L>
float time_it(L launch, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  launch(1u);
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) launch(7u + i);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return ms / reps;
}

int main() {
  const int r = 25, ld = 32;
  const int blocks = 148 * 8, threads = 256;
  const int64_t warps = (int64_t)blocks * threads / 32;
  void *M;
  cudaMalloc(&M, (size_t)4 << 30);
  cudaMemset(M, 0, (size_t)4 << 30);
  double *scr;
  cudaMalloc(&scr, 64);
  const int64_t pw = 4096;
  const double lane_ops = (double)warps * pw * r;
  for (int64_t rows : {int64_t(4096), int64_t(65536), int64_t(393216), int64_t(1805187), int64_t(4821207)}) {
    float ms = time_it([&](uint32_t s) { k_red_u64<<<blocks, threads>>>((unsigned long long *)M, rows, r, ld, pw, s); }, 3);
    printf("red.u64  x25 lanes rows=%8lld (%6.1f MB): %7.1f G lane-ops/s  %6.2f G rows/s\n", (long long)rows,
           rows * ld * 8 / 1e6, lane_ops / ms / 1e6, warps * pw / ms / 1e6);
    ms = time_it([&](uint32_t s) { k_red_u32<<<blocks, threads>>>((unsigned *)M, rows, r, ld, pw, s); }, 3);
    printf("red.u32  x25 lanes rows=%8lld: %7.1f G lane-ops/s  %6.2f G rows/s\n", (long long)rows, lane_ops / ms / 1e6,
           warps * pw / ms / 1e6);
    ms = time_it([&](uint32_t s) { k_red_f32x4<<<blocks, threads>>>((float *)M, rows, r, ld, pw, s); }, 3);
    printf("red.v4.f32 x7 lanes rows=%8lld: %6.2f G rows/s (= %7.1f G col-ops/s)\n", (long long)rows,
           warps * pw / ms / 1e6, lane_ops / ms / 1e6);
    ms = time_it([&](uint32_t s) { k_red_f32x4_4rows<<<blocks, threads>>>((float *)M, rows, r, ld, pw, s); }, 3);
    printf("red.v4.f32 4 rows/instr rows=%8lld: %6.2f G rows/s\n", (long long)rows, warps * pw / ms / 1e6);
    ms = time_it([&](uint32_t s) { k_store_u64<<<blocks, threads>>>((unsigned long long *)M, rows, r, ld, pw, s); }, 3);
    printf("st.u64 x25 lanes rows=%8lld: %7.1f G lane-ops/s  %6.2f G rows/s\n", (long long)rows, lane_ops / ms / 1e6,
           warps * pw / ms / 1e6);
  }
  for (int64_t rows : {int64_t(131072), int64_t(393216), int64_t(1805187)}) {
    const int64_t pwg = 1 << 14;
    float ms = time_it([&](uint32_t s) { k_gather<<<blocks, threads>>>((const double *)M, rows, ld, pwg, scr, s); }, 3);
    const double bytes = (double)warps * pwg * ld * 8;
    printf("gather 256-B rows from %8lld rows (%6.1f MB): %7.1f GB/s  %6.2f G rows/s\n", (long long)rows,
           rows * ld * 8 / 1e6, bytes / ms / 1e6, warps * pwg / ms / 1e6);
  }
  {
    unsigned long long *work;
    cudaMalloc(&work, 8);
    const int64_t total = 1 << 26;
    for (unsigned nsm : {37u, 74u, 111u, 148u}) {
      float ms = time_it([&](uint32_t s) {
        cudaMemset(work, 0, 8);
        k_red_u64_sm<<<blocks, threads>>>((unsigned long long *)M, 393216, r, ld, total, nsm, work, s);
      }, 3);
      printf("red.u64 x25 on %3u SMs: %6.2f G rows/s\n", nsm, total / ms / 1e6);
      ms = time_it([&](uint32_t s) {
        cudaMemset(work, 0, 8);
        k_gather_sm<<<blocks, threads>>>((const double *)M, 1805187, ld, total, nsm, work, scr, s);
      }, 3);
      printf("gather 256-B rows (1.8M rows) on %3u SMs: %6.2f G rows/s  %7.1f GB/s\n", nsm, total / ms / 1e6,
             total * 256.0 / ms / 1e6);
    }
  }
  {
    int srows = 800;
    size_t sm = (size_t)srows * ld * 8;
    cudaFuncSetAttribute(k_smem_atom, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    float ms = time_it([&](uint32_t s) { k_smem_atom<<<148, 256, sm>>>(srows, r, ld, pw, (unsigned long long *)scr, s); }, 3);
    const double lo = 148.0 * 8 * pw * r;
    printf("smem atom.u64 x25 (800-row tile, 1 CTA/SM x 8 warps): %7.1f G lane-ops/s\n", lo / ms / 1e6);
    srows = 96;
    sm = (size_t)8 * srows * ld * 8;
    cudaFuncSetAttribute(k_smem_rmw, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    ms = time_it([&](uint32_t s) { k_smem_rmw<<<148, 256, sm>>>(srows, r, ld, pw, (unsigned long long *)scr, s); }, 3);
    printf("smem rmw u64 x25 (warp-private 96 rows, 8 warps/SM): %7.1f G lane-ops/s\n", lo / ms / 1e6);
    cudaFuncSetAttribute(k_smem_rmw4, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    ms = time_it([&](uint32_t s) { k_smem_rmw4<<<148, 256, sm>>>(srows, r, ld, pw, (unsigned long long *)scr, s); }, 3);
    printf("smem rmw4 u64 x25 (4 rows in flight, 8 warps/SM): %7.1f G lane-ops/s\n", lo / ms / 1e6);
    ms = time_it([&](uint32_t s) { k_smem_rmw4<<<296, 256, sm>>>(srows, r, ld, pw, (unsigned long long *)scr, s); }, 3);
    printf("smem rmw4 u64 x25 (4 rows in flight, 2 CTAs x 8 warps/SM): %7.1f G lane-ops/s\n", 2 * lo / ms / 1e6);
  }
  return 0;
}
