// tma_red_probe.cu -- measurement-only: can the TMA bulk-reduction path
// (cp.reduce.async.bulk .add.u64, shared -> global) move r-wide int64 row
// accumulations faster than per-lane red.global.add.u64 (k_rhs today, bound by
// the SM -> L2 write-request interface, ~0.18 lines/clock/SM)?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_red_probe tma_red_probe.cu
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

// baseline: 25-lane u64 red per row
__global__ void k_red_u64(unsigned long long *M, int64_t rows, int r, int ld, int64_t per_warp, uint32_t salt) {
  const int lane = threadIdx.x & 31;
  const uint32_t wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  for (int64_t i = 0; i < per_warp; ++i) {
    const int64_t row = rnd_row(wid, i, salt, rows);
    if (lane < r) atomicAdd(M + row * ld + lane, 3ull);
  }
}

// TMA bulk reduce: each warp owns a ring of NSLOT staging rows of RB bytes;
// per row lanes write the row's values, one lane issues the bulk reduction.
// RPI rows are staged per warp step (lanes split over rows), each issued by
// its own lane so the uniform datapath loops over RPI issuers.
template <bool F64, int RPI>
__global__ void k_tma_red(void *M, int64_t rows, int ld, int rb_bytes, int nslot, int64_t per_warp, uint32_t salt) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int rw = rb_bytes / 8;                 // u64 words per staged row
  unsigned long long *ring = reinterpret_cast<unsigned long long *>(smem) + (size_t)w * nslot * RPI * rw;
  const uint32_t wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lpr = 32 / RPI;                    // lanes per row
  const int sub = lane / lpr, sl = lane % lpr;
  int slot = 0;
  for (int64_t i = 0; i < per_warp; i += RPI) {
    // slot reuse: at most nslot-1 older groups may still be reading
    if (sl == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(3) : "memory");
    __syncwarp();
    unsigned long long *dst = ring + (size_t)(slot * RPI + sub) * rw;
    for (int c = sl; c < rw; c += lpr) {
      if (F64) reinterpret_cast<double *>(dst)[c] = 1.0;
      else dst[c] = 3ull;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (sl == 0) {
      const int64_t row = rnd_row(wid, i + sub, salt, rows);
      const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
      if (F64) {
        double *g = reinterpret_cast<double *>(M) + row * ld;
        asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], %2;" ::"l"(g), "r"(sa),
                     "r"(rb_bytes) : "memory");
      } else {
        unsigned long long *g = reinterpret_cast<unsigned long long *>(M) + row * ld;
        asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.u64 [%0], [%1], %2;" ::"l"(g), "r"(sa),
                     "r"(rb_bytes) : "memory");
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    slot = (slot + 1) % nslot;
  }
  if (lane % lpr == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// TMA bulk store of the same staged rows (the write path without reduction)
template <int RPI>
__global__ void k_tma_st(void *M, int64_t rows, int ld, int rb_bytes, int nslot, int64_t per_warp, uint32_t salt) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int rw = rb_bytes / 8;
  unsigned long long *ring = reinterpret_cast<unsigned long long *>(smem) + (size_t)w * nslot * RPI * rw;
  const uint32_t wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lpr = 32 / RPI;
  const int sub = lane / lpr, sl = lane % lpr;
  int slot = 0;
  for (int64_t i = 0; i < per_warp; i += RPI) {
    if (sl == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(3) : "memory");
    __syncwarp();
    unsigned long long *dst = ring + (size_t)(slot * RPI + sub) * rw;
    for (int c = sl; c < rw; c += lpr) dst[c] = (unsigned long long)i;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (sl == 0) {
      const int64_t row = rnd_row(wid, i + sub, salt, rows);
      unsigned long long *g = reinterpret_cast<unsigned long long *>(M) + row * ld;
      const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g), "r"(sa), "r"(rb_bytes)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    slot = (slot + 1) % nslot;
  }
  if (sl == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
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
  void *M;
  cudaMalloc(&M, (size_t)4 << 30);
  cudaMemset(M, 0, (size_t)4 << 30);
  const int64_t pw = 4096;
  for (int64_t rows : {int64_t(65536), int64_t(393216), int64_t(4821207)}) {
    {
      const int blocks = 148 * 8, threads = 256;
      const int64_t warps = (int64_t)blocks * threads / 32;
      float ms = time_it([&](uint32_t s) { k_red_u64<<<blocks, threads>>>((unsigned long long *)M, rows, r, ld, pw, s); }, 3);
      printf("red.u64 x25 lanes       rows=%8lld: %6.2f G rows/s\n", (long long)rows, warps * pw / ms / 1e6);
    }
    for (int cps : {1, 2, 4}) {
      for (int nslot : {4, 8}) {
        const int threads = 256, rb = 224;
        const int blocks = 148 * cps;
        const int64_t warps = (int64_t)blocks * threads / 32;
#define RUN(F64, RPI, NAME)                                                                                         \
  {                                                                                                                 \
    const size_t sm = (size_t)(threads / 32) * nslot * RPI * rb;                                                   \
    if (sm * cps <= 220 * 1024) {                                                                                   \
      cudaFuncSetAttribute(k_tma_red<F64, RPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);              \
      float ms = time_it([&](uint32_t s) { k_tma_red<F64, RPI><<<blocks, threads, sm>>>(M, rows, ld, rb, nslot, pw, s); }, 3); \
      printf("%-22s rows=%8lld ctas/sm=%d slots=%d: %6.2f G rows/s\n", NAME, (long long)rows, cps, nslot,          \
             warps * pw / ms / 1e6);                                                                                \
    }                                                                                                               \
  }
        RUN(false, 1, "tma red.u64 1 row/step");
        RUN(false, 4, "tma red.u64 4 rows/step");
        RUN(true, 4, "tma red.f64 4 rows/step");
        {
          const size_t sm = (size_t)(threads / 32) * nslot * 4 * rb;
          if (sm * cps <= 220 * 1024) {
            cudaFuncSetAttribute(k_tma_st<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            float ms = time_it([&](uint32_t s) { k_tma_st<4><<<blocks, threads, sm>>>(M, rows, ld, rb, nslot, pw, s); }, 3);
            printf("%-22s rows=%8lld ctas/sm=%d slots=%d: %6.2f G rows/s\n", "tma store 4 rows/step", (long long)rows,
                   cps, nslot, warps * pw / ms / 1e6);
          }
        }
      }
    }
  }
  // correctness: one row, known count
  {
    unsigned long long *m = (unsigned long long *)M;
    cudaMemset(m, 0, 4096);
    const size_t sm = 8 * 4 * 4 * 224;
    cudaFuncSetAttribute(k_tma_red<false, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k_tma_red<false, 4><<<2, 256, sm>>>(M, 1, ld, 224, 4, 64, 3);
    unsigned long long h[32];
    cudaMemcpy(h, m, sizeof h, cudaMemcpyDeviceToHost);
    printf("check: row0 col0 %llu col27 %llu col28 %llu (expect %llu %llu 0)\n", h[0], h[27], h[28], 3ull * 16 * 64,
           3ull * 16 * 64);
  }
  return 0;
}
